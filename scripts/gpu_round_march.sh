export TASKFUSE_NO_BUILD=1
O=gpurun_out/rm
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_fullsize.py tests/test_gpu_peer.py tests/test_gpu_field.py tests/test_gpu_bench_line.py -q -x > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 900 python bench.py --workload cfg5 --steps 20 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "exit $?" >> $O/bench_cfg5.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_march --launch-skip 2 -c 1 -o $O/march_full -f python scripts/exp_march_one.py 512 > $O/ncu.log 2>&1
echo done
