export TASKFUSE_NO_BUILD=1
O=gpurun_out/pov3
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_peer.py tests/test_gpu_march.py tests/test_gpu_fullsize.py tests/test_gpu_bench_line.py -q -x > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 600 python scripts/exp_peer_overlap.py > $O/overlap.log 2>&1
timeout 600 python scripts/ab_march.py 8:0:16 > $O/ab.log 2>&1
timeout 900 python bench.py --workload cfg5 --steps 20 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "cfg5 exit $?" >> $O/bench_cfg5.err
echo done
