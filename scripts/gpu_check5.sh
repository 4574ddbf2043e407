export TASKFUSE_NO_BUILD=1
O=gpurun_out/c5
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_strategy3.py tests/test_gpu_field.py tests/test_gpu_peer.py tests/test_gpu_march.py -q -x > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
python scripts/probe_h2d_streams.py > $O/probe.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 900 python bench.py --workload cfg5 --steps 20 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "cfg5 exit $?" >> $O/bench_cfg5.err
echo done
