export TASKFUSE_NO_BUILD=1
O=gpurun_out/c3
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_strategy3.py tests/test_gpu_bench_line.py -q -x > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
echo done
