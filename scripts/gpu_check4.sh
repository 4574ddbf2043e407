export TASKFUSE_NO_BUILD=1
O=gpurun_out/c4
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_strategy3.py -q -x > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-sweep --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
echo done
