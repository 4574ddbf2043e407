export TASKFUSE_NO_BUILD=1
O=gpurun_out/q13
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_strategy3.py tests/test_gpu_hydrosim.py tests/test_gpu_bench_line.py -q -x  > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 300 python scripts/exp_consumer_chain.py > $O/chain.log 2>&1
timeout 300 python scripts/exp_queue.py > $O/queue.log 2>&1
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
echo done
