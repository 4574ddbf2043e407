export TASKFUSE_NO_BUILD=1
O=gpurun_out/q10
mkdir -p $O
timeout 300 python scripts/exp_consumer_chain.py > $O/chain.log 2>&1
echo done
timeout 600 python -m pytest tests/test_gpu_strategy3.py -q -x -k "queue" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 300 python scripts/exp_queue.py > $O/queue.log 2>&1
