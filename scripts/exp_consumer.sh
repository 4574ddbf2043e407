export TASKFUSE_NO_BUILD=1
timeout 600 python -m pytest tests/test_gpu_strategy3.py tests/test_gpu_hydrosim.py -q -x 2>&1 | tail -1
timeout 120 python scripts/exp_consumer.py
timeout 300 python scripts/exp_queue.py 2>&1 | grep "A="
