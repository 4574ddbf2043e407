export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
for d in 2 1 2 1; do TASKFUSE_QUEUE_DEPTH=$d timeout 300 python scripts/exp_queue_depth.py >> gpurun_out/r2n_queue.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_strategy3.py -q -x -k "queue" > gpurun_out/r2n_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2n_pytest.log
echo done
