export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_field.py -q -x > gpurun_out/pytest_e2e.log 2>&1; echo "exit $?" >> gpurun_out/pytest_e2e.log
timeout 300 python scripts/exp_e2e.py ${1:-} > gpurun_out/e2e.log 2>&1
