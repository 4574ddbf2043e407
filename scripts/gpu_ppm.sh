export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ppm.py -q -x -m gpu > gpurun_out/pytest_ppm.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ppm.log
echo done
