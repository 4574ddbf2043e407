export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_strategy3.py -q -x -k "device_launch or queue" > gpurun_out/r2i_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2i_pytest.log
timeout 600 python scripts/exp_dlexec.py > gpurun_out/r2i_dlexec.log 2>&1
echo done
