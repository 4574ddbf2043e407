export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out/march
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_peer.py -q -x > gpurun_out/march/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/march/pytest.log
timeout 600 python scripts/exp_march.py 512 > gpurun_out/march/exp.log 2>&1
echo done
