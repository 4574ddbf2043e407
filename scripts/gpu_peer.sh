export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -q -x > gpurun_out/pytest_peer.log 2>&1; echo "exit $?" >> gpurun_out/pytest_peer.log
echo done
