export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 300 python scripts/exp_e2e.py > gpurun_out/e2e.log 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 300 python scripts/exp_e2e.py > gpurun_out/e2e_conn32.log 2>&1
