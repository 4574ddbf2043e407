export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out/march
timeout 900 python scripts/ab_march.py "$@" > gpurun_out/march/ab.log 2>&1
echo done
