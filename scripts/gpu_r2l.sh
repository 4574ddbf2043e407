export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 python scripts/exp_cdp_effect.py > gpurun_out/r2l_cdp.log 2>&1
echo done
