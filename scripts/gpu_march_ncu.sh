export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out/march
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_march --launch-skip 2 -c 1 -o gpurun_out/march/march_full -f python scripts/exp_march_one.py 512 > gpurun_out/march/ncu.log 2>&1
echo done
