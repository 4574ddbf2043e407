export TASKFUSE_NO_BUILD=1
O=gpurun_out/${1:-m3}
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_march --launch-skip 2 -c 1 -o $O/march_full -f python scripts/exp_march_one.py 512 > $O/ncu.log 2>&1
echo done
