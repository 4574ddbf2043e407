export TASKFUSE_NO_BUILD=1
O=gpurun_out/m1
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_march --launch-skip 2 -c 1 -o $O/march_full -f python scripts/exp_march_one.py 512 > $O/ncu.log 2>&1
timeout 600 python scripts/ab_march.py 8:0:16 > $O/ab.log 2>&1
echo done
