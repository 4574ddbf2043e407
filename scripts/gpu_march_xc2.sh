export TASKFUSE_NO_BUILD=1
O=gpurun_out/mxc2
mkdir -p $O
timeout 900 python scripts/ab_march.py 8:0:16 8:0:8 8:0:12 8:0:10 > $O/ab.log 2>&1
for xc in 8 12; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --print-units base -k regex:k_step_march --launch-skip 2 -c 1 python scripts/exp_march_one.py 512 rows8 0 $xc > $O/ncu_xc$xc.csv 2>&1
done
echo done
