export TASKFUSE_NO_BUILD=1
O=gpurun_out/mxc
mkdir -p $O
for xc in 16 32 64; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --print-units base -k regex:k_step_march --launch-skip 2 -c 2 python scripts/exp_march_one.py 512 rows8 0 $xc > $O/ncu_xc$xc.csv 2>&1
done
echo done
