export TASKFUSE_NO_BUILD=1
O=gpurun_out/mh
mkdir -p $O
timeout 600 python scripts/exp_march_halo.py 512 > $O/exp.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --print-units base -k regex:k_step_march --launch-skip 6 -c 4 python scripts/exp_march_halo.py 512 > $O/ncu.csv 2>&1
echo done
