export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 ncu --replay-mode application --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:k_queue_consumer -s 6 -c 4 --csv python scripts/exp_queue_steady.py > gpurun_out/r2m_ncu_queue.csv 2> gpurun_out/r2m_ncu_queue.err
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_step_cols8s -s 3 -c 1 -o gpurun_out/r2m_step_cfg5 python bench.py --workload cfg5 --steps 3 --warmup 3 --cfg5-grid 512 > gpurun_out/r2m_ncu_step.log 2>&1
ncu -i gpurun_out/r2m_step_cfg5.ncu-rep --page raw --csv > gpurun_out/r2m_step_cfg5_raw.csv 2>/dev/null
rm -f gpurun_out/r2m_step_cfg5.ncu-rep
echo done
