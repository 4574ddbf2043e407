export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"k_recon_flux_ppm|k_recon_flux<|k_ghost_fill|k_update" -s 5 -c 5 -o gpurun_out/prof_others python scripts/ncu_others.py > gpurun_out/ncu_others.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_queue_consumer -s 3 -c 1 -o gpurun_out/prof_consumer python scripts/exp_consumer.py > gpurun_out/ncu_consumer.log 2>&1
tail -3 gpurun_out/ncu_others.log gpurun_out/ncu_consumer.log
