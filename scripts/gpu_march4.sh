export TASKFUSE_NO_BUILD=1
O=gpurun_out/${1:-m4}
mkdir -p $O
timeout 900 python scripts/ab_march.py 8:0:16 4:0:16 8:0:32 4:0:32 > $O/ab.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,power.draw,power.limit,temperature.gpu --format=csv >> $O/ab.log
echo done
