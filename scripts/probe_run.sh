cd scripts
for eb in 8 4; do for r in 2 3 4; do timeout 60 ./tma_probe2 $eb $r; done; done > ../gpurun_out/tma_probe2.log 2>&1
echo done
