export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
L=paper_2210_06438_b200/libtaskfuse_b200.so
cp $L /tmp/lib_new.so
for v in new old new old; do
  if [ $v = old ]; then cp exp_libs/lib_oldinit.so $L; else cp /tmp/lib_new.so $L; fi
  echo -n "$v " >> gpurun_out/r2g_recon.log; timeout 300 python scripts/exp_recon_time.py >> gpurun_out/r2g_recon.log 2>&1
done
cp /tmp/lib_new.so $L
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "recon_flux_bit_exact" > gpurun_out/r2g_race.log 2>&1
timeout 600 python scripts/exp_engine_cfg1.py > gpurun_out/r2g_engine.log 2>&1
echo done
