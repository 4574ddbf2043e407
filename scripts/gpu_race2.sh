export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
for k in "queue_executor_bit_exact" "device_launch" "reference_geometry"; do
  echo "== $k" >> gpurun_out/race2.log
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 3 python -m pytest tests/test_gpu_strategy3.py -q -x -k "$k" 2>&1 | grep -v "Host Frame" | grep -A8 "Warning\|Error\|SUMMARY" | head -40 >> gpurun_out/race2.log
done
for t in "tests/test_gpu_parity.py -k recon_flux_bit_exact" "tests/test_gpu_field.py -k field_iteration_matches" "tests/test_ppm.py -k ppm_matches" "tests/test_gpu_parity.py -k ghost_fill" "tests/test_gpu_parity.py -k two_kernel"; do
  echo "== $t" >> gpurun_out/race2.log
  timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 3 python -m pytest $t -q -x -m gpu 2>&1 | grep -v "Host Frame" | grep -A8 "Warning\|Error\|SUMMARY" | head -40 >> gpurun_out/race2.log
done
echo done
