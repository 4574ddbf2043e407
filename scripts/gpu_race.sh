export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_parity.py -q -x -k "recon_flux_bit_exact" > gpurun_out/race_recon.log 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_field.py -q -x -k "field_iteration_matches_reference and 16-8" > gpurun_out/race_field.log 2>&1
echo done
