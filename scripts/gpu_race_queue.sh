export TASKFUSE_NO_BUILD=1
O=gpurun_out/race
mkdir -p $O
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_strategy3.py -q -x -m gpu -k "queue" > $O/race_queue.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_parity.py tests/test_gpu_field.py tests/test_gpu_strategy3.py -q -x -m gpu -k "recon_flux_bit_exact or field_iteration_matches or device_launch" > $O/race_other.log 2>&1
echo done
