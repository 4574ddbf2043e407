export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
S="compute-sanitizer --error-exitcode 9"
{
echo "== memcheck parity"; timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_parity.py -q -x -k "not config2 and not config3" 2>&1 | tail -4
echo "== memcheck field/halo"; timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_field.py tests/test_gpu_halo.py -q -x 2>&1 | tail -4
echo "== memcheck strategy3"; timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_strategy3.py -q -x -k "form_teams or plan or field_pool" 2>&1 | tail -4
echo "== racecheck recon/field"; timeout 900 $S --tool racecheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_field.py -q -x -k "recon_flux_bit_exact or two_kernel or field_iteration_matches" 2>&1 | tail -4
echo "== synccheck"; timeout 900 $S --tool synccheck python -m pytest tests/test_gpu_parity.py -q -x -k "recon_flux_bit_exact" 2>&1 | tail -4
echo "== initcheck"; timeout 900 $S --tool initcheck python -m pytest tests/test_gpu_parity.py -q -x -k "recon_flux_bit_exact or prep_reduce" 2>&1 | tail -4
} > gpurun_out/sanitize.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_fused -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --workload cfg5 --cfg5-grid 256 --steps 2 --warmup 3 > gpurun_out/ncu_fused.log 2>&1
echo done
