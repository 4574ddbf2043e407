# compute-sanitizer over the parity tests (memcheck, racecheck, synccheck,
# initcheck), every kernel family: recon+flux, PPM, ghost fill, update,
# fused step, slab halos, queue consumer.
export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
S="compute-sanitizer --error-exitcode 9"
{
echo "== memcheck parity + PPM"; timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_ppm.py -q -x -m gpu -k "not config2 and not config3" 2>&1 | tail -4
echo "== memcheck field/halo/fuzz"; timeout 1200 $S --tool memcheck python -m pytest tests/test_gpu_field.py tests/test_gpu_halo.py "tests/test_gpu_fuzz.py::test_random_recon_flux_and_step[c0]" "tests/test_gpu_fuzz.py::test_random_recon_flux_and_step[c3]" -q -x 2>&1 | tail -4
echo "== memcheck strategy3 (plans, queue)"; timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_strategy3.py -q -x -k "form_teams or plan or field_pool or other_shapes" 2>&1 | tail -4
echo "== racecheck recon/PPM/field"; timeout 900 $S --tool racecheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_field.py tests/test_ppm.py -q -x -m gpu -k "recon_flux_bit_exact or two_kernel or field_iteration_matches or ppm_matches or ghost_fill" 2>&1 | tail -4
echo "== synccheck"; timeout 900 $S --tool synccheck python -m pytest tests/test_gpu_parity.py tests/test_ppm.py -q -x -m gpu -k "recon_flux_bit_exact or ppm_matches" 2>&1 | tail -4
echo "== initcheck"; timeout 900 $S --tool initcheck python -m pytest tests/test_gpu_parity.py -q -x -k "recon_flux_bit_exact or prep_reduce or ghost_fill" 2>&1 | tail -4
echo "== memcheck per-task HydroSim path + bench matrix (tests/test_gpu_hydrosim.py, test_gpu_bench_matrix.py, -k \"not matrix\")"; timeout 1200 $S --tool memcheck python -m pytest tests/test_gpu_hydrosim.py tests/test_gpu_bench_matrix.py -q -x -k "not matrix" 2>&1 | tail -3
echo "== memcheck multi-process peer path (tests/test_gpu_peer.py, --target-processes all)"; timeout 1200 $S --tool memcheck --target-processes all python -m pytest tests/test_gpu_peer.py -q -x 2>&1 | tail -3
echo "== racecheck fused step with halo writes (test_gpu_field.py -k halos)"; timeout 600 $S --tool racecheck python -m pytest tests/test_gpu_field.py -q -x -k "halos" 2>&1 | tail -2
} > gpurun_out/sanitize.log 2>&1
echo done
