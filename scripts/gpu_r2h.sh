export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2h_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r2h_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo "bench exit $?" >> gpurun_out/r2h_bench.err
timeout 900 python bench.py --workload cfg5 --steps 20 --warmup 5 > gpurun_out/r2h_cfg5.json 2> gpurun_out/r2h_cfg5.err; echo "cfg5 exit $?" >> gpurun_out/r2h_cfg5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2h_ref.json 2> gpurun_out/r2h_ref.err; echo "ref exit $?" >> gpurun_out/r2h_ref.err
S="compute-sanitizer --error-exitcode 9"
{
echo "== racecheck recon/PPM/field/queue"; timeout 1200 $S --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_parity.py tests/test_gpu_field.py tests/test_ppm.py tests/test_gpu_strategy3.py -q -x -m gpu -k "recon_flux_bit_exact or two_kernel or field_iteration_matches or ppm_matches or ghost_fill or queue_executor_bit_exact or reference_geometry" 2>&1 | tail -4
echo "== memcheck native engine + pipeline"; timeout 1200 $S --tool memcheck python -m pytest tests/test_gpu_hydrosim.py tests/test_gpu_strategy3.py -q -x -k "native or pipelined or reference_geometry" 2>&1 | tail -3
} > gpurun_out/r2h_sanitize.log 2>&1
echo done
