# Round evidence on one B200: tests, smoke, every bench arm and workload, the
# ncu graph-traffic capture and launch list, sanitizers, the per-task matrix.
export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/final
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref exit $?" >> $O/bench_ref.err
timeout 900 python bench.py --workload cfg5 --steps 20 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "cfg5 exit $?" >> $O/bench_cfg5.err
TASKFUSE_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 > $O/bench_2rank_gloo.json 2> $O/bench_2rank_gloo.err; echo "2rank exit $?" >> $O/bench_2rank_gloo.err
timeout 900 ncu --graph-profiling graph --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --launch-skip 40 --launch-count 6 --csv python bench.py --profile-only --steps 20 --warmup 10 > $O/ncu_plan_graph.csv 2> $O/ncu_plan_graph.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --profile-only --steps 2 --warmup 3 > $O/launches.csv 2> $O/launches.err
S="compute-sanitizer --error-exitcode 9"
{
echo "== racecheck: recon / PPM / field / queue / reference geometry / device launch"; timeout 1200 $S --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_parity.py tests/test_gpu_field.py tests/test_ppm.py tests/test_gpu_strategy3.py -q -x -m gpu -k "recon_flux_bit_exact or two_kernel or field_iteration_matches or ppm_matches or ghost_fill or queue_executor_bit_exact or reference_geometry or device_launch" 2>&1 | tail -4
echo "== memcheck: parity + PPM"; timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_ppm.py -q -x -m gpu -k "not config2 and not config3" 2>&1 | tail -3
echo "== memcheck: native engine, pipelined e2e, reference geometry, device launch, queue"; timeout 1200 $S --tool memcheck python -m pytest tests/test_gpu_hydrosim.py tests/test_gpu_strategy3.py -q -x -k "native or pipelined or reference_geometry or device_launch or queue" 2>&1 | tail -3
echo "== synccheck"; timeout 900 $S --tool synccheck python -m pytest tests/test_gpu_parity.py tests/test_ppm.py -q -x -m gpu -k "recon_flux_bit_exact or ppm_matches" 2>&1 | tail -3
echo "== initcheck"; timeout 900 $S --tool initcheck python -m pytest tests/test_gpu_parity.py -q -x -k "recon_flux_bit_exact or prep_reduce or ghost_fill" 2>&1 | tail -3
} > $O/compute_sanitizer.log 2>&1
timeout 600 python -m paper_2210_06438_b200.bench_matrix --executors 1 2 --max-team 1 8 64 --grid-n 32 --steps 3 --format markdown > $O/bench_matrix_cfg1.md 2>&1
timeout 900 python -m paper_2210_06438_b200.bench_matrix --executors 1 4 --max-team 1 8 64 --grid-n 64 --steps 2 --format markdown > $O/bench_matrix_g64.md 2>&1
echo done
