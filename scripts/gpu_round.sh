# Round evidence: GPU tests, smoke, bench (both arms), launch list, ncu captures.
export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?" >> gpurun_out/bench_ref.err
timeout 900 python bench.py --workload cfg5 --steps 20 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
# launch list of the bench's timed hot path (plan A=128)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
# full captures: one-launch recon+flux, one team launch, fused step (grid 256)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_recon_flux -s 2 -c 1 -o gpurun_out/prof_single python bench.py --profile-only --mode single --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_recon_flux -s 40 -c 1 -o gpurun_out/prof_team python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_team.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_cols8s -s 3 -c 1 -o gpurun_out/prof_fused python bench.py --workload cfg5 --cfg5-grid 256 --steps 2 --warmup 3 > gpurun_out/ncu_fused.log 2>&1
echo done
