export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_field.py tests/test_gpu_peer.py -q -x > gpurun_out/pytest_fused.log 2>&1; echo "exit $?" >> gpurun_out/pytest_fused.log
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 300 python scripts/exp_e2e.py > gpurun_out/e2e.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -o gpurun_out/prof_fused2 python bench.py --workload cfg5 --cfg5-grid 256 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_fused.log 2>&1
