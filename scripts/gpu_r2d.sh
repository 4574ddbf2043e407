export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
for v in 1 2 1 2; do TASKFUSE_GHOST_V=$v timeout 300 python scripts/exp_ghost.py >> gpurun_out/r2d_ghost.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_hydrosim.py tests/test_gpu_bench_matrix.py tests/test_gpu_strategy3.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x --durations=10 > gpurun_out/r2d_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2d_pytest.log
timeout 600 python scripts/exp_refapi.py > gpurun_out/r2d_refapi.json 2> gpurun_out/r2d_refapi.err; echo "refapi exit $?" >> gpurun_out/r2d_refapi.err
timeout 300 python -m paper_2210_06438_b200.bench_matrix --executors 1 4 --max-team 1 8 64 --grid-n 64 --steps 2 --format markdown > gpurun_out/r2d_matrix_g64.md 2>&1
echo done
