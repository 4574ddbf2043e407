export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_hydrosim.py tests/test_gpu_bench_matrix.py tests/test_gpu_strategy3.py -q -x > gpurun_out/pytest_hs.log 2>&1; echo "exit $?" >> gpurun_out/pytest_hs.log
timeout 600 python -m paper_2210_06438_b200.bench_matrix --grid-n 32 --executors 1 4 --max-team 1 4 16 64 --steps 3 --format markdown > gpurun_out/matrix_cfg1.md 2>&1
timeout 300 python scripts/prof_matrix.py 1 > gpurun_out/prof_matrix.log 2>&1
