export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m paper_2210_06438_b200.bench_matrix --grid-n 32 --executors 1 4 --max-team 1 4 16 64 --steps 3 --format markdown > gpurun_out/matrix_cfg1.md 2>&1
timeout 300 python -m paper_2210_06438_b200.bench_matrix --grid-n 32 --subgrid-n 16 --executors 1 4 --max-team 1 --steps 3 --format csv > gpurun_out/matrix_cfg1_16.csv 2>&1
timeout 900 python -m paper_2210_06438_b200.bench_matrix --grid-n 64 --executors 1 4 --max-team 1 16 64 128 --steps 2 --format markdown > gpurun_out/matrix_g64.md 2>&1
echo done
