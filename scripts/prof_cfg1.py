"""cProfile of the per-task API path (config 1 through HydroSim on the B200)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_2210_06438_b200.bench_matrix import run_cell  # noqa: E402

for cap in (1, 16):
    row, _, _ = run_cell(8, 1, cap, 2, grid_n=32)
    print(f"cap {cap}: {row.ms_per_step} ms/step (unprofiled)")
pr = cProfile.Profile()
pr.enable()
row, _, _ = run_cell(8, 1, 16, 2, grid_n=32)
pr.disable()
print(f"profiled cap 16: {row.ms_per_step} ms/step")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
