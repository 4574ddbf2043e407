"""cProfile of the per-task API path (bench_matrix.run_cell, config 1)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_2210_06438_b200.bench_matrix import run_cell  # noqa

A = int(sys.argv[1]) if len(sys.argv) > 1 else 1
run_cell(8, 1, A, 1, grid_n=32)
pr = cProfile.Profile()
pr.enable()
row, _, _ = run_cell(8, 1, A, 2, grid_n=32)
pr.disable()
print(row)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
st.sort_stats("cumulative").print_stats(40)
