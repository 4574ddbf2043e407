"""Where a config-1 HydroSim step goes in the native engine: host time
issuing device ops, idle polling, per iteration; E x A variants."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2210_06438_b200.bench_matrix import run_cell  # noqa: E402
from paper_2210_06438_b200.hydro import sod_field  # noqa: E402

for grid, E, A in ((32, 1, 1), (32, 1, 64), (32, 2, 1), (64, 1, 1),
                   (128, 1, 64)):
    row, sim, dev = run_cell(8, E, A, steps=3, grid_n=grid,
                             field=sod_field(grid, "cuda"))
    ht = sim.native.host_times()
    c = sim.native.counters()
    its = 3 * 4
    print(f"grid {grid} E{E} A{A}: {row.ms_per_step:.2f} ms/step, "
          f"kernels/step {row.kernels}, per iteration: "
          f"{ht['iteration_ns'] / its / 1e3:.0f} us, issue "
          f"{ht['issue_ns'] / its / 1e3:.0f} us, idle poll "
          f"{ht['idle_poll_ns'] / its / 1e3:.0f} us, polls/iter "
          f"{c['polls'] / its:.0f}", flush=True)
