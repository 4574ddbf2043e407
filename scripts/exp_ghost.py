"""Ghost-fill kernel timing (TASKFUSE_GHOST_V=1 selects the index-math
gather; default the compile-time shell table): config 2 and config 3 pools,
CUDA events, algorithmic bytes 16 B per ghost cell."""
import os
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_06438_b200 import ops  # noqa: E402
from paper_2210_06438_b200.hydro import pool_from_field, sod_field  # noqa

peak = bench.peaks()[0]
out = {}
for grid in (128, 256):
    n = 8
    m = grid // n
    pools = [pool_from_field(sod_field(grid, "cuda"), n) for _ in range(2)]
    stream = torch.cuda.current_stream()
    ms = bench.timed(lambda k: ops.ghost_fill(pools[k % 2], n, m), 30, 5, 1,
                     stream)
    ghost = (n + 6) ** 3 - n ** 3
    alg = m ** 3 * ghost * 16
    out[grid] = (round(ms * 1e3, 1), round(alg / (ms * 1e-3) / 1e9 / peak, 3))
print("ghost", os.environ.get("TASKFUSE_GHOST_V", "shell"), out, flush=True)
