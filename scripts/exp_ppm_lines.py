"""PPM reconstruct + KT (and upwind with a < 0) on config 2, one launch of
all 4096 slices: the phased kernel vs a thread per line
(TASKFUSE_PPM_LINES=0/1, read once per process)."""
import os
import sys
sys.path.insert(0, ".")
import torch
import bench

wl = bench.Workload()
peak = 6551.4
per = 8 * (14 ** 3 + 9 * 10 ** 3)
for name, ff, vel in (("ppm_kt", 1, bench.VELOCITY),
                      ("ppm_upwind_neg", 0, (-1.0, 0.5, -0.25))):
    old = bench.VELOCITY
    bench.VELOCITY = vel
    ms = bench.timed(bench.single_runner(wl, "ppm", ff), 30, 5, 1,
                     torch.cuda.current_stream())
    bench.VELOCITY = old
    print(f"lines={os.environ.get('TASKFUSE_PPM_LINES', '1')} {name:16s} "
          f"{ms*1e3:6.1f} us  {wl.S * per / (ms * 1e-3) / 1e9 / peak:.3f} of HBM",
          flush=True)
