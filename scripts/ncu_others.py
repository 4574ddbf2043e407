"""One launch of each secondary kernel on config 2, for ncu captures:
PPM + upwind, PPM + KT, minmod + KT, ghost fill, update (materialising
path), prep, the fused step team launch."""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2210_06438_b200 import ops  # noqa: E402
from paper_2210_06438_b200.hydro.scenario import dt_over_dx  # noqa: E402

wl = bench.Workload()
for _ in range(2):
    bench.single_runner(wl, "ppm", 0)(0)
    bench.single_runner(wl, "ppm", 1)(0)
    bench.single_runner(wl, "minmod", 1)(0)
    ops.ghost_fill(wl.pools[0], wl.n, wl.grid // wl.n)
    nxt = torch.empty_like(wl.pools[1])
    ops.update(wl.pools[0], wl.n, wl.F, dt_over_dx(bench.VELOCITY), nxt)
torch.cuda.synchronize()
print("ok")
