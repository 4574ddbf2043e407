import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2210_06438_b200 import ops
wl = bench.Workload()
st = torch.cuda.current_stream()
for vel in ((1.0, 1.0, 1.0), (-1.0, -1.0, -1.0), (-1.0, 0.5, -0.25)):
    for ff in (0, 1):
        def step(k, vel=vel, ff=ff):
            ops.recon_flux(wl.pools[k % 2], 8, vel, wl.um, wl.up, wl.F, out_mode=1, amax=wl.amax, flux_form=ff)
        ms = bench.timed(step, 50, 3, 1, st)
        print(vel, "kt" if ff else "upwind", round(wl.S * bench.b_alg(8) / (ms * 1e-3) / 6549.8e9, 3))
