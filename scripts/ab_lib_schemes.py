"""One-launch recon+flux rates of the four schemes (minmod / PPM x upwind /
KT) on config 2 with the in-tree library, or (argv[1] = path) another
build saved for an A/B — run alternately in separate processes."""
import pathlib
import statistics
import sys
sys.path.insert(0, ".")
from paper_2210_06438_b200 import _lib
if len(sys.argv) > 1:
    _lib.LIB_PATH = pathlib.Path(sys.argv[1]).resolve()
import torch
import bench

wl = bench.Workload()
stream = torch.cuda.current_stream()
tag = sys.argv[1] if len(sys.argv) > 1 else "in-tree"
for name, rec, vel, ff in (("minmod_kt", "minmod", (1.0, 1.0, 1.0), 1),
                           ("ppm_upwind", "ppm", (1.0, 1.0, 1.0), 0),
                           ("ppm_upwind_neg", "ppm", (-1.0, 0.5, -0.3), 0),
                           ("ppm_kt", "ppm", (1.0, 1.0, 1.0), 1)):
    from paper_2210_06438_b200 import ops

    def step(k, rec=rec, vel=vel, ff=ff):
        ops.recon_flux(wl.pools[k % 2], wl.n, vel, wl.um, wl.up, wl.F,
                       out_mode=1, amax=wl.amax, flux_form=ff,
                       reconstruction=rec)
    v = [bench.timed(step, 20, 5, 1, stream) for _ in range(5)]
    print(f"{tag:12s} {name:16s} median {statistics.median(v)*1e3:6.1f} us"
          f"  min {min(v)*1e3:6.1f} us", flush=True)
