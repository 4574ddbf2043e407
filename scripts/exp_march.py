"""A/B of the config-5 fused iteration kernels on one GPU (grid 512,
262 144 sub-grids): k_step_cols8s (one CTA per sub-grid, PeerSlab 'cols')
vs the whole-slab march kernel (rows 8 / 4, chunk lengths).  CUDA events,
median of 3 runs of 20 iterations each."""
import sys
sys.path.insert(0, ".")
import torch
from oracle import hydro_oracle as HO
from paper_2210_06438_b200 import _lib
from paper_2210_06438_b200.field import MarchFieldIteration, PeerSlabFieldIteration
from paper_2210_06438_b200.parallel_halo import SlabPartition

G = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dev = torch.device("cuda", 0)
f = torch.from_numpy(HO.initial_field(G)).to(dev)
cells = G ** 3


def timeit(fn, iters=20, reps=3):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / iters)
    out.sort()
    return out[len(out) // 2]


def report(name, ms):
    floor = cells * 16 / 6524.6e9 * 1e3
    print(f"{name:40s} {ms*1e3:8.1f} us  {cells/ms/1e6:7.1f} G/s  "
          f"frac16={floor/ms:.3f}", flush=True)


for kernel in ("cols", "march"):
    r = PeerSlabFieldIteration(SlabPartition(G, 8, 1, 0), None, device=dev,
                               kernel=kernel)
    r.load(f)
    r._prime()
    report(f"peer {kernel}", timeit(r.iteration))
    r.check()
    del r
for rows4, nb, xcs in ((False, 4, (16, 16, 16)), (False, 5, (16,))):
    for xc in xcs:
        it = MarchFieldIteration(G, 8, device=dev, xc=xc, rows4=rows4)
        it.flags |= nb << 8
        it.load(f)
        report(f"march rows{'4' if rows4 else '8'} nb{nb} xc{xc}",
               timeit(it.step))
        del it
torch.cuda.empty_cache()
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,power.draw,temperature.gpu", "--format=csv"], capture_output=True, text=True).stdout)
