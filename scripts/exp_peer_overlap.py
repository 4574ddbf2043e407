"""Config 5 on one GPU through the peer path (the N > 1 headline's code):
march + ring barrier per iteration, with / without the PDL overlap of the
barrier and the next iteration's interior (overlap_barrier)."""
import statistics
import sys
sys.path.insert(0, ".")
import torch
import bench
from oracle import hydro_oracle as HO
from paper_2210_06438_b200.field import PeerSlabFieldIteration
from paper_2210_06438_b200.parallel_halo import SlabPartition

G = 512
dev = torch.device("cuda", 0)
part = SlabPartition(G, 8, 1, 0)
slab = bench.cfg5_slab(part, G)
its = {}
for ov in (False, True):
    try:
        its[ov] = PeerSlabFieldIteration(part, slab, bench.VELOCITY,
                                         device=dev, overlap_barrier=ov)
    except TypeError:
        its[ov] = PeerSlabFieldIteration(part, slab, bench.VELOCITY,
                                         device=dev)
for it in its.values():
    for _ in range(3):
        it.iteration()
torch.cuda.synchronize()
print("equal after 3 iterations:", torch.equal(its[False].owned(),
                                               its[True].owned()), flush=True)


def once(fn, iters=20):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


res = {k: [] for k in its}
for rnd in range(6):
    for k in (list(its) if rnd % 2 == 0 else list(reversed(list(its)))):
        res[k].append(once(its[k].iteration))
for k, v in res.items():
    print(f"overlap_barrier={k}: median {statistics.median(v)*1e3:.1f} us "
          f"min {min(v)*1e3:.1f} us  " + " ".join(f"{x*1e3:.0f}" for x in v),
          flush=True)
for it in its.values():
    it.check()
