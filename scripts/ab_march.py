"""Interleaved A/B of config-5 fused-iteration kernels (grid 512): every
config timed in each of several rounds (CUDA events, 20 iterations), so a
drift of the box (clocks, power) hits all configs alike; median / min per
config and the SM clock under load."""
import statistics
import sys
sys.path.insert(0, ".")
import torch
import bench
from oracle import hydro_oracle as HO
from paper_2210_06438_b200.field import MarchFieldIteration, PeerSlabFieldIteration
from paper_2210_06438_b200.parallel_halo import SlabPartition

G = 512
dev = torch.device("cuda", 0)
f = torch.from_numpy(HO.initial_field(G)).to(dev)
cells = G ** 3
configs = {}
r = PeerSlabFieldIteration(SlabPartition(G, 8, 1, 0), None, device=dev,
                           kernel="cols")
r.load(f)
r._prime()
configs["peer cols"] = r.iteration
for spec in sys.argv[1:] or ["8:4:16", "8:5:16", "8:4:32"]:
    R, nb, xc = (int(x) for x in spec.split(":"))
    it = MarchFieldIteration(G, 8, device=dev, xc=xc, rows4=(R == 4))
    it.flags |= nb << 8
    it.load(f)
    configs[f"march R{R} nb{nb} xc{xc} #{len(configs)}"] = it.step


def once(fn, iters=20):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


for fn in configs.values():
    for _ in range(3):
        fn()
torch.cuda.synchronize()
res = {k: [] for k in configs}
with bench.ClockSampler(0) as clk:
    for rnd in range(6):
        keys = list(configs)
        if rnd % 2:
            keys.reverse()
        for k in keys:
            res[k].append(once(configs[k]))
floor = cells * 16 / 6524.6e9 * 1e3
for k, v in res.items():
    med, mn = statistics.median(v), min(v)
    print(f"{k:28s} median {med*1e3:7.1f} us  min {mn*1e3:7.1f} us  "
          f"frac16 {floor/med:.3f} " + " ".join(f"{x*1e3:.0f}" for x in v), flush=True)
print("clocks", clk.summary())
