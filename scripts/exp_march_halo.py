"""March kernel with the next field's y/z halos written in the kernel (the
face items' halo-writing loop) vs written by the y/z halo kernels after it
(every item then runs the unrolled interior loop, in chunk-major order).
Equality of the two after several iterations, then interleaved timing."""
import statistics
import sys
sys.path.insert(0, ".")
import torch
import bench
from oracle import hydro_oracle as HO
from paper_2210_06438_b200 import _lib
from paper_2210_06438_b200.field import MarchFieldIteration

G = int(sys.argv[1]) if len(sys.argv) > 1 else 512
dev = torch.device("cuda", 0)
f = torch.from_numpy(HO.initial_field(G)).to(dev)
a = MarchFieldIteration(G, 8, device=dev)
b = MarchFieldIteration(G, 8, device=dev)
a.load(f)
b.load(f)
lib = b.lib


def step_b():
    if not b.halo_fresh:
        b.halo(True)
    b.march(_lib.TF_STEP_HALO_X)
    nxt = b.P[1 - b.cur]
    _lib.check(lib.tf_field_halo_layers_f64(
        nxt.data_ptr(), b.X, b.G, b.G, 2, b.X,
        torch.cuda.current_stream().cuda_stream), "halo layers")
    b.swap()
    b.halo_fresh = True


for _ in range(3):
    a.step()
    step_b()
torch.cuda.synchronize()
print("owned equal after 3 iterations:", torch.equal(a.owned(), b.owned()),
      flush=True)


def once(fn, iters=20):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


res = {"halo in kernel": [], "halo kernels after": []}
with bench.ClockSampler(0) as clk:
    for rnd in range(6):
        order = list(res) if rnd % 2 == 0 else list(reversed(list(res)))
        for k in order:
            res[k].append(once(a.step if k == "halo in kernel" else step_b))
floor = G ** 3 * 16 / 6524.6e9 * 1e3
for k, v in res.items():
    print(f"{k:22s} median {statistics.median(v)*1e3:7.1f} us  min "
          f"{min(v)*1e3:7.1f} us  frac16 {floor/min(v):.3f}  "
          + " ".join(f"{x*1e3:.0f}" for x in v), flush=True)
print("clocks", clk.summary())
