"""Queue consumer in isolation: every slice published (and the queue closed)
before the launch, so the kernel time is pure consumer throughput."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_06438_b200 import _lib  # noqa: E402

lib = _lib.load(build_if_missing=False)
wl = bench.Workload()
S = wl.S
ids = torch.arange(S, dtype=torch.int64)
ring_h = ids.clone().pin_memory()  # tagged per run: (epoch << 32) | id
ctl_h = torch.tensor([S, S, 0, 0, 0], dtype=torch.int64).pin_memory()
ring_d = torch.zeros(S + 2, dtype=torch.int64, device="cuda")  # tagged entries
# QueueDev: published, final_count, claim, done, one 128-B line each
init = torch.zeros(64, dtype=torch.int64, device="cuda")
qdev = init.clone()
st = torch.cuda.current_stream()




def run(k):
    ring_h.copy_(ids | ((k + 1) << 32))
    qdev.copy_(init)
    ctl_h[2] = 0
    rc = lib.tf_queue_consumer_launch(
        wl.pools[k % 2].data_ptr(), S, 8, ring_h.data_ptr(), ctl_h.data_ptr(),
        ring_d.data_ptr(), S, qdev.data_ptr(), 0, k + 1, 1.0, 1.0,
        1.0,
        wl.um.data_ptr(), wl.up.data_ptr(), wl.F.data_ptr(),
        wl.amax.data_ptr(), 0, 2_000_000_000, 0, st.cuda_stream)
    assert rc == 0, rc


for k in range(5):
    run(k)
    torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for k in range(20):
    ev[0].record()
    run(k)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
ts.sort()
print(f"consumer alone, all {S} slices pre-published: median {ts[10]:.1f} us "
      f"min {ts[0]:.1f} us (one CTA per slice)")
single = bench.single_runner(wl)
ts = []
for k in range(20):
    ev[0].record()
    single(k)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
ts.sort()
print(f"plain single launch: median {ts[10]:.1f} us min {ts[0]:.1f} us")
