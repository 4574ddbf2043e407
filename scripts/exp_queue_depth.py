"""A/B of the device-queue consumer's box ring depth (TASKFUSE_QUEUE_DEPTH
is read once per process): ms per 4096 real-time arrivals, A sweep, plus
correctness against the one-launch kernel."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_06438_b200 import ops  # noqa: E402
from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents  # noqa

wl = bench.Workload(field="stress") if False else bench.Workload()
arr = np.arange(wl.S, dtype=np.int32)
stream = torch.cuda.current_stream()
ref = [torch.empty_like(wl.um) for _ in range(3)]
ops.recon_flux(wl.pools[0], 8, bench.VELOCITY, *ref, out_mode=1)
res = {}
for A in (1, 4, 16, 64, 128):
    q = QueueExecutor("reconstruct", A, default_parents(wl.S, A), wl.n)
    step = lambda k: q.run(wl.pools[k % 2], bench.VELOCITY, arr, wl.um,  # noqa
                           wl.up, wl.F, amax=wl.amax)
    ms = bench.timed(step, 40, 10, 1, stream)
    q.wait()
    wl.um.fill_(float("nan"))
    q.run(wl.pools[0], bench.VELOCITY, arr, wl.um, wl.up, wl.F, amax=wl.amax)
    q.wait()
    ok = torch.equal(wl.um, ref[0])
    st = q.stats()
    mean = sum(k * v for k, v in st["size_histogram"].items()) / \
        st["teams_formed"]
    res[A] = (round(ms * 1e3, 1), round(bench.rate(wl.S, 8, ms) / 1e9, 2),
              round(mean, 1), ok)
    del q
print("depth", __import__("os").environ.get("TASKFUSE_QUEUE_DEPTH", "2"),
      res, flush=True)
