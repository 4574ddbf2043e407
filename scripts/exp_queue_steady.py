"""Back-to-back real-time device-queue runs (config 2, A = 128) for an ncu
capture of the consumer grid in steady state (application replay: every
pass reruns this script, so the host publishes while the kernel runs)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents  # noqa

wl = bench.Workload()
arr = np.arange(wl.S, dtype=np.int32)
q = QueueExecutor("reconstruct", 128, default_parents(wl.S, 128), wl.n)
for k in range(12):
    q.run(wl.pools[k % 2], bench.VELOCITY, arr, wl.um, wl.up, wl.F,
          amax=wl.amax)
q.wait()
torch.cuda.synchronize()
print("ok")
