"""Device-launch executor vs device queue vs plan (config 2), A sweep."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_06438_b200.strategy3 import (DeviceLaunchExecutor,  # noqa
                                             QueueExecutor, default_parents)

wl = bench.Workload()
arr = np.arange(wl.S, dtype=np.int32)
stream = torch.cuda.current_stream()
for name, cls in (("dlexec", DeviceLaunchExecutor), ("queue", QueueExecutor)):
    res = {}
    for A in (1, 4, 16, 64, 128):
        ex = cls("reconstruct", A, default_parents(wl.S, A), wl.n)

        def step(k, ex=ex):
            ex.run(wl.pools[k % 2], bench.VELOCITY, arr, wl.um, wl.up, wl.F,
                   amax=wl.amax)
        ms = bench.timed(step, 20, 5, 1, stream)
        ex.wait()
        st = ex.stats()
        mean = sum(k * v for k, v in st["size_histogram"].items()) / \
            st["teams_formed"]
        res[A] = (round(ms * 1e3, 1), round(bench.rate(wl.S, 8, ms) / 1e9, 2),
                  round(mean, 1))
        del ex
    print(name, res, flush=True)
