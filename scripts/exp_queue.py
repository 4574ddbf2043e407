"""Real-time device-queue executor: host formation time vs GPU time."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents  # noqa

wl = bench.Workload()
arr = np.arange(wl.S, dtype=np.int32)
for A, early, srt in ((1, True, False), (4, True, False), (128, True, False),
                      (1, True, True), (4, True, True), (128, True, True)):
    q = QueueExecutor("reconstruct", A, default_parents(wl.S, A), wl.n,
                      early_loads=early, sorted_dispatch=srt)
    for k in range(10):
        q.run(wl.pools[k % 2], bench.VELOCITY, arr, wl.um, wl.up, wl.F,
              amax=wl.amax)
    torch.cuda.synchronize()
    K = 50
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    host = []
    e0.record()
    for k in range(K):
        t = time.perf_counter()
        q.run(wl.pools[k % 2], bench.VELOCITY, arr, wl.um, wl.up, wl.F,
              amax=wl.amax)
        host.append(time.perf_counter() - t)
    e1.record()
    torch.cuda.synchronize()
    gpu = e0.elapsed_time(e1) / K
    st = q.stats()
    print(f"A={A} early={early} sorted={srt}: gpu {gpu*1e3:.1f} us/iter, host q.run median "
          f"{np.median(host)*1e6:.1f} us (min {min(host)*1e6:.1f}), "
          f"{q.host_times()}, "
          f"teams {st['teams_formed']}, solo {st['solo_fast_path']}", flush=True)
    del q

# timeline of a few runs (kernel durations and gaps)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
import json  # noqa: E402
A = 64
q = QueueExecutor("reconstruct", A, default_parents(wl.S, A), wl.n)
for k in range(10):
    q.run(wl.pools[k % 2], bench.VELOCITY, arr, wl.um, wl.up, wl.F, amax=wl.amax)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for k in range(6):
        q.run(wl.pools[k % 2], bench.VELOCITY, arr, wl.um, wl.up, wl.F,
              amax=wl.amax)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/queue_trace.json")
ev = [e for e in json.load(open("gpurun_out/queue_trace.json"))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in ev)
for e in sorted(ev, key=lambda e: e["ts"]):
    print(f"{e['ts'] - t0:8.1f} {e['dur']:7.1f} {e['name'][:50]}")
