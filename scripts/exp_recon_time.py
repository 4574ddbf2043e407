"""recon+flux one launch and A=128 plan timing (config 2), for A/B runs."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.Workload()
stream = torch.cuda.current_stream()
peak = bench.peaks()[0]
res = {}
for name, step in (("single", bench.single_runner(wl)),
                   ("plan128", bench.plan_runner(wl, 128, 2,
                                                 team_buffers=True)[0])):
    ms = min(bench.timed(step, 30, 10, 1, stream) for _ in range(3))
    res[name] = (round(ms * 1e3, 1),
                 round(wl.S * bench.b_alg(8) / (ms * 1e-3) / 1e9 / peak, 3))
print("recon", res, flush=True)
