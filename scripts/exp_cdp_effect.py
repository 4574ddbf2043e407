"""Does running the device-launch executor once change later timings?
e2e recon_flux pipeline + plan A=128 before / after one dlexec run."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_06438_b200.hydro import sod_field  # noqa: E402
from paper_2210_06438_b200.strategy3 import (AggregatedIteration,  # noqa
                                             DeviceLaunchExecutor,
                                             ReconFluxHostPipeline,
                                             default_parents)

stream = torch.cuda.current_stream()
wl = bench.Workload()
it = AggregatedIteration(128, 8, (1.0, 1.0, 1.0), max_team=128, executors=2)
host_in = sod_field(128, "cpu").pin_memory()
amax = torch.empty(it.S, dtype=torch.float64).pin_memory()
pipe = ReconFluxHostPipeline(it, host_in, amax)
plan_step = bench.plan_runner(wl, 128, 2, team_buffers=True)[0]


def measure(tag):
    e = bench.timed(lambda k: pipe.run(), 20, 5, 1, stream)
    p = bench.timed(plan_step, 20, 5, 1, stream)
    u = bench.timed(lambda k: it.recon_flux_host(host_in, amax), 20, 5, 1,
                    stream)
    print(f"{tag}: e2e pipeline {e * 1e3:.1f} us, plain {u * 1e3:.1f} us, "
          f"plan {p * 1e3:.1f} us", flush=True)


measure("fresh")
measure("fresh again")
ex = DeviceLaunchExecutor("reconstruct", 128, default_parents(wl.S, 128), 8)
ex.run(wl.pools[0], bench.VELOCITY, np.arange(wl.S, dtype=np.int32), wl.um,
       wl.up, wl.F, amax=wl.amax)
ex.wait()
measure("after dlexec")
