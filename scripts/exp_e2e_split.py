"""e2e host->host recon+flux (config 2) with the field upload on 1 / 2 / 4
copy streams, plain and pipelined call, interleaved rounds on one box."""
import statistics
import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2210_06438_b200 import strategy3 as S3
from paper_2210_06438_b200.hydro import sod_field

it = S3.AggregatedIteration(bench.GRID, bench.N_SUB, bench.VELOCITY,
                            max_team=128, executors=2)
itq = S3.AggregatedIteration(bench.GRID, bench.N_SUB, bench.VELOCITY,
                             max_team=128, executors=1, formation="queue")
host_in = sod_field(bench.GRID, "cpu").pin_memory()
amax = torch.empty(it.S, dtype=torch.float64).pin_memory()
orig = S3.copy_split


def with_parts(p, fn):
    def run():
        S3.copy_split = lambda d, s, parts=p: orig(d, s, parts)
        try:
            fn()
        finally:
            S3.copy_split = orig
    return run


cfgs = {}
for p in (1, 2, 4):
    cfgs[f"plain parts={p}"] = with_parts(p, lambda: it.recon_flux_host(host_in, amax))
    cfgs[f"queue parts={p}"] = with_parts(p, lambda: itq.recon_flux_host(host_in, amax))
pipes = {}
for k in (1, 2, 4):
    # the pipeline's copy-stream count is fixed at construction
    src = open(S3.__file__).read()
    pipes[k] = None
for cs in (1, 2):
    pipe = S3.ReconFluxHostPipeline(it, host_in, amax, copy_streams=cs)
    cfgs[f"pipelined, {cs} copy stream(s)"] = pipe.run


def once(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


res = {k: [] for k in cfgs}
for rnd in range(4):
    for k in (list(cfgs) if rnd % 2 == 0 else list(reversed(list(cfgs)))):
        res[k].append(once(cfgs[k]))
for k, v in res.items():
    print(f"{k:30s} median {statistics.median(v)*1e3:7.1f} us  min {min(v)*1e3:7.1f} us")
