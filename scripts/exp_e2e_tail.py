"""e2e pipeline (config 2, strategy3.ReconFluxHostPipeline) against its
floor: the 16.8 MB field upload alone (one copy, and in the pipeline's
chunks), and the pipeline with other layer tapers (how much of the step is
the tail after the last chunk lands)."""
import statistics
import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2210_06438_b200 import strategy3 as S3
from paper_2210_06438_b200.hydro import sod_field

it = S3.AggregatedIteration(bench.GRID, bench.N_SUB, bench.VELOCITY,
                            max_team=128, executors=2)
host_in = sod_field(bench.GRID, "cpu").pin_memory()
amax = torch.empty(it.S, dtype=torch.float64).pin_memory()
dev_f = it.field_dev
fin = host_in.view(bench.GRID, bench.GRID, bench.GRID)
n = bench.N_SUB


def upload_one():
    dev_f.copy_(fin, non_blocking=True)


def upload_chunks(layers=(1, 3, 4, 4, 3, 1)):
    def run():
        s = 0
        for k in layers:
            dev_f[s * n:(s + k) * n].copy_(fin[s * n:(s + k) * n],
                                           non_blocking=True)
            s += k
    return run


def upload_amax():
    dev_f.copy_(fin, non_blocking=True)
    amax[:it.S].copy_(it.amax, non_blocking=True)


cfgs = {"upload, one copy": upload_one,
        "upload, 6 chunks": upload_chunks(),
        "upload + amax back": upload_amax}
TAPERS = ((1, 3, 4, 4, 3, 1), (1, 4, 4, 4, 2, 1), (1, 5, 5, 4, 1),
          (1, 6, 6, 2, 1), (1, 7, 7, 1), (2, 6, 6, 1, 1), (1, 5, 5, 3, 1, 1))
for lay in TAPERS:
    for cs in ((1, 2) if lay == TAPERS[0] else (1,)):
        p = S3.ReconFluxHostPipeline(it, host_in, amax, layers=lay,
                                     copy_streams=cs)
        cfgs[f"pipe {'-'.join(map(str, lay))} cs{cs}"] = p.run


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
    print(f"{k:34s} median {statistics.median(v)*1e3:7.1f} us  "
          f"min {min(v)*1e3:7.1f} us", flush=True)
