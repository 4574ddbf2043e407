"""e2e experiment: download CTA count per chunk (0 = copy engine) in the
tapered host pipeline — does throttling the zero-copy download while the
last uploads are in flight shorten the tail?  (Ran against a
run_host_pipelined that took a per-chunk CTA list; no variant beat a
uniform 16, so that option was not kept — lists fail on the current code.)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_06438_b200.field import FieldIteration, HostPipeline  # noqa
from paper_2210_06438_b200.hydro import sod_field  # noqa

G = 128


def t(fn, K=100):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


it = FieldIteration(G, 8, (1.0, 1.0, 1.0), max_team=128, executors=1)
hin = sod_field(G, "cpu").pin_memory()
hout = torch.empty_like(hin).pin_memory()
variants = [16, [16, 16, 16, 16, 16, 32], [16, 16, 16, 8, 8, 32],
            [16, 16, 12, 12, 12, 32], [16, 16, 16, 16, 16, 0],
            [24, 16, 16, 12, 8, 32], [16, 16, 16, 16, 8, 32],
            [32, 24, 16, 16, 16, 32]]
for rep in range(2):
    for dc in variants:
        p = HostPipeline(it, hin, hout, chunks="taper", down_ctas=dc)
        print(f"down_ctas={dc}: {t(p.run):.4f} ms", flush=True)
