"""e2e variants: graph vs eager submission, zero-copy vs copy-engine download."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_06438_b200.field import FieldIteration, HostPipeline  # noqa
from paper_2210_06438_b200.hydro import sod_field  # noqa

G = 128


def t(fn, K=50):
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
for ch in ("taper", [1, 2, 3, 4, 3, 2, 1], [1, 1, 2, 4, 4, 2, 1, 1], 8):
    for dc in (16, 32, 0):
        for ds in (True,):
            def eager():
                it.cur = 0
                it.run_host_pipelined(hin, hout, ch, dc, ds)
            e = t(eager)
            p = HostPipeline(it, hin, hout, chunks=ch, down_ctas=dc,
                             down_stream=ds)
            g = t(p.run)
            print(f"chunks={ch} down_ctas={dc}: eager {e:.3f} graph {g:.3f}",
                  flush=True)
