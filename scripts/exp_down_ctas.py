import sys
sys.path.insert(0, ".")
import torch
from paper_2210_06438_b200.field import FieldIteration, HostPipeline
from paper_2210_06438_b200.hydro import sod_field
G = 128
def t(fn, K=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / K
it = FieldIteration(G, 8, (1.0, 1.0, 1.0), max_team=128, executors=2)
hin = sod_field(G, "cpu").pin_memory(); hout = torch.empty_like(hin).pin_memory()
for dc in (4, 6, 8, 12, 16, 24):
    p = HostPipeline(it, hin, hout, down_ctas=dc)
    print(dc, round(t(p.run), 4), flush=True)
