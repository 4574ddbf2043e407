"""Config-2 fused full iteration (team plans, halo-writing step): time per
iteration for a few team sizes / executor counts."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_06438_b200.field import FieldIteration  # noqa
from paper_2210_06438_b200.hydro import sod_field  # noqa


def t(fn, K=200):
    for _ in range(10):
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


for A, E in ((128, 2), (128, 4), (128, 1), (64, 4)):
    it = FieldIteration(128, 8, (1.0, 1.0, 1.0), max_team=A, executors=E)
    it.load(sod_field(128, "cuda"))
    print(f"A={A} E={E}: {1e3 * t(it.step):.2f} us", flush=True)
