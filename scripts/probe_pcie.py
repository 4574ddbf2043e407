"""PCIe probe: H2D alone, D2H alone, both concurrently (16 MiB pinned)."""
import torch
n = 2 * 1024 * 1024
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, K=20):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / K
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
mb = n * 8 / 1e6
for name, fn in (("h2d", lambda: d1.copy_(h1, non_blocking=True)),
                 ("d2h", lambda: h2.copy_(d2, non_blocking=True)),
                 ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms  {mb / ms:.1f} GB/s per direction")
