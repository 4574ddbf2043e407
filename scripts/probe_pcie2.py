"""PCIe probe 2: copy engines split over streams vs zero-copy kernels.

Usage (GPU box): python scripts/probe_pcie2.py   (builds scripts/_pcie_probe.so
here first if missing: nvcc -shared ...)."""
import ctypes
import os
import subprocess
import sys

import torch

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "_pcie_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC",
                           "-gencode", "arch=compute_100a,code=sm_100a",
                           os.path.join(here, "pcie_probe.cu"), "-o", so])
if not torch.cuda.is_available():
    sys.exit(0)
lib = ctypes.CDLL(so)
lib.probe_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p]

n = 128 ** 3
h1 = torch.rand(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.rand(n, dtype=torch.float64, device="cuda")
mb = n * 8 / 1e6


def t(fn, K=20):
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


def rep(name, ms, factor=1):
    print(f"{name:44s} {ms:.3f} ms  {factor * mb / ms:.1f} GB/s", flush=True)


rep("CE h2d 1 stream", t(lambda: d1.copy_(h1, non_blocking=True)))
rep("CE d2h 1 stream", t(lambda: h2.copy_(d2, non_blocking=True)))
for k in (2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(k)]

    def split(dst, src, ss=ss, k=k):
        cur = torch.cuda.current_stream()
        c = n // k
        for i, s in enumerate(ss):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                dst[i * c:(i + 1) * c].copy_(src[i * c:(i + 1) * c],
                                             non_blocking=True)
        for s in ss:
            cur.wait_stream(s)
    rep(f"CE h2d split over {k} streams", t(lambda: split(d1, h1)))
    rep(f"CE d2h split over {k} streams", t(lambda: split(h2, d2)))

cs = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
for blocks in (148, 296, 592, 1184):
    for threads in (256, 512):
        rep(f"ZC read  host->dev kernel {blocks}x{threads}",
            t(lambda: lib.probe_copy(h1.data_ptr(), d1.data_ptr(), n * 8,
                                     blocks, threads, cs())))
        rep(f"ZC write dev->host kernel {blocks}x{threads}",
            t(lambda: lib.probe_copy(d2.data_ptr(), h2.data_ptr(), n * 8,
                                     blocks, threads, cs())))
assert torch.equal(d1.cpu(), h1)
torch.cuda.synchronize()
assert torch.equal(h2, d2.cpu())

s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both_zc():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    lib.probe_copy(h1.data_ptr(), d1.data_ptr(), n * 8, 592, 512,
                   s1.cuda_stream)
    lib.probe_copy(d2.data_ptr(), h2.data_ptr(), n * 8, 592, 512,
                   s2.cuda_stream)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def both_ce():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


rep("both directions, copy engines (per dir)", t(both_ce))
rep("both directions, zero-copy kernels (per dir)", t(both_zc))


def ce_up_zc_down():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    lib.probe_copy(d2.data_ptr(), h2.data_ptr(), n * 8, 148, 512,
                   s2.cuda_stream)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def zc_up_ce_down():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    lib.probe_copy(h1.data_ptr(), d1.data_ptr(), n * 8, 148, 512,
                   s1.cuda_stream)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


rep("both: CE up + ZC-kernel down (per dir)", t(ce_up_zc_down))
rep("both: ZC-kernel up + CE down (per dir)", t(zc_up_ce_down))
for name, fn in (("CE both", both_ce), ("CE up + ZC down", ce_up_zc_down)):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        fn()
    rep(f"graph-captured {name} (per dir)", t(g.replay))
