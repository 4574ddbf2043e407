"""e2e experiment: HostPipeline chunk counts vs the PCIe lower bound."""
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
d1 = torch.empty_like(hin, device="cuda")
d2 = torch.empty_like(hin, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d1.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


print(f"h2d alone {t(lambda: d1.copy_(hin, non_blocking=True)):.3f} ms")
print(f"d2h alone {t(lambda: hout.copy_(d2, non_blocking=True)):.3f} ms")
print(f"h2d+d2h concurrent {t(both):.3f} ms")
print(f"device step {t(it.step):.3f} ms")
print(f"run_host (serial) {t(lambda: it.run_host(hin, hout)):.3f} ms")
def graph_of(fn):
    it.cur = 0
    fn()
    it.cur = 0
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=st):
        fn()
    it.cur = 0
    torch.cuda.synchronize()
    return g


for ch in ([1, 3, 4, 4, 3, 1], [1, 2, 3, 4, 3, 2, 1], 8, 16):
    g = graph_of(lambda: it.run_host_pipelined(hin, hout, ch, 16, True))
    print(f"chunks={ch}: {t(g.replay):.3f} ms", flush=True)
import numpy as np  # noqa
from oracle import hydro_oracle as HO  # noqa
g.replay()
torch.cuda.synchronize()
print("bit-exact:", np.array_equal(hout.numpy(), HO.advect_once(hin.numpy())))

# timeline of one pipelined iteration (kineto/CUPTI activity records)
if len(sys.argv) > 1 and sys.argv[1] == "trace":
    import json
    from torch.profiler import ProfilerActivity, profile
    for ch in ("taper", [1, 2, 3, 4, 3, 2, 1]):
        p = HostPipeline(it, hin, hout, chunks=ch, down_ctas=16)
        for _ in range(3):
            p.run()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            p.run()
            torch.cuda.synchronize()
        path = f"gpurun_out/e2e_trace_{len(p.fi.P)}.json"
        prof.export_chrome_trace(path)
        ev = [e for e in json.load(open(path))["traceEvents"]
              if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")]
        t0 = min(e["ts"] for e in ev)
        print(f"--- chunks={ch}: {len(ev)} device activities")
        for e in sorted(ev, key=lambda e: e["ts"]):
            print(f"{e['ts'] - t0:8.1f} {e['dur']:7.1f} "
                  f"s{e['args'].get('stream')} {e['name'][:60]}")

if False:
    for ch in (4, 8, 16):
        print(f"run_host_pipelined (no graph) chunks={ch}: "
              f"{t(lambda: it.run_host_pipelined(hin, hout, ch)):.3f} ms",
              flush=True)
