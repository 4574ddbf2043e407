"""Host->device upload of config 2's field (16.8 MB pinned) split over 1, 2,
4 streams (copy engines): does more than one engine raise the rate?"""
import torch
N = 128 ** 3
src = torch.randn(N, dtype=torch.float64).pin_memory()
dst = torch.empty(N, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
for k in (1, 2, 4, 8):
    ts = []
    for rep in range(30):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        step = N // k
        for i in range(k):
            s = streams[i]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step],
                                                   non_blocking=True)
        for i in range(k):
            torch.cuda.current_stream().wait_stream(streams[i])
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{k} streams: median {ts[15]*1e3:.1f} us  ({N*8/ts[15]/1e6:.1f} GB/s)"
          f"  min {ts[0]*1e3:.1f} us", flush=True)
