"""Queue consumer grids back to back with every slice pre-published (no
host formation in the loop): the device-side throughput of the chained
consumer (programmatic dependent launches, early box loads) against the
one-launch kernel and the A=128 team plan on the same slices."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2210_06438_b200 import _lib  # noqa: E402

lib = _lib.load(build_if_missing=False)
wl = bench.Workload()
S = wl.S
st = torch.cuda.current_stream()
slots = []
for _ in range(2):
    slots.append({
        "ctl_h": torch.tensor([S, S, 0, 0, 0], dtype=torch.int64).pin_memory(),
        "ring_d": torch.zeros(S + 2, dtype=torch.int64, device="cuda"),
        "qdev": torch.zeros(64, dtype=torch.int64, device="cuda"),
        "epoch": 0, "done": 0})


rings = {}
ORDER = torch.arange(S, dtype=torch.int64)


def ring(epoch):
    """The host ring as published for `epoch` (read-only for the GPU, so
    runs of both slots with the same epoch share it)."""
    key = (epoch, id(ORDER))
    if key not in rings:
        rings[key] = (ORDER | (epoch << 32)).pin_memory()
    return rings[key]


def run(k, flags):
    s = slots[k % 2]
    s["epoch"] += 1
    rc = lib.tf_queue_consumer_launch(
        wl.pools[k % 2].data_ptr(), S, 8, ring(s["epoch"]).data_ptr(),
        s["ctl_h"].data_ptr(), s["ring_d"].data_ptr(), S,
        s["qdev"].data_ptr(), s["done"], s["epoch"], 1.0, 1.0, 1.0,
        wl.um.data_ptr(), wl.up.data_ptr(), wl.F.data_ptr(),
        wl.amax.data_ptr(), 0, 2_000_000_000, flags, st.cuda_stream)
    assert rc == 0, rc
    s["done"] += S


def timeit(fn, K=40):
    for k in range(10):
        fn(k)
    torch.cuda.synchronize()
    ts = []
    for rep in range(5):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for k in range(K):
            fn(k)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / K * 1e3)
    return min(ts), sorted(ts)[2]


for name, flags in (("chained+early", 3), ("chained", 2), ("plain", 0)):
    mn, med = timeit(lambda k: run(k, flags))
    print(f"consumer {name:14s}: min {mn:.1f} us  median {med:.1f} us "
          f"per {S} slices", flush=True)
# the order the formation core publishes at A = 128 (strided teams: parent
# = arrival % 32, so a team's members are 32 sub-grids apart)
from paper_2210_06438_b200.strategy3 import form_teams  # noqa: E402
ORDER = torch.tensor([g for t in form_teams(range(S), 128, 1)
                      for g in t.ids], dtype=torch.int64)
mn, med = timeit(lambda k: run(k, 3))
print(f"consumer chained+early, A=128 team order: min {mn:.1f} us  "
      f"median {med:.1f} us", flush=True)
single = bench.single_runner(wl)
mn, med = timeit(single)
print(f"one launch           : min {mn:.1f} us  median {med:.1f} us")
step, nk, hist, plans = bench.plan_runner(wl, 128, 2, overlap=True,
                                          team_buffers=False)
mn, med = timeit(step)
print(f"plan A=128 2 exec    : min {mn:.1f} us  median {med:.1f} us")
