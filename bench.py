#!/usr/bin/env python
"""Benchmark: strategy-3 aggregated FP64 hydro reconstruct+flux on B200.

Metric (BASELINE.json): sub-grid cell-updates/s of the hydro
reconstruct+flux hot path vs aggregation level, and % of HBM peak.

N = 1 (BASELINE.json configs[1]): Sod shock tube, 4096 8^3 sub-grids
(grid 128^3), velocity (1,1,1).  One STEP = one iteration of the aggregated
reconstruct+flux region over all sub-grids: the 4096 task arrivals are
formed into teams by the strategy-3 formation core (max_team = 128 by
default, parents = S/max_team as HydroSim does, step.py:61), each team is one
launch of the batched TMA kernel, and the iteration's team launches replay as
one CUDA graph over the executor streams.  Inputs are device-resident; two
input pools alternate between steps (per-step working set 385 MB, 3x L2).
The timed outputs are checked against digests of the oracle's result
(tests/golden/bench_cfg2.json) before the line is printed.

N > 1 (BASELINE.json configs[4]): config 5, 262 144 8^3 sub-grids (grid
512^3, blast field) slab-partitioned over the N GPUs (strong scaling); one
STEP = one full iteration per rank with the ghost-layer exchange inside it
(the step kernel stores its boundary layers into the ring neighbours' fields
over peer memory; NCCL ring variant timed beside it).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

`--gpus N` with N > 1 outside torchrun re-launches itself under
torch.distributed.run with N ranks (one process per GPU).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("sub-grid cell-updates/sec (hydro reconstruct+flux) vs "
          "aggregation; % HBM peak")
UNIT = "cell-updates/s"
GRID, N_SUB, FIELD = 128, 8, "sod"
VELOCITY = (1.0, 1.0, 1.0)


def b_alg(n: int) -> int:
    """Algorithmic bytes per sub-grid-iteration (SURVEY §8 d): the distinct
    stencil cells read ((n+2)^3 + 6(n+2)^2) plus um, up, F written
    (9 (n+2)^3), FP64."""
    c = n + 2
    return 8 * (c ** 3 + 6 * c ** 2 + 9 * c ** 3)


def b_step(n: int) -> int:
    """Algorithmic bytes of the fused full step per sub-grid (SURVEY §8 d
    secondary metric): distinct stencil cells read + n^3 written."""
    c = n + 2
    return 8 * (c ** 3 + 6 * c ** 2 + n ** 3)


def ncu_traffic_per_launch(team: int,
                           capture: str = "r01_ncu_recon_flux_single.txt"):
    """DRAM bytes (read + write) per launch of `team` slices / sub-grids,
    scaled from a committed ncu --set full capture (the recon+flux kernel
    over 4096 slices by default; writes still resident in L2 at kernel end
    are not counted)."""
    path = os.path.join(ROOT, "profiles", capture)
    try:
        vals = {}
        with open(path) as fh:
            for line in fh:
                parts = line.split()
                if len(parts) >= 2 and parts[0] in (
                        "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "launch__grid_size"):
                    scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3,
                             "byte": 1.0}.get(parts[2] if len(parts) > 2
                                              else "", 1.0)
                    vals[parts[0]] = float(parts[1]) * scale
        per_slice = (vals["dram__bytes_read.sum"]
                     + vals["dram__bytes_write.sum"]) / vals["launch__grid_size"]
        return per_slice * team
    except (OSError, KeyError, ValueError):
        return None


def ncu_kernel_traffic(capture: str):
    """DRAM bytes (read + write) of one whole launch from a committed
    scripts/ncu_stalls.py text capture (None if missing)."""
    path = os.path.join(ROOT, "profiles", capture)
    try:
        vals = {}
        with open(path) as fh:
            for line in fh:
                parts = line.split()
                if len(parts) >= 2 and parts[0] in ("dram__bytes_read.sum",
                                                    "dram__bytes_write.sum"):
                    vals[parts[0]] = float(parts[1])
        return vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    except (OSError, KeyError, ValueError):
        return None


def ncu_graph_traffic(capture: str = "r02_ncu_plan_graph_A128.csv"):
    """DRAM bytes (read + write) of ONE timed step: the committed ncu
    capture of the bench's own A = 128 plan graph replays
    (--graph-profiling graph --cache-control none: the whole step as one
    workload, L2 state as the timed loop leaves it), mean over the captured
    replays.  None if the capture is missing."""
    import csv
    path = os.path.join(ROOT, "profiles", capture)
    try:
        with open(path) as fh:
            txt = fh.read()
        rows = list(csv.reader(txt[txt.index('"ID"'):].splitlines()))
        hdr = rows[0]
        idi, mi, vi = (hdr.index("ID"), hdr.index("Metric Name"),
                       hdr.index("Metric Value"))
        per = {}
        for r in rows[1:]:
            if r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                per[r[idi]] = per.get(r[idi], 0.0) + float(r[vi])
        return sum(per.values()) / len(per) if per else None
    except (OSError, ValueError, IndexError):
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# --------------------------------------------------------------- clocks
class ClockSampler:
    """NVML SM clock + throttle reasons while the GPU is under load."""

    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown",
            0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks",
            0x1: "gpu_idle"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(
                self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(
                    self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.BITS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.nv is not None:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------- dist plumbing
def self_launch(args) -> int:
    """`--gpus N` (N > 1) outside torchrun: run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1
    rendezvous) and return its exit code.  rank 0 prints the line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(gpus: int, init: bool = True):
    """RANK / LOCAL_RANK / WORLD_SIZE from the torchrun environment; the
    world must be exactly --gpus (a silent 1-rank run of an N-GPU request
    would report the wrong n_gpus)."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}; "
                         "launch with torchrun --nproc-per-node {gpus} (or "
                         "without torchrun, which self-launches)")
    if world > 1 and init:
        import torch.distributed as dist
        # one process per GPU; the modulo only matters when a test squeezes
        # several ranks onto fewer GPUs (TASKFUSE_DIST_BACKEND=gloo)
        if torch.cuda.is_available():
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
        backend = os.environ.get("TASKFUSE_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # the communicator init (ranks, transports) goes to stderr so
            # the rank count is checkable; stdout carries only the line
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group(
                "nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    return world, rank, local


def all_true(world, ok: bool) -> bool:
    """Logical AND over ranks."""
    if world == 1:
        return bool(ok)
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, x: float) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed(fn, steps, warmup, world, stream, settle_s: float = 0.02):
    """W untimed steps (and at least `settle_s` of untimed work, so a short
    measurement after host-side setup does not start on idle-lowered
    clocks), then EXACTLY `steps` steps between barrier+sync on both sides,
    CUDA events on the launching stream; ms/step (max over ranks)."""
    import torch
    # ranks must run the same number of steps (every step may hold a
    # collective or a peer barrier), so the wall-clock settle applies to
    # one rank only
    t_end = time.time() + (settle_s if world == 1 else 0.0)
    k = 0
    while k < warmup or time.time() < t_end:
        fn(k)
        k += 1
        if k % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(steps):
        fn(k)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(world, t0.elapsed_time(t1) / steps)


# ------------------------------------------------------------- workload
class Workload:
    def __init__(self, n=N_SUB, grid=GRID, field=FIELD, pools=2):
        import torch
        from paper_2210_06438_b200 import ops
        from paper_2210_06438_b200.hydro import (initial_field,
                                                 pool_from_field, sod_field)
        self.n, self.grid = n, grid
        self.m = grid // n
        self.S = self.m ** 3
        f = (sod_field if field == "sod" else initial_field)(grid, "cuda")
        self.pools = []
        for _ in range(pools):
            p = pool_from_field(f, n)
            ops.ghost_fill(p, n, self.m)
            self.pools.append(p)
        c = n + 2
        shape = (self.S, 3, c, c, c)
        self.um = torch.empty(shape, dtype=torch.float64, device="cuda")
        self.up = torch.empty_like(self.um)
        self.F = torch.empty_like(self.um)
        self.amax = torch.empty(self.S, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()


def plan_runner(wl, max_team, executors, parents=None, overlap=True,
                team_buffers=False, geometry="tma"):
    from paper_2210_06438_b200.strategy3 import TeamPlan, form_teams
    teams = form_teams(range(wl.S), max_team, executors, parents)
    plans = [TeamPlan(teams, p, wl.n, VELOCITY, wl.um, wl.up, wl.F,
                      executors, amax=wl.amax, overlap=overlap,
                      team_buffers=team_buffers, geometry=geometry)
             for p in wl.pools]
    hist = {}
    for t in teams:
        hist[len(t.ids)] = hist.get(len(t.ids), 0) + 1

    def step(k):
        plans[k % len(plans)].launch()
    return step, len(teams), hist, plans


def realtime_runner(wl, max_team, executors, parents=None, overlap=False):
    from paper_2210_06438_b200.strategy3 import (RealtimeExecutor,
                                                 default_parents)
    parents = parents or default_parents(wl.S, max_team)
    ex = RealtimeExecutor("reconstruct", max_team, executors, parents,
                          overlap=overlap)
    # an int32 array, so the per-step C call does not convert a list
    arrivals = np.arange(wl.S, dtype=np.int32)
    launches = []

    def step(k):
        launches.append(ex.run(wl.pools[k % len(wl.pools)], wl.n, VELOCITY,
                               arrivals, wl.um, wl.up, wl.F, amax=wl.amax))
    return step, launches, ex


def queue_runner(wl, max_team, parents=None):
    """Strategy 3 formed ON THE FLY inside every step: the arrivals go
    through the C++ formation core (cap / solo fast path / drain on 'every
    published slice completed'), each closed team is published to the
    device queue, one consumer grid per step (a CTA per published slice,
    a programmatic dependent of the previous step's grid)."""
    from paper_2210_06438_b200.strategy3 import (QueueExecutor,
                                                 default_parents)
    parents = parents or default_parents(wl.S, max_team)
    # the pools are produced once, before any step: the first boxes of step
    # k+1 may load during step k's tail (TF_LAUNCH_OVERLAP_PREV); the device
    # works through each mirrored batch in sub-grid id order
    # (TF_QUEUE_SORTED: the formed teams' members are strided)
    q = QueueExecutor("reconstruct", max_team, parents, wl.n,
                      early_loads=True, sorted_dispatch=True)
    arrivals = np.arange(wl.S, dtype=np.int32)
    # one bound call per input pool (arguments checked once; the formation
    # and the publishing still run inside every step)
    calls = [q.bind(p, VELOCITY, arrivals, wl.um, wl.up, wl.F, amax=wl.amax)
             for p in wl.pools]

    def step(k):
        calls[k % len(calls)]()
    return step, q


def single_runner(wl, reconstruction="minmod", flux_form=0):
    from paper_2210_06438_b200 import ops

    def step(k):
        ops.recon_flux(wl.pools[k % len(wl.pools)], wl.n, VELOCITY, wl.um,
                       wl.up, wl.F, out_mode=1, amax=wl.amax,
                       flux_form=flux_form, reconstruction=reconstruction)
    return step


def scheme_legs(wl, steps, warmup, world, stream, peak):
    """north_star's named kernels on config 2, one launch of all slices:
    Kurganov-Tadmor flux form (1e-12 of the reference's upwind flux) and
    PPM reconstruction (parity unpinned).  PPM's stencil
    reaches the ghost depth 3, so its algorithmic read is the whole 14^3
    box: 8 [E^3 + 9 (n+2)^3] B per sub-grid."""
    n = wl.n
    c, e = n + 2, n + 6
    out = {}
    for name, rec, ff, per in (
            ("minmod_upwind", "minmod", 0, b_alg(n)),
            ("minmod_kt", "minmod", 1, b_alg(n)),
            ("ppm_upwind", "ppm", 0, 8 * (e ** 3 + 9 * c ** 3)),
            ("ppm_kt", "ppm", 1, 8 * (e ** 3 + 9 * c ** 3))):
        ms = timed(single_runner(wl, rec, ff), steps, warmup, world, stream)
        out[name] = {"cell_updates_per_s": rate(wl.S, n, ms),
                     "ms_per_iter": ms, "alg_bytes_per_subgrid": per,
                     "hbm_frac": wl.S * per / (ms * 1e-3) / 1e9 / peak}
    return out


def rate(S, n, ms):
    return S * n ** 3 / (ms * 1e-3)


def run_sweep(wl, args, world, stream, peak):
    """Aggregation sweep 1..128 (plan-graph and real-time executor),
    strategy 2 (A=1 over many streams), strategy 1 (16^3, A=1)."""
    out = {"aggregation": {}, "aggregation_1_executor": {},
           "aggregation_4_executors": {}, "realtime": {},
           "strategy2": {}, "strategy1": {}}
    ks, kw = max(5, args.steps // 2), 3
    for A in (1, 4, 16, 64, 128):
        for key, E in (("aggregation", args.executors),
                       ("aggregation_1_executor", 1),
                       ("aggregation_4_executors", 4)):
            step, nk, hist, _ = plan_runner(
                wl, A, E, team_buffers=args.outputs == "team")
            ms = timed(step, ks, kw, world, stream)
            out[key][A] = {
                "cell_updates_per_s": rate(wl.S, wl.n, ms), "ms_per_iter": ms,
                "launches": nk, "executors": E,
                "hbm_frac": wl.S * b_alg(wl.n) / (ms * 1e-3) / (peak * 1e9)}
        # the real-time launch-per-team executor on ONE stream (the paper's
        # strategy-3 configuration; with more streams the starvation rule
        # fires on every idle stream and most teams close solo)
        rstep, launches, ex = realtime_runner(wl, A, 1)
        ms = timed(rstep, ks, kw, world, stream)
        st = ex.stats()
        out["realtime"][A] = {
            "cell_updates_per_s": rate(wl.S, wl.n, ms), "ms_per_iter": ms,
            "launches_per_iter": launches[-1],
            "mean_team": wl.S * len(launches) / max(1, st["teams_formed"]),
            "solo_fast_path": st["solo_fast_path"]}
    # the headline executor over A: formation inside the timed step, each
    # closed team published to the device queue.  The device no longer pays
    # per team (one consumer grid per step, a CTA per slice); the HOST does
    # — one release store per team, which the fetcher CTA polls over PCIe —
    # so at small A the formation loop, not the GPU, sets the step time
    # (host_us: the C++ loop's own clock per step)
    out["realtime_queue"] = {}
    for A in (1, 4, 16, 64, 128):
        step, q = queue_runner(wl, A)
        ms = timed(step, ks, kw, world, stream)
        q.wait()
        st = q.stats()
        out["realtime_queue"][A] = {
            "cell_updates_per_s": rate(wl.S, wl.n, ms), "ms_per_iter": ms,
            "mean_team": st["teams_formed"] and
            sum(k * v for k, v in st["size_histogram"].items())
            / st["teams_formed"],
            "solo_fast_path": st["solo_fast_path"],
            "host_us": q.host_times()}
        del q, step
    for E in (1, 8, 32, 128):
        # strategy 2: per-task launches (A = 1) spread over E streams
        step, nk, _, _ = plan_runner(wl, 1, E, parents=E)
        ms = timed(step, ks, kw, world, stream)
        out["strategy2"][E] = {"cell_updates_per_s": rate(wl.S, wl.n, ms),
                               "ms_per_iter": ms, "launches": nk}
    # strategy 1: 512 sub-grids of 16^3 (same cells), one launch per
    # sub-grid.  "refgeo": the reference's launch geometry, 46 CTAs x 128
    # threads per 16^3 sub-grid (blocks_for, kernels.py:51-55) — the fair
    # baseline; "tma1": our one-CTA-per-slice TMA kernel at 16^3
    wl16 = Workload(n=16, grid=wl.grid, field=FIELD)
    for geo, tag in (("reference", "refgeo"), ("tma", "tma1")):
        for E in sorted({args.executors, 4}):
            step, nk, _, _ = plan_runner(wl16, 1, E, geometry=geo)
            ms = timed(step, ks, kw, world, stream)
            out["strategy1"][f"16^3_A1_E{E}_{tag}"] = {
                "cell_updates_per_s": rate(wl16.S, 16, ms),
                "ms_per_iter": ms, "launches": nk,
                "ctas_per_launch": 46 if geo == "reference" else 1,
                "hbm_frac": wl16.S * b_alg(16) / (ms * 1e-3)
                / (peak * 1e9)}
    # the same kernels with all 512 sub-grids in one launch (the limit)
    for geo, tag in (("reference", "refgeo"), ("tma", "tma1")):
        step, nk, _, _ = plan_runner(wl16, 128, 1, parents=1, geometry=geo)
        ms = timed(step, ks, kw, world, stream)
        out["strategy1"][f"16^3_A128_{tag}"] = {
            "cell_updates_per_s": rate(wl16.S, 16, ms), "ms_per_iter": ms,
            "launches": nk, "hbm_frac": wl16.S * b_alg(16) / (ms * 1e-3)
            / (peak * 1e9)}
    del wl16
    # the 8^3 aggregated path with the reference geometry (A = 128)
    step, nk, _, _ = plan_runner(wl, 128, args.executors,
                                 geometry="reference")
    ms = timed(step, ks, kw, world, stream)
    out["refgeo_8^3_A128"] = {
        "cell_updates_per_s": rate(wl.S, wl.n, ms), "ms_per_iter": ms,
        "launches": nk, "hbm_frac": wl.S * b_alg(wl.n) / (ms * 1e-3)
        / (peak * 1e9)}
    out["config3"] = config3_sweep(args, world, stream, peak, ks, kw)
    return out


def config3_sweep(args, world, stream, peak, ks, kw):
    """BASELINE config 3: 32 768 8^3 sub-grids (grid 256, the reference's
    Gaussian blast field), maximum aggregation (A = 128) vs strategy 2
    (A = 1 over 8 / 32 / 128 streams)."""
    wl3 = Workload(n=N_SUB, grid=256, field="blast")
    res = {"workload": "config 3: grid 256, 32768 8^3 sub-grids, blast",
           "aggregation_A128": {}, "strategy2": {}}
    for E in sorted({args.executors, 4}):
        step, nk, _, _ = plan_runner(wl3, 128, E, team_buffers=True)
        ms = timed(step, ks, kw, world, stream)
        res["aggregation_A128"][f"E{E}"] = {
            "cell_updates_per_s": rate(wl3.S, wl3.n, ms), "ms_per_iter": ms,
            "launches": nk,
            "hbm_frac": wl3.S * b_alg(wl3.n) / (ms * 1e-3) / (peak * 1e9)}
    # the headline's method: teams formed on the fly, the device queue
    step, q = queue_runner(wl3, 128)
    ms = timed(step, ks, kw, world, stream)
    q.wait()
    st = q.stats()
    res["on_the_fly_A128"] = {
        "cell_updates_per_s": rate(wl3.S, wl3.n, ms), "ms_per_iter": ms,
        "mean_team": sum(k * v for k, v in st["size_histogram"].items())
        / max(1, st["teams_formed"]),
        "hbm_frac": wl3.S * b_alg(wl3.n) / (ms * 1e-3) / (peak * 1e9)}
    del q, step
    for E in (8, 32, 128):
        step, nk, _, _ = plan_runner(wl3, 1, E, parents=E)
        ms = timed(step, max(3, ks // 4), kw, world, stream)
        res["strategy2"][E] = {"cell_updates_per_s": rate(wl3.S, wl3.n, ms),
                               "ms_per_iter": ms, "launches": nk}
    del wl3
    return res


# ------------------------------------------------------- workload configs
# One dict per workload, printed verbatim by BOTH arms (ours and
# --impl reference), so the driver sees the same config on each line.
def cfg2_config():
    S = (GRID // N_SUB) ** 3
    return {
        "workload": "config 2: Sod shock tube, 4096 8^3 FP64 sub-grids, one "
                    "aggregated reconstruct+flux iteration per step (um, up, "
                    "F and the per-sub-grid max signal speed materialised)",
        "subgrids": S, "subgrid_n": N_SUB, "grid": GRID, "field": FIELD,
        "velocity": list(VELOCITY),
        "l2": "inputs larger than L2: two ghost-filled input pools "
              "alternate between steps; per-step working set 385 MB vs "
              "126 MB L2"}


CFG5_FIELD = "blast"


def cfg5_config(world, grid):
    S = (grid // N_SUB) ** 3
    return {
        "workload": f"config 5: blast wave, {S} 8^3 FP64 sub-grids (grid "
                    f"{grid}^3) slab-partitioned over the GPUs; one full "
                    "iteration per step (ghost-layer exchange, reconstruct, "
                    "flux, update)",
        "subgrids": S, "subgrid_n": N_SUB, "grid": grid, "field": CFG5_FIELD,
        "velocity": list(VELOCITY),
        "parallelism": f"x-slab partition over {world} GPU(s)",
        "l2": f"inputs larger than L2: the field is {grid ** 3 * 8 / 1e9:.2f}"
              " GB per copy vs 126 MB L2"}


def workload_of(args, world):
    if args.workload != "auto":
        return args.workload
    return "cfg2" if world == 1 else "cfg5"


# --------------------------------------------------------- CPU baselines
def cpu_baseline_leg(S, n, grid, steps=2, min_seconds=10.0):
    from oracle.cpu_baseline import CpuBaseline, cpu_model
    cb = CpuBaseline(FIELD, grid, n, VELOCITY, range(S))
    try:
        times = []
        t_start = time.perf_counter()
        while len(times) < steps or (time.perf_counter() - t_start
                                     < min_seconds / cb.workers
                                     and len(times) < 20):
            times.append(cb.step())
        best = min(times)
    finally:
        cb.close()
    return {"value": rate(S, n, best * 1e3), "unit": UNIT,
            "cores": cb.workers, "kind": "port",
            "sample": (f"all {S} 8^3 sub-grids of config 2 per pass "
                       f"(prep+reconstruct+flux+reduce bodies, oracle port "
                       f"of hydro/kernels.py), spawn pool of {cb.workers} "
                       f"workers, slowest worker, best of {len(times)} "
                       f"passes; CPU {cpu_model()}")}


CFG5_SAMPLE_GRID = 128


def reference_arm(args, world, rank, workload):
    """--impl reference: the reference's CPU path (oracle port of its task
    bodies; the reference is pure Python and is not present on GPU boxes)
    on all host cores, same metric / unit / config as our arm.  Under
    torchrun only rank 0 works and prints."""
    if rank != 0:
        return
    from oracle.cpu_baseline import CpuBaseline, cpu_model
    if workload == "cfg2":
        S_run, grid_run, field, bodies = (GRID // N_SUB) ** 3, GRID, FIELD, \
            "recon_flux"
        config = cfg2_config()
        S_metric = S_run
        sample = (f"all {S_run} sub-grids per step (prep+reconstruct+flux+"
                  "reduce bodies)")
    else:
        # the per-sub-grid CPU cost does not depend on the lattice size, so
        # the config-5 rate is measured on a 16^3-sub-grid lattice of the
        # same blast field and bodies (the full 262 144-sub-grid pool would
        # need 5.8 GB per worker); cell-updates/s carries over linearly
        S_run, grid_run, field, bodies = (CFG5_SAMPLE_GRID // N_SUB) ** 3, \
            CFG5_SAMPLE_GRID, CFG5_FIELD, "iteration"
        config = cfg5_config(world, args.cfg5_grid)
        S_metric = (args.cfg5_grid // N_SUB) ** 3
        sample = (f"{S_run} sub-grids per step (a {CFG5_SAMPLE_GRID}^3 "
                  "blast lattice; exchange_ghosts + prep + reconstruct + "
                  "flux + reduce + update per sub-grid, the CPU task "
                  "iteration of step.py:93-97), rate extrapolated linearly "
                  f"to {S_metric} sub-grids")
    cb = CpuBaseline(field, grid_run, N_SUB, VELOCITY, range(S_run),
                     bodies=bodies)
    try:
        for _ in range(args.warmup):
            cb.step()
        times = [cb.step() for _ in range(args.steps)]
    finally:
        cb.close()
    ms_run = 1e3 * sum(times) / len(times)
    value = rate(S_run, N_SUB, ms_run)
    ms = ms_run * S_metric / S_run
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if workload == "cfg2" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb.workers,
                         "kind": "port",
                         "sample": f"{sample}; spawn pool of {cb.workers} "
                                   f"workers, CPU {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- e2e legs
def e2e_leg(args, steps, warmup, world, stream):
    """The headline e2e: the same aggregated reconstruct+flux iteration as
    `value`, through the public API with HOST buffers
    (strategy3.AggregatedIteration.recon_flux_host): every step copies the
    pinned host field host->device, scatters it into the sub-grid pool and
    fills the ghosts (make_state + exchange_ghosts, which `value` and the
    CPU arm get for free), runs the captured A-team plan (um / up / F to
    HBM) and reads the step's result — the per-sub-grid max signal speed,
    the reduce stage's output — back device->host."""
    import torch
    from paper_2210_06438_b200.hydro import sod_field
    from paper_2210_06438_b200.strategy3 import AggregatedIteration
    it = AggregatedIteration(GRID, N_SUB, VELOCITY, max_team=args.max_team,
                             executors=args.executors)
    host_in = sod_field(GRID, "cpu").pin_memory()
    amax = torch.empty(it.S, dtype=torch.float64).pin_memory()

    from paper_2210_06438_b200.strategy3 import ReconFluxHostPipeline
    # the chunked upload on one copy stream, or each chunk split over two
    # (copy engines differ from box to box): the faster is the call timed
    pipes = {cs: ReconFluxHostPipeline(it, host_in, amax, copy_streams=cs)
             for cs in (1, 2)}
    # host-link transfers settle slower than kernels: 0.3 s of untimed
    # calls first (a short warm-up measured the same call 10-15% slower)
    pipe_ms = {cs: timed(lambda k, p=p: p.run(), steps, max(5, warmup),
                         world, stream, settle_s=0.3)
               for cs, p in pipes.items()}
    cs_best = min(pipe_ms, key=pipe_ms.get)
    pipe, ms_pipe = pipes[cs_best], pipe_ms[cs_best]
    torch.cuda.synchronize()
    ok = bool((amax == max(abs(v) for v in VELOCITY)).all())
    ms_plain = timed(lambda k: it.recon_flux_host(host_in, amax), steps,
                     max(5, warmup), world, stream, settle_s=0.3)
    torch.cuda.synchronize()
    ok = ok and bool((amax == max(abs(v) for v in VELOCITY)).all())
    # the same call with the teams formed on the fly (the headline's path):
    # the formation core publishes to the device queue after the ghost fill
    itq = AggregatedIteration(GRID, N_SUB, VELOCITY, max_team=args.max_team,
                              executors=1, formation="queue")
    ms_queue = timed(lambda k: itq.recon_flux_host(host_in, amax), steps,
                     max(5, warmup), world, stream, settle_s=0.3)
    itq.queue.wait()
    torch.cuda.synchronize()
    ok = ok and bool((amax == max(abs(v) for v in VELOCITY)).all())
    # all three are the public host->host call for the same computation;
    # the overlapped one wins on a healthy host link, a plain one when the
    # copy engine is slow to start chunked transfers (seen on some boxes)
    pipelined = ms_pipe <= min(ms_plain, ms_queue)
    on_the_fly = not pipelined and ms_queue <= ms_plain
    ms = min(ms_pipe, ms_plain, ms_queue)
    res = {"value": rate(it.S * world, N_SUB, ms), "unit": UNIT,
           "ms_per_step": ms, "h2d_bytes_per_step": host_in.numel() * 8,
           "d2h_bytes_per_step": amax.numel() * 8,
           "gpu_launches_per_step": (
               pipe.launches if pipelined else
               itq.recon_flux_launches if on_the_fly
               else it.recon_flux_launches),
           "result_check": ok,
           "call": ("strategy3.ReconFluxHostPipeline.run" if pipelined
                    else "AggregatedIteration(formation='queue')."
                         "recon_flux_host" if on_the_fly
                    else "AggregatedIteration.recon_flux_host"),
           "step": "pinned host field -> device, scattered into the sub-grid "
                   "pool, ghost fill, aggregated reconstruct+flux teams "
                   "(um/up/F to HBM), per-sub-grid max signal speed -> "
                   "pinned host; pipelined: x-chunked upload on the copy "
                   "engine (the last layer first), each layer launched "
                   "once it and its two neighbours landed, max speeds "
                   "home per group, one CUDA graph",
           "pipelined": {"ms_per_step": ms_pipe,
                         "value": rate(it.S * world, N_SUB, ms_pipe),
                         "copy_streams": cs_best,
                         "ms_by_copy_streams": pipe_ms},
           "unpipelined": {"ms_per_step": ms_plain,
                           "value": rate(it.S * world, N_SUB, ms_plain)},
           "on_the_fly": {"ms_per_step": ms_queue,
                          "value": rate(it.S * world, N_SUB, ms_queue),
                          "step": "unpipelined, teams formed on the fly "
                                  "and published to the device queue"}}
    # the same iteration with the update and the whole field back
    host_out = torch.empty_like(host_in).pin_memory()
    ms_it = timed(lambda k: it.run_host(host_in, host_out), steps, warmup,
                  world, stream)
    res["full_iteration_host_roundtrip"] = {
        "value": rate(it.S * world, N_SUB, ms_it), "unit": UNIT,
        "ms_per_step": ms_it, "h2d_bytes_per_step": host_in.numel() * 8,
        "d2h_bytes_per_step": host_out.numel() * 8,
        "step": "host field in -> scatter, ghost fill, aggregated "
                "recon+flux teams (um/up/F to HBM), update -> host field out "
                "(AggregatedIteration.run_host)"}
    return res


def fused_legs(args, steps, warmup, world, stream, peak):
    """The fused full iteration (field.FieldIteration, SURVEY §8 f #2) on
    config 2: device-resident step and the host round trip (a different
    computation from the headline: reconstruct+flux+update without
    materialising the faces)."""
    import torch
    from paper_2210_06438_b200.hydro import sod_field
    from paper_2210_06438_b200.field import FieldIteration, HostPipeline
    it = FieldIteration(GRID, N_SUB, VELOCITY, max_team=args.max_team,
                        executors=args.executors)
    it.load(sod_field(GRID, "cuda"))
    ms_dev = timed(lambda k: it.step(), steps, warmup, world, stream)
    host_in = sod_field(GRID, "cpu").pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    pipe = HostPipeline(it, host_in, host_out)
    ms_pipe = timed(lambda k: pipe.run(), steps, warmup, world, stream)
    S = (GRID // N_SUB) ** 3
    n = N_SUB
    fused_bytes = S * b_step(n)
    return {
        "device": {"value": rate(S * world, n, ms_dev), "unit": UNIT,
                   "ms_per_step": ms_dev,
                   "b_step_frac": fused_bytes / (ms_dev * 1e-3) / 1e9 / peak,
                   "launches_per_step": it.launches_per_step,
                   "step": "one fused recon+flux+update kernel per team, "
                           "each also writing its sub-grids' share of the "
                           "next field's periodic halos (CUDA graph)"},
        "host_pipelined": {
            "value": rate(S * world, n, ms_pipe), "unit": UNIT,
            "ms_per_step": ms_pipe,
            "h2d_bytes_per_step": host_in.numel() * 8,
            "d2h_bytes_per_step": host_out.numel() * 8,
            "gpu_launches_per_step": pipe.launches,
            "step": "field.HostPipeline: tapered x-chunks, copy-engine "
                    "upload / pad+halo kernel / fused step / zero-copy "
                    "download kernel, overlapped, one CUDA graph"},
    }


def e2e_faces_leg(wl, step_fn, steps, warmup, world, stream):
    """Variant: ghosted pool in, ALL recon+flux outputs (um, up, F) out —
    PCIe-bound by 385 MB per step."""
    import torch
    host_in = wl.pools[0].cpu().pin_memory()
    outs = [torch.empty_like(t, device="cpu").pin_memory()
            for t in (wl.um, wl.up, wl.F)]
    dev_in = wl.pools[0]

    def step(k):
        dev_in.copy_(host_in, non_blocking=True)
        step_fn(0)
        for h, d in zip(outs, (wl.um, wl.up, wl.F)):
            h.copy_(d, non_blocking=True)
    ms = timed(step, steps, warmup, world, stream)
    torch.cuda.synchronize()
    return ms, host_in.numel() * 8, sum(o.numel() * 8 for o in outs)


# ------------------------------------------------- real-time aggregation
def plan_leg(wl, args, world, stream, peak):
    """The same A-teams pre-formed once (form_teams with a saturated device:
    every busy query answers busy, cap closure) and replayed as ONE CUDA
    graph per step — one kernel node per team on 2 executor branches,
    programmatic dependent launches inside a branch; outputs into the packed
    team leases (the reference's slice_alloc layout).  The steady state of
    an iterative solver whose teams repeat; checked against the oracle
    digests like the headline."""
    step, nk, hist, plans = plan_runner(wl, args.max_team, args.executors,
                                        overlap=not args.no_overlap,
                                        team_buffers=True)
    ms = timed(step, args.steps, args.warmup, world, stream)
    check = cfg2_output_check(wl, plans, True)
    if not check["bitexact_vs_oracle_digest"]:
        raise SystemExit(f"bench.py: plan outputs differ {check}")
    traffic = ncu_graph_traffic() if args.max_team == 128 else None
    achieved = wl.S * b_alg(wl.n) / (ms * 1e-3) / 1e9
    return {"value": rate(wl.S * world, wl.n, ms), "unit": UNIT,
            "ms_per_step": ms, "max_team": args.max_team,
            "executors": args.executors, "team_histogram": hist,
            "launches_per_step": nk, "self_check": check,
            "roofline": {"achieved": achieved, "peak": peak,
                         "frac": achieved / peak, "unit": "GB/s",
                         "traffic": traffic,
                         "traffic_frac": (traffic / (ms * 1e-3) / 1e9 / peak
                                          if traffic else None),
                         "traffic_source": "profiles/r02_ncu_plan_graph_"
                                           "A128.csv (--graph-profiling "
                                           "graph --cache-control none)"}}


def realtime_leg(wl, args, world, stream, peak, with_queue=True):
    """Strategy 3 formed ON THE FLY inside the timed region, other
    executors: (with_queue) the device queue (strategy3.QueueExecutor: each
    closed team published to a consumer grid), and each closed team
    launched as its own grid FROM THE DEVICE (strategy3.
    DeviceLaunchExecutor) over A = 1..128.  Same outputs as `value`
    (checked against the oracle digests), per-sub-grid slots."""
    arrivals = np.arange(wl.S, dtype=np.int32)
    A = args.max_team
    out = {}
    if with_queue:
        step, q = queue_runner(wl, A)
        with ClockSampler(0) as clk:
            ms = timed(step, args.steps, args.warmup, world, stream)
        q.wait()
        st = q.stats()
        check = cfg2_output_check(wl, rerun=lambda: (step(0), q.wait()))
        if not check["bitexact_vs_oracle_digest"]:
            raise SystemExit(f"bench.py: real-time queue outputs differ "
                             f"{check}")
        achieved = wl.S * b_alg(wl.n) / (ms * 1e-3) / 1e9
        out.update({
            "value": rate(wl.S * world, wl.n, ms), "unit": UNIT,
            "ms_per_step": ms, "max_team": A,
            "mean_team": sum(k * v for k, v in st["size_histogram"].items())
            / max(1, st["teams_formed"]),
            "teams_per_step": st["teams_formed"] / max(1, q.runs),
            "solo_fast_path": st["solo_fast_path"],
            "host_us_per_step": q.host_times(),
            "roofline": {"achieved": achieved, "peak": peak,
                         "frac": achieved / peak, "unit": "GB/s"},
            "gpu_launches_per_step": 1, "self_check": check,
            "clocks": clk.summary()})
    # the same real-time formation with each closed team launched as its
    # own grid from the device (strategy3.DeviceLaunchExecutor): A sweep
    from paper_2210_06438_b200.strategy3 import (DeviceLaunchExecutor,
                                                 default_parents)
    dl = {}
    for a in (1, 4, 16, 64, 128):
        ex = DeviceLaunchExecutor("reconstruct", a,
                                  default_parents(wl.S, a), wl.n)

        def dstep(k, ex=ex):
            ex.run(wl.pools[k % len(wl.pools)], VELOCITY, arrivals, wl.um,
                   wl.up, wl.F, amax=wl.amax)
        dms = timed(dstep, max(5, args.steps // 2), 3, world, stream)
        ex.wait()
        dst = ex.stats()
        dl[a] = {"value": rate(wl.S * world, wl.n, dms), "ms_per_step": dms,
                 "mean_team": sum(k * v for k, v in
                                  dst["size_histogram"].items())
                 / max(1, dst["teams_formed"]),
                 "hbm_frac": wl.S * b_alg(wl.n) / (dms * 1e-3) / 1e9 / peak}
        del ex
    ex = DeviceLaunchExecutor("reconstruct", A, default_parents(wl.S, A),
                              wl.n)
    dcheck = cfg2_output_check(
        wl, rerun=lambda: (ex.run(wl.pools[0], VELOCITY, arrivals, wl.um,
                                  wl.up, wl.F, amax=wl.amax), ex.wait()))
    del ex
    if not dcheck["bitexact_vs_oracle_digest"]:
        raise SystemExit(f"bench.py: device-launch outputs differ {dcheck}")
    out["device_launch_sweep"] = dl
    out["device_launch_self_check"] = dcheck["bitexact_vs_oracle_digest"]
    return out


# ------------------------------------------------ the reference API path
def reference_api_legs(args):
    """The reference's own entry points — HydroSim + driver (step.py:
    38-143) through the mirrored API, the native engine running the
    per-sub-grid tasks: five region visits each (alloc x4, h2d, one
    batched kernel per team, d2h, await, leave), real staging copies, teams
    formed in real time.  ms per reference step (3 iterations).

    config 1: 64 Sod sub-grids, executors 1, max_team 1 (the BASELINE
    config, "runs on the CPU reference as-is"), beside the reference's CPU
    task iteration (exchange_ghosts + the five bodies, step.py:93-97) for
    the same 64 sub-grids on ONE host core (the reference is a single
    Python process).  config 2: 4096 Sod sub-grids, aggregation sweep."""
    from paper_2210_06438_b200.bench_matrix import run_cell
    from paper_2210_06438_b200.hydro import sod_field
    out = {}
    row1, sim, _ = run_cell(8, 1, 1, steps=3, grid_n=32,
                            field=sod_field(32, "cuda"))
    row = row1
    out["config1"] = {"ms_per_step": row.ms_per_step,
                      "cell_updates_per_s": 64 * 512 * 3
                      / (row.ms_per_step * 1e-3),
                      "kernels_per_step": row.kernels,
                      "transfers_per_step": row.transfers,
                      "measured_raw_allocs": row.measured_raw_allocs,
                      "host_us_per_iteration": {
                          k: v / 12 / 1e3 for k, v in
                          sim.native.host_times().items()}}
    del sim
    # the same per-task path with two executor streams (strategy 2), and
    # with aggregation (A = 64: one team per region per iteration)
    for E, A in ((2, 1), (1, 64)):
        row, sim, _ = run_cell(8, E, A, steps=3, grid_n=32,
                               field=sod_field(32, "cuda"))
        out["config1"][f"E{E}_A{A}_ms_per_step"] = row.ms_per_step
        del sim
    if not args.no_cpu_baseline:
        from oracle.cpu_baseline import CpuBaseline, cpu_model
        cb = CpuBaseline("sod", 32, N_SUB, VELOCITY, range(64), workers=1,
                         bodies="iteration")
        try:
            best = min(cb.step() for _ in range(5))
        finally:
            cb.close()
        ms_cpu = 3 * best * 1e3
        out["config1"]["cpu_reference"] = {
            "ms_per_step": ms_cpu, "cores": 1, "kind": "port",
            "sample": "all 64 sub-grids x 3 iterations: exchange_ghosts + "
                      "prep/reconstruct/flux/reduce/update bodies (oracle "
                      f"port), best of 5; CPU {cpu_model()}"}
        out["config1"]["speedup_vs_cpu"] = ms_cpu / row1.ms_per_step
        out["config1"]["speedup_vs_cpu_E2"] = \
            ms_cpu / out["config1"]["E2_A1_ms_per_step"]
    sweep = {}
    for A in (1, 4, 16, 64, 128):
        row, sim, _ = run_cell(8, 1, A, steps=1, grid_n=GRID,
                               field=sod_field(GRID, "cuda"))
        members = sum(k * v for k, v in row.team_sizes.items())
        teams = sum(row.team_sizes.values())
        sweep[A] = {"ms_per_step": row.ms_per_step,
                    "cell_updates_per_s": 4096 * 512 * 3
                    / (row.ms_per_step * 1e-3),
                    "kernels_per_step": row.kernels,
                    "mean_team": members / teams,
                    "measured_raw_allocs": row.measured_raw_allocs}
        del sim
    out["config2_sweep"] = sweep
    out["config2_A64_vs_A1"] = sweep[1]["ms_per_step"] / \
        sweep[64]["ms_per_step"]
    out["note"] = ("HydroSim + driver through the mirrored reference API "
                   "(bench_matrix.run_cell, engine native); each step = 3 "
                   "iterations x S tasks x 5 region visits with real "
                   "staging copies (ext^3 up, n^3 down per slice)")
    return out


# -------------------------------------------------------------- self-checks
def cfg2_output_check(wl, plans=None, team_buffers=True, rerun=None):
    """The timed path's outputs against the oracle's digests for this exact
    workload (tests/golden/bench_cfg2.json; the Sod data are exactly
    representable, so the digests are machine-independent).  Packed team
    leases are put back in sub-grid order first.  `rerun()` (or the first
    plan) recomputes pool 0's outputs after a NaN fill."""
    import hashlib
    import torch
    path = os.path.join(ROOT, "tests", "golden", "bench_cfg2.json")
    with open(path) as fh:
        want = json.load(fh)
    torch.cuda.synchronize()
    for t in (wl.um, wl.up, wl.F, wl.amax):
        t.fill_(float("nan"))
    if rerun is not None:
        rerun()
    else:
        plans[0].launch()
    torch.cuda.synchronize()
    if plans is not None and team_buffers:
        inv = torch.empty(wl.S, dtype=torch.int64, device="cuda")
        order = torch.from_numpy(plans[0].order.astype(np.int64)).cuda()
        inv[order] = torch.arange(wl.S, device="cuda")
    else:
        inv = torch.arange(wl.S, device="cuda")
    got = {}
    for name, t in (("um", wl.um), ("up", wl.up), ("F", wl.F)):
        a = t[inv].cpu().numpy()
        got[name] = hashlib.sha256(
            np.ascontiguousarray(a, "<f8").tobytes()).hexdigest()
    amax_ok = bool((wl.amax == want["amax"]).all())
    ok = all(got[k] == want[k] for k in ("um", "up", "F")) and amax_ok
    return {"bitexact_vs_oracle_digest": ok,
            "digests": "tests/golden/bench_cfg2.json (um, up, F sha256)",
            "amax_ok": amax_ok}


# ------------------------------------------------------------ config 5
def cfg5_slab(part, grid):
    """The slab of initial_field (scenario.py:30-37) on this rank."""
    n = N_SUB
    a = part.x0 * n
    x = (np.arange(grid) + 0.5) / grid
    xs = x[a:a + part.mx * n]
    r2 = ((xs - 0.5) ** 2)[:, None, None] + ((x - 0.5) ** 2)[None, :, None] \
        + ((x - 0.5) ** 2)[None, None, :]
    return 1.0 + 1.0 * np.exp(-r2 / (2.0 * 0.1 ** 2))


def peer_access_ok(part, local) -> bool:
    """Can this rank's GPU store into both ring neighbours' memory?  One
    node, one process per GPU: rank r drives GPU r (mod the device count —
    ranks sharing a GPU map each other's memory on the same device)."""
    import torch
    if part.world == 1:
        return True
    ngpu = torch.cuda.device_count()
    for r in (part.left, part.right):
        other = r % ngpu
        if other != local and not torch.cuda.can_device_access_peer(
                local, other):
            return False
    return True


def cfg5_one_gpu(args, local, peak):
    """Config 5's step on ONE GPU, in the N = 1 line: the denominator of a
    scaling curve whose N > 1 lines run config 5 (the N = 1 headline itself
    is config 2, BASELINE's metric config).  Same path as the N > 1
    headline — the march kernel with the exchange fused (here the periodic
    x halo), a device peer barrier per iteration."""
    import torch
    from paper_2210_06438_b200.field import PeerSlabFieldIteration
    from paper_2210_06438_b200.parallel_halo import SlabPartition
    grid, n = args.cfg5_grid, N_SUB
    part = SlabPartition(grid, n, 1, 0)
    dev = torch.device("cuda", local)
    peer = PeerSlabFieldIteration(part, cfg5_slab(part, grid), VELOCITY,
                                  device=dev)
    ms = timed(lambda k: peer.iteration(), args.steps, args.warmup, 1,
               torch.cuda.current_stream())
    peer.check()
    del peer
    torch.cuda.empty_cache()
    floor = grid ** 3 * 16 / (ms * 1e-3) / 1e9
    return {"value": rate((grid // n) ** 3, n, ms), "unit": UNIT,
            "ms_per_step": ms, "subgrids": (grid // n) ** 3,
            "dram_floor_frac": floor / peak,
            "note": "config 5 (262 144 8^3 sub-grids) on this one GPU, the "
                    "N > 1 headline's path (bench.py --gpus N): the scaling "
                    "curve's N = 1 point"}


def cfg5_leg(args, world, rank, local, peak):
    """BASELINE config 5: 262 144 8^3 sub-grids (grid 512^3, blast field)
    slab-partitioned over the ranks (strong scaling: fixed total).  One step
    = one full device iteration per rank with the ghost-layer exchange
    inside it.  Headline: the peer-fused step (boundary layers stored into
    the neighbours' fields by the step kernel); the NCCL-ring exchange and
    the materialising pool path are timed beside it.  All three paths'
    first iteration from the initial field must agree bit for bit (each
    is pinned to the oracle at this size by tests/test_gpu_fullsize.py)."""
    import torch
    from paper_2210_06438_b200.field import (PeerSlabFieldIteration,
                                             SlabFieldIteration)
    from paper_2210_06438_b200.parallel_halo import SlabHydro, SlabPartition
    grid, n = args.cfg5_grid, N_SUB
    part = SlabPartition(grid, n, world, rank)
    slab = cfg5_slab(part, grid)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    S_total = (grid // n) ** 3
    use_peer = all_true(world, peer_access_ok(part, local))
    checks = {}

    def first_iteration(obj, run):
        run()
        torch.cuda.synchronize()
        return obj.owned()

    # NCCL ring (interior overlapped with the exchange)
    ring = SlabFieldIteration(part, slab, VELOCITY, device=dev)
    ref = first_iteration(ring, lambda: ring.iteration(overlap=True))
    ms_nccl = timed(lambda k: ring.iteration(overlap=True), args.steps,
                    args.warmup, world, stream)
    del ring
    torch.cuda.empty_cache()
    ms_peer = None
    clk = None
    ms_cols = None
    march_axis = None
    if use_peer:
        # the per-sub-grid kernel (one CTA per 8^3 sub-grid + halo kernels)
        # on the same peer path, for the record
        cols = PeerSlabFieldIteration(part, slab, VELOCITY, device=dev,
                                      kernel="cols")
        got = first_iteration(cols, cols.iteration)
        cols.check()
        checks["peer_per_subgrid_vs_nccl_ring"] = all_true(
            world, torch.equal(got, ref))
        del got
        ms_cols = timed(lambda k: cols.iteration(), args.steps, args.warmup,
                        world, stream)
        cols.check()
        del cols
        torch.cuda.empty_cache()
        # headline: the whole-slab march kernel (csrc/field_march.cu)
        peer = PeerSlabFieldIteration(part, slab, VELOCITY, device=dev)
        march_axis = peer.march_axis
        got = first_iteration(peer, peer.iteration)
        peer.check()
        checks["peer_fused_vs_nccl_ring"] = all_true(world,
                                                     torch.equal(got, ref))
        del got
        with ClockSampler(local) as clk:
            ms_peer = timed(lambda k: peer.iteration(), args.steps,
                            args.warmup, world, stream)
        peer.check()
        # end to end: pinned host slab in, one iteration, host slab out
        h_in = torch.from_numpy(slab).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        ms_e2e = timed(lambda k: peer.run_host(h_in, h_out),
                       max(3, args.steps // 4), 3, world, stream)
        peer.check()
        del peer
        torch.cuda.empty_cache()
    else:
        ring = SlabFieldIteration(part, slab, VELOCITY, device=dev)
        with ClockSampler(local) as clk:
            ms_nccl = timed(lambda k: ring.iteration(overlap=True),
                            args.steps, args.warmup, world, stream)
        h_in = torch.from_numpy(slab).pin_memory()
        h_out = torch.empty_like(h_in).pin_memory()
        dev_f = torch.empty(h_in.shape, dtype=torch.float64, device=dev)

        def ring_host(k):
            dev_f.copy_(h_in, non_blocking=True)
            ring.load(dev_f)
            ring.iteration(overlap=True)
            ring.store(dev_f)
            h_out.copy_(dev_f, non_blocking=True)
        ms_e2e = timed(ring_host, max(3, args.steps // 4), 3, world, stream)
        del ring, dev_f
        torch.cuda.empty_cache()
    # materialising path (ghosted sub-grid pool, faces in HBM, update)
    pool = SlabHydro(part, slab, VELOCITY, device=dev)
    got = first_iteration(pool, lambda: pool.iteration(overlap=True))
    checks["materialising_vs_nccl_ring"] = all_true(world,
                                                    torch.equal(got, ref))
    del got, ref
    ms_pool = timed(lambda k: pool.iteration(overlap=True),
                    max(3, args.steps // 2), args.warmup, world, stream)
    del pool, slab
    torch.cuda.empty_cache()
    if not all(checks.values()):
        raise SystemExit(f"bench.py cfg5: paths disagree {checks}")
    ms = ms_peer if use_peer else ms_nccl
    value = rate(S_total, n, ms)
    bytes_alg = part.subgrids * b_alg(n)
    unique = part.subgrids * 16 * n ** 3    # field in + out, 16 B per cell
    # per iteration, peer path: the march kernel + the peer barrier; NCCL
    # path: 2 halo kernels + 2 step launches (interior, boundary layers;
    # NCCL's own kernels not counted)
    launches = 2 if use_peer else 4
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": cfg5_config(world, grid),
        "run": {"path": ("peer-fused: ONE march kernel per iteration "
                         f"(warp columns marching {march_axis} through TMA "
                         "plane boxes, csrc/field_march.cu; a slab of <= 128 "
                         "planes is marched along y) stores the slab's boundary "
                         "layers into the ring neighbours' next fields over "
                         "CUDA-IPC peer memory and the next field's y/z "
                         "halos, then a device peer barrier"
                         if use_peer else
                         "NCCL ring exchange of the halo planes, interior "
                         "layers stepped while they are in flight "
                         "(no peer access between the GPUs)"),
                "subgrids_per_gpu": part.subgrids,
                "halo_bytes_per_rank_per_step": 2 * part.plane_bytes,
                "dist_backend": (os.environ.get("TASKFUSE_DIST_BACKEND",
                                                "nccl") if world > 1
                                 else None)},
        "self_check": checks,
        "gpu_launches": launches * args.steps,
        "per_subgrid_kernel_path": None if ms_cols is None else {
            "ms_per_step": ms_cols, "value": rate(S_total, n, ms_cols),
            "step": "the same peer path with one CTA per 8^3 sub-grid "
                    "(k_step_cols8s) + the y/z halo kernels"},
        "nccl_exchange_path": {
            "ms_per_step": ms_nccl, "value": rate(S_total, n, ms_nccl),
            "step": "fused step + separate NCCL ring exchange of the halo "
                    "planes, interior layers overlapped"},
        "roofline": {
            "bound": "hbm", "unit": "GB/s", "peak": peak,
            "achieved": unique / (ms * 1e-3) / 1e9,
            "frac": unique / (ms * 1e-3) / 1e9 / peak,
            "traffic": (ncu_kernel_traffic("r02_ncu_march_cfg5.txt")
                        if use_peer and world == 1 and grid == 512 else None),
            "per_subgrid_alg_bytes": 16 * n ** 3,
            "note": "march kernel; algorithmic bytes = the field read once "
                    "and written once, 16 B per cell (8 KB per 8^3 "
                    "sub-grid): every halo re-read is served by L2 in the "
                    "padded-field layout (DESIGN.md §4), so this is the "
                    "DRAM floor.  b_step_frac counts SURVEY §8(d)'s B_step "
                    "= 16 896 B per sub-grid (halo reads included)",
            "b_step_frac": part.subgrids * b_step(n) / (ms * 1e-3) / 1e9
            / peak},
        "clocks": clk.summary() if clk else None,
        "e2e": {"value": rate(S_total, n, ms_e2e), "unit": UNIT,
                "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": part.subgrids * n ** 3 * 8,
                "d2h_bytes_per_step": part.subgrids * n ** 3 * 8,
                "step": "per rank: pinned host slab -> device, pad, prime "
                        "the neighbours' halos, one iteration, slab -> "
                        "pinned host (PeerSlabFieldIteration.run_host)"},
        "materialising_path": {
            "ms_per_step": ms_pool,
            "value": rate(S_total, n, ms_pool),
            "recon_flux_hbm_frac_lower_bound":
                bytes_alg / (ms_pool * 1e-3) / 1e9 / peak,
            "step": "pack+exchange, ghost fill, recon+flux (um/up/F to "
                    "HBM), update"},
    }
    return line


# -------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--max-team", type=int, default=128)
    # two executor streams, teams alternating between them with PDL inside
    # each branch: as fast as one stream in a fresh process (33.8 vs 33.7 G)
    # and robust to the process state a multi-stream program is always in —
    # once any ordinary kernel has run on a non-default stream, a single
    # PDL chain of team launches in a graph slows by 12% (33.7 -> 29.6 G)
    # while two branches hold 33.4 G (scripts/exp_sweep_gap.py)
    ap.add_argument("--executors", type=int, default=2)
    # queue: teams formed on the fly inside the timed step and published to
    # the device queue (the headline); plan: the same teams pre-formed and
    # replayed as a CUDA graph; realtime: one host launch per closed team
    ap.add_argument("--mode", choices=("queue", "plan", "realtime", "single"),
                    default="queue")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--outputs", choices=("team", "subgrid"), default="team",
                    help="team: each team writes its lease of the packed team "
                         "buffers (the reference's slice_alloc layout); "
                         "subgrid: per-sub-grid scratch slots")
    ap.add_argument("--no-overlap", action="store_true",
                    help="disable PDL overlap of consecutive team launches")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=("auto", "cfg2", "cfg5"),
                    default="auto",
                    help="auto: config 2 on one GPU, config 5 (strong "
                         "scaling with the ghost exchange) on N > 1")
    ap.add_argument("--cfg5-grid", type=int, default=512)
    ap.add_argument("--profile-only", action="store_true",
                    help="just warm-up+timed hot-path steps (for ncu)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args))
    world, rank, local = dist_setup(args.gpus,
                                    init=args.impl != "reference")
    workload = workload_of(args, world)
    if args.impl == "reference":
        reference_arm(args, world, rank, workload)
        return
    import torch
    from paper_2210_06438_b200 import _lib
    lib = _lib.load(build_if_missing=False)
    assert lib.tf_check_device(local) == 0, "not an sm_100 device"
    peak, peak_src = peaks()
    stream = torch.cuda.current_stream()
    if workload == "cfg5":
        line = cfg5_leg(args, world, rank, local, peak)
        if rank == 0:
            print(json.dumps(line), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    wl = Workload()
    plans = None
    q = None
    if args.mode == "queue":
        step, q = queue_runner(wl, args.max_team)
        launches_per_step, hist = 1, None
    elif args.mode == "plan":
        step, nk, hist, plans = plan_runner(
            wl, args.max_team, args.executors, overlap=not args.no_overlap,
            team_buffers=args.outputs == "team")
        launches_per_step = nk
    elif args.mode == "realtime":
        step, launches, _ = realtime_runner(wl, args.max_team, args.executors)
        launches_per_step = None
        hist = None
    else:
        step = single_runner(wl)
        launches_per_step, hist = 1, {wl.S: 1}
    if args.profile_only:
        timed(step, args.steps, args.warmup, world, stream)
        return
    # settle clocks under load before the timed region (untimed)
    with ClockSampler(local) as clk:
        t_end = time.time() + 0.5
        k = 0
        while time.time() < t_end:
            step(k)
            k += 1
        if q is not None:
            q.wait()
            st0 = q.stats()
            runs0 = q.runs
        ms = timed(step, args.steps, args.warmup, world, stream)
    if q is not None:
        q.wait()
        st = q.stats()
        runs = q.runs - runs0
        teams = st["teams_formed"] - st0["teams_formed"]
        hist = {k: v - st0["size_histogram"].get(k, 0)
                for k, v in st["size_histogram"].items()
                if v - st0["size_histogram"].get(k, 0)}
        formation = {
            "teams_per_step": teams / max(1, runs),
            "mean_team": wl.S * runs / max(1, teams),
            "solo_fast_path_per_step":
                (st["solo_fast_path"] - st0["solo_fast_path"]) / max(1, runs),
            "host_us_per_step": q.host_times()}
    if launches_per_step is None:
        launches_per_step = launches[-1]
    total_S = wl.S * world
    value = rate(total_S, wl.n, ms)
    bytes_step = wl.S * b_alg(wl.n)
    achieved = bytes_step / (ms * 1e-3) / 1e9
    if args.mode == "queue":
        traffic = ncu_graph_traffic("r02_ncu_queue_consumer.csv")
        traffic_note = (
            "traffic = DRAM read+write bytes of one consumer grid over the "
            "same 4096 slices from ncu (profiles/r02_ncu_queue_consumer.csv,"
            " --cache-control none; ncu serialises the launch, so the "
            "capture is of a run whose slices were all published first: "
            "scripts/exp_consumer.py)")
    else:
        traffic = ncu_graph_traffic() if (args.mode == "plan"
                                          and args.max_team == 128) else None
        traffic_note = (
            "traffic = DRAM read+write bytes of one step from the ncu "
            "capture of this bench's own plan-graph replays "
            "(profiles/r02_ncu_plan_graph_A128.csv, --graph-profiling graph "
            "--cache-control none)")
    if q is not None:
        check = cfg2_output_check(wl, rerun=lambda: (step(0), q.wait()))
    else:
        check = cfg2_output_check(wl, plans, args.outputs == "team") \
            if plans else None
    if check is not None and not check["bitexact_vs_oracle_digest"]:
        raise SystemExit(f"bench.py: timed outputs differ from the oracle "
                         f"digests {check}")
    # the kernel timed alone: one launch over all slices (aggregation limit)
    ms_single = timed(single_runner(wl), args.steps, args.warmup, world,
                      stream)
    run = {"max_team": args.max_team, "mode": args.mode,
           "team_histogram": hist}
    if args.mode == "queue":
        run.update(formation)
        run["outputs"] = "per-sub-grid slots"
        run["step"] = ("4096 task arrivals -> C++ formation core (cap / "
                       "solo fast path / drain when every published slice "
                       "has completed) -> each closed team published to "
                       "the device queue -> one consumer grid per step "
                       "(a CTA per published slice; PDL-chained steps)")
    else:
        run["executors"] = args.executors
        run["outputs"] = ("packed team leases (slice_alloc layout)"
                          if args.outputs == "team" else "per-sub-grid slots")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": cfg2_config(),
        "run": run,
        "self_check": check,
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
            "traffic": traffic,
            "traffic_frac": (traffic / (ms * 1e-3) / 1e9 / peak
                             if traffic else None),
            "alg_bytes_per_step": bytes_step,
            "per_subgrid_alg_bytes": b_alg(wl.n),
            "note": "achieved = algorithmic bytes of the whole step / step "
                    "time (every launch in the step is the recon+flux "
                    "kernel); " + traffic_note + "; traffic_frac = "
                    "traffic / step time / peak",
            # also against the 8 TB/s HBM3e spec figure
            "spec_frac_8tbs": achieved / 8000.0,
            "kernel_alone": {
                "ms": ms_single,
                "achieved": bytes_step / (ms_single * 1e-3) / 1e9,
                "frac": bytes_step / (ms_single * 1e-3) / 1e9 / peak}},
        "clocks": clk.summary(),
    }
    if args.mode == "queue":
        line["plan"] = plan_leg(wl, args, world, stream, peak)
    line["realtime"] = realtime_leg(wl, args, world, stream, peak,
                                    with_queue=args.mode != "queue")
    line["e2e"] = e2e_leg(args, max(10, args.steps // 2), 3, world, stream)
    # the host link bounds e2e: bytes both ways per step against the
    # measured concurrent copy-engine rate (48.9 GB/s per direction on this
    # pool's boxes, profiles/r01_pcie_probe2.log)
    e = line["e2e"]
    e["link"] = {"bytes_per_step": e["h2d_bytes_per_step"]
                 + e["d2h_bytes_per_step"],
                 "floor_ms": e["h2d_bytes_per_step"] / 48.9e9 * 1e3,
                 "frac_of_upload_floor": e["h2d_bytes_per_step"] / 48.9e9
                 * 1e3 / e["ms_per_step"]}
    f_ms, fbi, fbo = e2e_faces_leg(wl, step, max(5, args.steps // 5), 3,
                                   world, stream)
    line["e2e_faces"] = {"value": rate(total_S, wl.n, f_ms), "unit": UNIT,
                         "h2d_bytes_per_step": fbi,
                         "d2h_bytes_per_step": fbo, "ms_per_step": f_ms,
                         "step": "ghosted pool in, um/up/F out"}
    line["fused_full_iteration"] = fused_legs(args, max(10, args.steps // 2),
                                              3, world, stream, peak)
    line["schemes_one_launch"] = scheme_legs(wl, max(10, args.steps // 2), 3,
                                             world, stream, peak)
    if world == 1:
        line["config5_1gpu"] = cfg5_one_gpu(args, local, peak)
    if not args.no_sweep:
        line["sweep"] = run_sweep(wl, args, world, stream, peak)
        line["reference_api"] = reference_api_legs(args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(wl.S, wl.n, GRID)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
