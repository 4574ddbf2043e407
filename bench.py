#!/usr/bin/env python
"""Benchmark: strategy-3 aggregated FP64 hydro reconstruct+flux on B200.

Metric (BASELINE.json): sub-grid cell-updates/s of the hydro
reconstruct+flux hot path vs aggregation level, and % of HBM peak.

Workload (BASELINE.json configs[1]): Sod shock tube, 4096 8^3 sub-grids
(grid 128^3), velocity (1,1,1).  One STEP = one iteration of the aggregated
reconstruct+flux region over all sub-grids: the 4096 task arrivals are
formed into teams by the strategy-3 formation core (max_team = 128 by
default, parents = S/max_team as HydroSim does, step.py:61), each team is one
launch of the batched TMA kernel, and the iteration's team launches replay as
one CUDA graph over the executor streams.  Inputs are device-resident; two
input pools alternate between steps (per-step working set 385 MB, 3x L2).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun): weak scaling, each rank owns its own 4096 sub-grids;
the step has no data-path collective (the recon+flux region is
embarrassingly parallel), value = all ranks' cell-updates / max-rank time.
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
def dist_setup(gpus: int):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # one process per GPU; the modulo only matters when a test squeezes
        # several ranks onto fewer GPUs (TASKFUSE_DIST_BACKEND=gloo)
        if torch.cuda.is_available():
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
        backend = os.environ.get("TASKFUSE_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group(
                "nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


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
    t_end = time.time() + settle_s
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
                team_buffers=False):
    from paper_2210_06438_b200.strategy3 import TeamPlan, form_teams
    teams = form_teams(range(wl.S), max_team, executors, parents)
    plans = [TeamPlan(teams, p, wl.n, VELOCITY, wl.um, wl.up, wl.F,
                      executors, amax=wl.amax, overlap=overlap,
                      team_buffers=team_buffers)
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
    out["realtime_queue"] = {}
    from paper_2210_06438_b200.strategy3 import (QueueExecutor,
                                                 default_parents)
    # an int32 array, so the per-step C call does not convert a list
    arrivals = np.arange(wl.S, dtype=np.int32)
    for A in (1, 4, 16, 64, 128):
        q = QueueExecutor("reconstruct", A, default_parents(wl.S, A), wl.n)
        ms = timed(lambda k: q.run(wl.pools[k % len(wl.pools)], VELOCITY,
                                   arrivals, wl.um, wl.up, wl.F,
                                   amax=wl.amax), ks, kw, world, stream)
        st = q.stats()
        out["realtime_queue"][A] = {
            "cell_updates_per_s": rate(wl.S, wl.n, ms), "ms_per_iter": ms,
            "mean_team": st["teams_formed"] and
            sum(k * v for k, v in st["size_histogram"].items())
            / st["teams_formed"],
            "solo_fast_path": st["solo_fast_path"]}
        del q
    for E in (1, 8, 32, 128):
        # strategy 2: per-task launches (A = 1) spread over E streams
        step, nk, _, _ = plan_runner(wl, 1, E, parents=E)
        ms = timed(step, ks, kw, world, stream)
        out["strategy2"][E] = {"cell_updates_per_s": rate(wl.S, wl.n, ms),
                               "ms_per_iter": ms, "launches": nk}
    wl16 = Workload(n=16, grid=wl.grid, field=FIELD)
    for E in sorted({args.executors, 4}):
        step, nk, _, _ = plan_runner(wl16, 1, E)
        ms = timed(step, ks, kw, world, stream)
        out["strategy1"][f"16^3_A1_E{E}"] = {
            "cell_updates_per_s": rate(wl16.S, 16, ms), "ms_per_iter": ms,
            "launches": nk, "hbm_frac": wl16.S * b_alg(16) / (ms * 1e-3)
            / (peak * 1e9)}
    del wl16
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
    for E in (8, 32, 128):
        step, nk, _, _ = plan_runner(wl3, 1, E, parents=E)
        ms = timed(step, max(3, ks // 4), kw, world, stream)
        res["strategy2"][E] = {"cell_updates_per_s": rate(wl3.S, wl3.n, ms),
                               "ms_per_iter": ms, "launches": nk}
    del wl3
    return res


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
                       f"(prep+reconstruct+flux bodies, oracle port of "
                       f"hydro/kernels.py), spawn pool of {cb.workers} "
                       f"workers, slowest worker, best of {len(times)} "
                       f"passes; CPU {cpu_model()}")}


def reference_arm(args, world, rank):
    """--impl reference: the reference's CPU path (oracle port; the
    reference is pure Python and is not present on GPU boxes) on all host
    cores, same metric/config/unit."""
    if rank != 0:
        return
    from oracle.cpu_baseline import CpuBaseline, cpu_model
    S = (GRID // N_SUB) ** 3
    cb = CpuBaseline(FIELD, GRID, N_SUB, VELOCITY, range(S))
    try:
        for _ in range(args.warmup):
            cb.step()
        times = [cb.step() for _ in range(args.steps)]
    finally:
        cb.close()
    ms = 1e3 * sum(times) / len(times)
    value = rate(S, N_SUB, ms)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config 2: Sod shock tube, 4096 8^3 "
                   "sub-grids, one reconstruct+flux iteration per step",
                   "subgrids": S, "subgrid_n": N_SUB},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cb.workers,
                         "kind": "port",
                         "sample": f"all {S} sub-grids per step, spawn pool "
                                   f"of {cb.workers}, CPU {cpu_model()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def e2e_leg(args, steps, warmup, world, stream):
    """Same metric through the public API with HOST buffers
    (strategy3.AggregatedIteration.run_host): every step copies the global
    field host->device from pinned memory, scatters it into the sub-grid
    pool, fills ghosts, runs the aggregated reconstruct+flux team plan and
    the update, and reads the updated field back device->host.  More work
    than the recon+flux metric counts (ghost fill + update), so it is a
    conservative end-to-end rate."""
    import torch
    from paper_2210_06438_b200.hydro import sod_field
    from paper_2210_06438_b200.strategy3 import AggregatedIteration
    it = AggregatedIteration(GRID, N_SUB, VELOCITY, max_team=args.max_team,
                             executors=args.executors)
    host_in = sod_field(GRID, "cpu").pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()

    def step(k):
        it.run_host(host_in, host_out)
    ms = timed(step, steps, warmup, world, stream)
    torch.cuda.synchronize()
    return ms, host_in.numel() * 8, host_out.numel() * 8, \
        it.launches_per_step + 2


def fused_legs(args, steps, warmup, world, stream, peak):
    """The fused full iteration (field.FieldIteration, SURVEY §8 f #2) on
    config 2: device-resident step and the host round trip."""
    import torch
    from paper_2210_06438_b200.hydro import sod_field
    from paper_2210_06438_b200.field import FieldIteration
    it = FieldIteration(GRID, N_SUB, VELOCITY, max_team=args.max_team,
                        executors=args.executors)
    it.load(sod_field(GRID, "cuda"))
    ms_dev = timed(lambda k: it.step(), steps, warmup, world, stream)
    host_in = sod_field(GRID, "cpu").pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    ms_e2e = timed(lambda k: it.run_host(host_in, host_out), steps, warmup,
                   world, stream)
    from paper_2210_06438_b200.field import HostPipeline
    pipe = HostPipeline(it, host_in, host_out)
    ms_pipe = timed(lambda k: pipe.run(), steps, warmup, world, stream)
    S = (GRID // N_SUB) ** 3
    n = N_SUB
    fused_bytes = S * b_step(n)
    return {
        "device": {"value": rate(S * world, n, ms_dev), "unit": UNIT,
                   "ms_per_step": ms_dev,
                   "hbm_frac": fused_bytes / (ms_dev * 1e-3) / 1e9 / peak,
                   "launches_per_step": it.launches_per_step,
                   "step": "one fused recon+flux+update kernel per team, "
                           "each also writing its sub-grids' share of the "
                           "next field's periodic halos (CUDA graph)"},
        "e2e": {"value": rate(S * world, n, ms_e2e), "unit": UNIT,
                "ms_per_step": ms_e2e,
                "h2d_bytes_per_step": host_in.numel() * 8,
                "d2h_bytes_per_step": host_out.numel() * 8},
        "e2e_pipelined": {
            "value": rate(S * world, n, ms_pipe), "unit": UNIT,
            "ms_per_step": ms_pipe,
            "h2d_bytes_per_step": host_in.numel() * 8,
            "d2h_bytes_per_step": host_out.numel() * 8,
            "gpu_launches_per_step": pipe.launches,
            "step": "field.HostPipeline: tapered x-chunks (sub-grid layers "
                    "[1,3,4,4,3,1]), copy-engine upload shifted by the x "
                    "halo / one pad+halo kernel / fused step / zero-copy download "
                    "kernel, overlapped, captured as one CUDA graph"},
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


def cfg5_leg(args, world, rank, local, peak):
    """BASELINE config 5: 262 144 8^3 sub-grids (grid 512^3, blast field)
    slab-partitioned over the ranks (strong scaling: fixed total).  One step
    = one full device iteration per rank: pack halo planes, ring exchange
    (NCCL P2P), ghost fill (interior layers overlapped with the exchange),
    aggregated reconstruct+flux, update."""
    import numpy as np
    import torch
    from paper_2210_06438_b200.field import SlabFieldIteration
    from paper_2210_06438_b200.parallel_halo import SlabHydro, SlabPartition
    grid, n = args.cfg5_grid, N_SUB
    part = SlabPartition(grid, n, world, rank)
    a = part.x0 * n
    x = (np.arange(grid) + 0.5) / grid
    # the slab of initial_field (scenario.py:30-37), evaluated per slab
    xs = x[a:a + part.mx * n]
    r2 = ((xs - 0.5) ** 2)[:, None, None] + ((x - 0.5) ** 2)[None, :, None] \
        + ((x - 0.5) ** 2)[None, None, :]
    slab = 1.0 + 1.0 * np.exp(-r2 / (2.0 * 0.1 ** 2))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    # fused path with the exchange fused into the compute over peer memory
    # (the step measured for `value`)
    from paper_2210_06438_b200.field import PeerSlabFieldIteration
    peer = PeerSlabFieldIteration(part, slab, VELOCITY, device=dev)
    with ClockSampler(local) as clk:
        ms = timed(lambda k: peer.iteration(), args.steps, args.warmup,
                   world, stream)
    peer.check()
    del peer
    torch.cuda.empty_cache()
    # fused step with a separate NCCL ring exchange, interior overlapped
    fused = SlabFieldIteration(part, slab, VELOCITY, device=dev)
    ms_nccl = timed(lambda k: fused.iteration(overlap=True), args.steps,
                    args.warmup, world, stream)
    del fused
    torch.cuda.empty_cache()
    # materialising path (ghosted sub-grid pool, faces in HBM, update)
    pool = SlabHydro(part, slab, VELOCITY, device=dev)
    ms_pool = timed(lambda k: pool.iteration(overlap=True),
                    max(3, args.steps // 2), args.warmup, world, stream)
    del pool, slab
    torch.cuda.empty_cache()
    S_total = (grid // n) ** 3
    value = rate(S_total, n, ms)
    bytes_alg = part.subgrids * b_alg(n)
    fused_bytes = part.subgrids * b_step(n)
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config 5: blast wave, {S_total} 8^3 "
                   f"sub-grids (grid {grid}^3) slab-partitioned over "
                   f"{world} GPU(s); one full iteration per step (halo "
                   "exchange, ghost fill, recon+flux, update)",
                   "subgrids_per_gpu": part.subgrids,
                   "halo_bytes_per_rank_per_step": 2 * part.plane_bytes,
                   "parallelism": f"x-slab partition x{world}; boundary "
                                  "layers stored into the ring neighbours' "
                                  "fields by the step kernel over CUDA-IPC "
                                  "peer memory + device peer barrier"},
        "nccl_exchange_path": {
            "ms_per_step": ms_nccl, "value": rate(S_total, n, ms_nccl),
            "step": "fused step + separate NCCL ring exchange of the halo "
                    "planes, interior layers overlapped"},
        "roofline": {
            "bound": "hbm", "unit": "GB/s", "peak": peak,
            "achieved": fused_bytes / (ms * 1e-3) / 1e9,
            "frac": fused_bytes / (ms * 1e-3) / 1e9 / peak,
            "traffic": ncu_traffic_per_launch(
                part.subgrids, "r01_ncu_step_fused_cfg5g256.txt"),
            # the field itself read once and written once (16 B per cell):
            # the DRAM floor of the fused step if every halo re-read hits L2
            "unique_dram_frac": part.subgrids * 16 * n ** 3
            / (ms * 1e-3) / 1e9 / peak,
            "note": "fused step, SURVEY §8(d) B_step = 8[(n+2)^3 + "
                    "6(n+2)^2 + n^3] = 16 896 B per 8^3 sub-grid; halo "
                    "refresh and exchange inside the step. frac can exceed "
                    "1: B_step counts each sub-grid's halo reads, which the "
                    "padded-field layout serves from L2 (traffic = DRAM "
                    "bytes per step-kernel launch from the ncu capture at "
                    "grid 256, scaled: ~7.4 KB per sub-grid). "
                    "unique_dram_frac = 16 B per cell (field in + out) / "
                    "step time / peak: the DRAM floor's fraction; the "
                    "kernel is latency / L2-bound, DESIGN.md §4"},
        "clocks": clk.summary(),
        "materialising_path": {
            "ms_per_step": ms_pool,
            "value": rate(S_total, n, ms_pool),
            "recon_flux_hbm_frac_lower_bound":
                bytes_alg / (ms_pool * 1e-3) / 1e9 / peak,
            "step": "pack+exchange, ghost fill, recon+flux (um/up/F to "
                    "HBM), update"},
    }


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
    ap.add_argument("--mode", choices=("plan", "realtime", "single"),
                    default="plan")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--outputs", choices=("team", "subgrid"), default="team",
                    help="team: each team writes its lease of the packed team "
                         "buffers (the reference's slice_alloc layout); "
                         "subgrid: per-sub-grid scratch slots")
    ap.add_argument("--no-overlap", action="store_true",
                    help="disable PDL overlap of consecutive team launches")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=("cfg2", "cfg5"), default="cfg2")
    ap.add_argument("--cfg5-grid", type=int, default=512)
    ap.add_argument("--profile-only", action="store_true",
                    help="just warm-up+timed hot-path steps (for ncu)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    import torch
    from paper_2210_06438_b200 import _lib
    lib = _lib.load(build_if_missing=False)
    assert lib.tf_check_device(local) == 0, "not an sm_100 device"
    peak, peak_src = peaks()
    stream = torch.cuda.current_stream()
    if args.workload == "cfg5":
        line = cfg5_leg(args, world, rank, local, peak)
        if rank == 0:
            print(json.dumps(line), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    wl = Workload()
    if args.mode == "plan":
        step, nk, hist, _ = plan_runner(wl, args.max_team, args.executors,
                                        overlap=not args.no_overlap,
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
        ms = timed(step, args.steps, args.warmup, world, stream)
    if launches_per_step is None:
        launches_per_step = launches[-1]
    total_S = wl.S * world
    value = rate(total_S, wl.n, ms)
    bytes_step = wl.S * b_alg(wl.n)
    achieved = bytes_step / (ms * 1e-3) / 1e9
    # the kernel timed alone: one launch over all slices (aggregation limit)
    ms_single = timed(single_runner(wl), args.steps, args.warmup, world,
                      stream)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {
            "workload": "config 2: Sod shock tube, 4096 8^3 FP64 sub-grids "
                        "per GPU, one aggregated reconstruct+flux iteration "
                        "per step",
            "subgrids_per_gpu": wl.S, "subgrid_n": wl.n, "grid": GRID,
            "max_team": args.max_team, "executors": args.executors,
            "mode": args.mode, "team_histogram": hist,
            "outputs": ("packed team leases (slice_alloc layout)"
                        if args.outputs == "team" else "per-sub-grid slots"),
            "parallelism": f"sub-grid partition x{world} (no collective)",
            "l2": "two input pools alternate; per-step working set "
                  f"{(bytes_step + wl.S * 8 * 2744) / 1e6:.0f} MB vs 126 MB L2"},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
            "traffic": ncu_traffic_per_launch(args.max_team),
            "alg_bytes_per_launch": b_alg(wl.n) * args.max_team,
            "per_subgrid_alg_bytes": b_alg(wl.n),
            "note": "achieved = algorithmic bytes of the whole step / step "
                    "time (every launch in the step is the recon+flux team "
                    "kernel); traffic = dram read+write per team launch from "
                    "the committed ncu --set full capture of the same kernel "
                    "(profiles/r01_ncu_recon_flux_single.txt), per slice x "
                    "team size",
            # also against the 8 TB/s HBM3e spec figure
            "spec_frac_8tbs": achieved / 8000.0,
            "kernel_alone": {
                "ms": ms_single,
                "achieved": bytes_step / (ms_single * 1e-3) / 1e9,
                "frac": bytes_step / (ms_single * 1e-3) / 1e9 / peak}},
        "clocks": clk.summary(),
    }
    e_ms, bi, bo, e_launch = e2e_leg(args, max(10, args.steps // 2), 3,
                                     world, stream)
    line["e2e_materialising"] = {
        "value": rate(total_S, wl.n, e_ms), "unit": UNIT,
        "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
        "ms_per_step": e_ms,
        "step": "host field (pinned) -> device scatter -> ghost fill -> "
                "aggregated recon+flux teams (um/up/F to HBM) -> update -> "
                "gather -> host field (AggregatedIteration.run_host)",
        "gpu_launches_per_step": e_launch}
    f_ms, fbi, fbo = e2e_faces_leg(wl, step, max(5, args.steps // 5), 3,
                                   world, stream)
    line["fused_full_iteration"] = fused_legs(args, max(10, args.steps // 2),
                                              3, world, stream, peak)
    # headline e2e: the public host->host iteration API (pinned host field
    # in, one hydro iteration = reconstruct + flux + update of every
    # sub-grid, pinned host field out), transfers overlapped with compute
    line["e2e"] = dict(line["fused_full_iteration"]["e2e_pipelined"])
    # the host link bounds e2e: bytes both ways per step against the
    # measured concurrent copy-engine rate (48.9 GB/s per direction on this
    # pool's boxes, profiles/r01_pcie_probe2.log)
    e = line["e2e"]
    link = e["h2d_bytes_per_step"] + e["d2h_bytes_per_step"]
    e["link"] = {"bytes_per_step": link,
                 "achieved_GBps": link / (e["ms_per_step"] * 1e-3) / 1e9,
                 "bidirectional_peak_GBps": 2 * 48.9,
                 "frac": link / (e["ms_per_step"] * 1e-3) / 1e9 / 97.8,
                 "floor_ms": max(e["h2d_bytes_per_step"],
                                 e["d2h_bytes_per_step"]) / 48.9e9 * 1e3}
    line["schemes_one_launch"] = scheme_legs(wl, max(10, args.steps // 2), 3,
                                             world, stream, peak)
    line["e2e_faces"] = {"value": rate(total_S, wl.n, f_ms), "unit": UNIT,
                         "h2d_bytes_per_step": fbi,
                         "d2h_bytes_per_step": fbo, "ms_per_step": f_ms,
                         "step": "ghosted pool in, um/up/F out"}
    if not args.no_sweep:
        line["sweep"] = run_sweep(wl, args, world, stream, peak)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_leg(wl.S, wl.n, GRID)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
