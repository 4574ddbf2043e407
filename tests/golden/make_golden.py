"""Generate the golden fixtures from the UNMODIFIED reference implementation.

Run in the build container (the reference is not present on GPU boxes):

    cd /tmp && PYTHONDONTWRITEBYTECODE=1 python /root/repo/tests/golden/make_golden.py

It imports `taskfuse` from /root/reference/pkg/src (read-only; no bytecode is
written) and records:

* hydro.json.gz — per case (grid, sub-grid edge, field, velocity): sha256
  digests of every stage output of every sub-grid, computed by the
  reference's own task bodies (prep/reconstruct/flux/reduce/update after
  exchange_ghosts; hydro/kernels.py, hydro/scenario.py), plus whole-grid
  reference_step digests (hydro/reference.py) and the minmod edge vectors.
* hydro_small.npz — full arrays of two sub-grids of one case, for debugging.
* traces.json.gz — aggregation formation traces: the signal log the
  reference's AggregationRegion saw (arrivals with the stream_busy answer,
  stream drains) and the teams it closed, captured by wrapping
  (not modifying) AggregationRegion.enter/_close and VirtualDevice
  .stream_busy/_op_finished.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import sys
import time
from fractions import Fraction
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from taskfuse import aggregator as agg_mod  # noqa: E402
from taskfuse import device as dev_mod  # noqa: E402
from taskfuse.aggregator import AggregationRegion  # noqa: E402
from taskfuse.bench import calibrate, run_cell  # noqa: E402
from taskfuse.bufferpool import BufferPool  # noqa: E402
from taskfuse.device import (DeviceProfile, KernelSpec, VirtualDevice,  # noqa
                             load_profile)
from taskfuse.executorpool import ExecutorPool  # noqa: E402
from taskfuse.hydro import kernels as K  # noqa: E402
from taskfuse.hydro import (HydroSim, driver, exchange_ghosts,  # noqa: E402
                            initial_field, make_state, reference_step)
from taskfuse.hydro.scenario import GHOST, dt_over_dx  # noqa: E402
from taskfuse.sched import (Scheduler, SchedulerConfig, await_all,  # noqa
                            charge)

OUT = Path(__file__).resolve().parent


def digest(a) -> str:
    arr = np.ascontiguousarray(a, dtype="<f8")
    return hashlib.sha256(arr.tobytes()).hexdigest()


def sod(g):
    x = (np.arange(g) + 0.5) / g
    col = np.where(x < 0.5, 1.0, 0.125)
    return np.broadcast_to(col[:, None, None], (g, g, g)).copy()


def stress(g, seed=20221012):
    return 1.0 + 0.1 * np.random.default_rng(seed).random((g, g, g))


FIELDS = {"blast": initial_field, "sod": sod, "stress": stress}

CASES = [
    # name, grid, n, field, velocity
    ("blast16_n8_v111", 16, 8, "blast", (1.0, 1.0, 1.0)),
    ("stress16_n8_vneg", 16, 8, "stress", (-1.0, 0.5, -0.25)),
    ("stress16_n8_vmix", 16, 8, "stress", (0.7, -1.3, 0.0)),
    ("sod32_n8_v111", 32, 8, "sod", (1.0, 1.0, 1.0)),       # BASELINE config 1
    ("stress32_n8_vneg", 32, 8, "stress", (-1.0, 0.5, -0.25)),
    ("stress32_n16_v111", 32, 16, "stress", (1.0, 1.0, 1.0)),  # strategy 1
    ("stress32_n16_vmix", 32, 16, "stress", (0.7, -1.3, 0.0)),
]


def hydro_case(name, grid, n, field_name, velocity, keep=None):
    field = FIELDS[field_name](grid)
    state = make_state(n, grid, field=field)
    dt_dx = dt_over_dx(velocity)
    per = {"w": [], "um": [], "up": [], "F": [], "reduce": [], "next": []}
    stacks = {k: [] for k in ("w", "um", "up", "F", "next")}
    kept = {}
    for b in state.blocks:
        exchange_ghosts(state, b)
    for idx, b in enumerate(state.blocks):
        scratch = K.make_scratch(n)
        u_ext = state.u[b]
        out_ext = state.u_next[b]
        K.prep_body(u_ext, scratch)
        K.reconstruct_body(scratch, n)
        K.flux_body(scratch, n, velocity)
        K.reduce_body(scratch, velocity)
        K.update_body(u_ext, out_ext, scratch, n, dt_dx)
        own = out_ext[GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n]
        for key, arr in (("w", scratch["w"]), ("um", scratch["um"]),
                         ("up", scratch["up"]), ("F", scratch["F"]),
                         ("next", own)):
            per[key].append(digest(arr))
            stacks[key].append(np.array(arr))
        per["reduce"].append(float(scratch["reduce_out"][0]))
        if keep and idx in keep:
            for key in ("w", "um", "up", "F"):
                kept[f"{name}_{idx}_{key}"] = np.array(scratch[key])
            kept[f"{name}_{idx}_next"] = np.array(own)
    one = reference_step(field, velocity)
    two = reference_step(one, velocity)
    return {
        "name": name, "grid": grid, "n": n, "field": field_name,
        "velocity": list(velocity), "dt_dx": dt_dx,
        "field_digest": digest(field),
        "per_subgrid": per,
        "stacked": {k: digest(np.stack(v)) for k, v in stacks.items()},
        "reference_step_1": digest(one),
        "reference_step_2": digest(two),
        "advect_once": digest(reference_step(field, velocity, iterations=1)),
    }, kept


def minmod_vectors():
    # SURVEY Appendix A probe P8 plus signed zeros, infinities and ties
    a = np.array([1e-200, -1e-200, 2.0, 3.0, -0.0, np.nan, 1.0, -2.0, 0.5,
                  np.inf, -np.inf, 5e-324, 2.0, -3.0, 4.0])
    b = np.array([1e-200, -1e-200, 2.0, -3.0, 1.0, 1.0, np.nan, -2.5, 0.25,
                  1.0, -np.inf, 5e-324, 2.0, -1.0, 3.9999999999999996])
    out = K._minmod(a, b)
    enc = lambda v: [float(x).hex() for x in v]  # noqa: E731
    return {"a": enc(a), "b": enc(b), "out": enc(out)}


# ------------------------------------------------------------ trace capture
class Recorder:
    def __init__(self, tracked, labeler):
        self.tracked = set(tracked)
        self.labeler = labeler
        self.events = []
        self.closes = {name: [] for name in tracked}
        self.current = None

    def install(self):
        rec = self
        orig_enter = AggregationRegion.enter
        orig_close = AggregationRegion._close
        orig_busy = VirtualDevice.stream_busy
        orig_fin = VirtualDevice._op_finished

        def enter(region):
            if region.name not in rec.tracked:
                return orig_enter(region)
            task = region.sched._current
            ev = ["arrive", region.name, rec.labeler(task.label), None]
            rec.events.append(ev)
            rec.current = (region, ev)
            try:
                return orig_enter(region)
            finally:
                rec.current = None

        def stream_busy(device, sid, at=None):
            res = orig_busy(device, sid, at)
            if rec.current is not None:
                rec.current[1][3] = bool(res)
            return res

        def close(region, team):
            if region.name in rec.tracked:
                if rec.current is not None and rec.current[0] is region:
                    reason = ("cap" if len(team.members) >= region.max_team
                              else "solo")
                else:
                    reason = "drain"
                tags = [rec.labeler(m._task.label) for m in team.members]
                rec.closes[region.name].append(
                    [team.parent.index, tags, reason])
            return orig_close(region, team)

        def op_finished(device, op):
            stream = op.stream
            if len(stream.queue) == 1 and stream.idle_callbacks:
                rec.events.append(["drain", stream.index])
            return orig_fin(device, op)

        self._saved = (orig_enter, orig_close, orig_busy, orig_fin)
        AggregationRegion.enter = enter
        AggregationRegion._close = close
        VirtualDevice.stream_busy = stream_busy
        VirtualDevice._op_finished = op_finished

    def uninstall(self):
        (AggregationRegion.enter, AggregationRegion._close,
         VirtualDevice.stream_busy, VirtualDevice._op_finished) = self._saved


def task_labeler(label):
    # "task:N" -> N
    return int(label.split(":")[1])


def hydro_labeler(m):
    def lab(label):
        # "hydro(bx, by, bz)" -> lexicographic sub-grid id
        bx, by, bz = (int(v) for v in label[len("hydro("):-1].split(","))
        return (bx * m + by) * m + bz
    return lab


PROF = DeviceProfile(
    cu_count=4, resident_blocks_per_cu=2, t_block=100, t_launch=10,
    t_copy_base=5, t_copy_per_byte=Fraction(1, 2),
    max_concurrent_kernels=8, concurrency_penalty=Fraction(0),
    t_device_sync=0,
)


def rig_trace(name, max_team, executors, visits, primes=()):
    """The reference test_aggregator.py Rig scenarios (:23-55)."""
    rec = Recorder(["r"], task_labeler)
    rec.install()
    try:
        sched = Scheduler(SchedulerConfig(worker_count=32))
        device = VirtualDevice(sched, PROF)
        pool = ExecutorPool(sched, device, executors)
        buffers = BufferPool(device)
        region = AggregationRegion(sched, pool, buffers, "r", max_team)
        for idx in primes:
            device.enqueue_kernel(pool.executors[idx].stream_id,
                                  KernelSpec("prime", 1, Fraction(1)))

        def visit(delay, length=4, bps=2):
            def body():
                if delay:
                    yield charge(delay)
                member = yield region.enter()
                member.slice_alloc("pinned_host", "f8", length)
                member.slice_alloc("device", "f8", length)
                member.slice_copy("h2d", length * 8)
                member.slice_launch("fused", bps, Fraction(1))
                d2h = member.slice_copy("d2h", length * 8)
                yield await_all(d2h)
                member.leave()
            return body

        for i, (delay, bps) in enumerate(visits):
            sched.spawn(visit(delay, bps=bps), label=f"task:{i}")
        sched.run()
        st = region.stats()
    finally:
        rec.uninstall()
    return {
        "name": name, "executors": executors,
        "regions": [{"name": "r", "max_team": max_team,
                     "parents": len(region.parents)}],
        "events": rec.events, "closes": rec.closes,
        "stats": {"r": {"teams_formed": st.teams_formed,
                        "solo_fast_path": st.solo_fast_path,
                        "histogram": {str(k): v for k, v in
                                      st.size_histogram.items()}}},
    }


def hydro_trace(name, profile, work_factors, n, grid, executors, max_team,
                steps=1, policy="round_robin", tracked=("reconstruct", "flux")):
    m = grid // n
    rec = Recorder(list(tracked), hydro_labeler(m))
    rec.install()
    try:
        if work_factors is None:
            row, sim, device = run_cell(profile, calibrate(profile)
                                        .work_factors, n, executors,
                                        max_team, steps, policy=policy,
                                        grid_n=grid)
        else:
            sched = Scheduler(SchedulerConfig(worker_count=32))
            state = make_state(n, grid)
            device = VirtualDevice(sched, profile)
            pool = ExecutorPool(sched, device, executors, policy)
            sim = HydroSim(sched, state, pool, max_team=max_team,
                           work_factors=work_factors)
            sched.spawn(lambda: driver(sim, steps), label="driver")
            sched.run()
    finally:
        rec.uninstall()
    regions = []
    stats = {}
    for rname in tracked:
        reg = sim.regions[rname]
        st = reg.stats()
        regions.append({"name": rname, "max_team": max_team,
                        "parents": len(reg.parents)})
        stats[rname] = {"teams_formed": st.teams_formed,
                        "solo_fast_path": st.solo_fast_path,
                        "histogram": {str(k): v for k, v in
                                      st.size_histogram.items()}}
    return {"name": name, "executors": executors, "regions": regions,
            "events": rec.events, "closes": rec.closes, "stats": stats,
            "subgrids": m ** 3}


def main():
    t0 = time.time()
    cases, kept = [], {}
    for case in CASES:
        keep = {0, 5} if case[0] == "stress16_n8_vneg" else None
        res, k = hydro_case(*case, keep=keep)
        cases.append(res)
        kept.update(k)
        print(f"hydro {case[0]}: {time.time() - t0:.1f}s", flush=True)
    hydro = {"generator": "tests/golden/make_golden.py",
             "reference": "/root/reference/pkg/src/taskfuse",
             "numpy": np.__version__, "cases": cases,
             "minmod": minmod_vectors()}
    with gzip.open(OUT / "hydro.json.gz", "wt") as fh:
        json.dump(hydro, fh)
    np.savez_compressed(OUT / "hydro_small.npz", **kept)

    traces = []
    # test_aggregator.py scenarios
    traces.append(rig_trace("rig_close_paths", 2, 1, [(0, 2)] * 4))
    traces.append(rig_trace("rig_drain", 8, 1, [(0, 2), (5, 2), (6, 2)]))
    traces.append(rig_trace("rig_team16", 16, 1, [(0, 8)] * 16, primes=(0,)))
    traces.append(rig_trace("rig_parents_rr", 2, 2, [(0, 2)] * 4,
                            primes=(0, 1)))
    traces.append(rig_trace("rig_cap4_delays", 4, 1,
                            [((i * 7) % 40, 2) for i in range(20)]))
    func = DeviceProfile(cu_count=100, resident_blocks_per_cu=2, t_block=100,
                         t_launch=10, t_copy_base=5,
                         t_copy_per_byte=Fraction(0),
                         max_concurrent_kernels=128,
                         concurrency_penalty=Fraction(0), t_device_sync=10)
    wf = {k: Fraction(35000, 3) for k in K.KERNEL_ORDER}
    traces.append(hydro_trace("hydro_func_e4_cap8", func, wf, 8, 16, 4, 8,
                              steps=2, policy="load_balanced",
                              tracked=K.KERNEL_ORDER))
    a100 = load_profile("a100like")
    for cap in (1, 4, 16, 64):
        traces.append(hydro_trace(f"cfg1_a100_e1_cap{cap}", a100, None, 8, 32,
                                  1, cap))
        print(f"trace cfg1 cap{cap}: {time.time() - t0:.1f}s", flush=True)
    traces.append(hydro_trace("cfg1_a100_e4_cap16", a100, None, 8, 32, 4, 16))
    for cap in (1, 4, 16, 64, 128):
        traces.append(hydro_trace(f"cfg2_a100_e1_cap{cap}", a100, None, 8,
                                  128, 1, cap, tracked=("reconstruct",)))
        print(f"trace cfg2 cap{cap}: {time.time() - t0:.1f}s", flush=True)
    with gzip.open(OUT / "traces.json.gz", "wt") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "traces": traces}, fh)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
