"""Strategy-3 work aggregation on real CUDA streams — the bulk (throughput)
interface to the C++ formation core and the batched sm_100a kernels.

Three ways to run one iteration of the aggregated reconstruct+flux region
over a set of sub-grid task arrivals:

* `RealtimeExecutor.run` — the reference's demand-driven policy
  (aggregator.py:284-345) in real time: an arrival finding its parent's
  stream idle runs alone; otherwise it joins the forming team, which closes
  at `max_team` or when the stream drains (observed with cudaEventQuery).
  One kernel launch per closed team, team ids inside the launch parameters.
* `form_teams` + `TeamPlan` — the teams a saturated device forms (every
  busy query answers "busy", so teams close at the cap; the arrival stream's
  end closes the rest) captured once into a CUDA graph with one kernel node
  per team on its parent's executor branch.  An iterative solver re-forms the
  same teams every iteration, so replaying the graph is the steady state.
* `recon_flux_all` — the limit of aggregation: one launch over all slices.

Arrival order follows HydroSim.driver (step.py:133-137): sub-grids in
lexicographic order, parents = max(1, S // max_team) (step.py:61), parent of
arrival i = i % parents (aggregator.py:298), parent p on executor
(crc32(region) % E + p) % E (aggregator.py:273-277).
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ValidationError

_CLOSE = {1: "cap", 2: "solo", 3: "drain"}


def _check_recon_args(pool, n, um, up, F, amax, slots=None) -> int:
    """The checks ops.recon_flux makes (shape, dtype, device, capacity of
    every output) before a bulk path hands raw pointers to TMA maps and
    device stores; returns the pool's slice count."""
    from . import ops
    ops._check_n(n)
    S = ops._check_pool(pool, n)
    slots = S if slots is None else slots
    for t, nm in ((um, "um"), (up, "up"), (F, "F")):
        ops._check_faces(t, n, slots, nm)
    if amax is not None:
        ops._need_cuda_f64(amax, "amax")
        if amax.numel() < slots:
            raise ValidationError(f"amax must hold >= {slots} values")
    return S


def default_parents(subgrids: int, max_team: int) -> int:
    """step.py:61 — one parent per expected team."""
    return max(1, subgrids // max_team)


class FormationCore:
    """Owns one C++ tf_region (AggregationRegion formation state)."""

    def __init__(self, name: str, max_team: int, parents: int,
                 executors: int):
        self.lib = _lib.load()
        if not 1 <= max_team <= _lib.MAX_TEAM:
            raise ValidationError(
                f"max_team must be in 1..{_lib.MAX_TEAM}, got {max_team}")
        if parents < 1 or executors < 1:
            raise ValidationError("parents and executors must be >= 1")
        h = C.c_void_p()
        _lib.check(self.lib.tf_region_create(name.encode(), max_team, parents,
                                             executors, C.byref(h)),
                   "tf_region_create")
        self.handle = h
        self.name = name
        self.max_team = max_team
        self.parents = parents
        self.executors = executors

    def parent_executor(self, parent: int) -> int:
        return self.lib.tf_region_parent_executor(self.handle, parent)

    def enter(self, tag: int, busy) -> _lib.EnterResult:
        res = _lib.EnterResult()
        cb = _lib.BUSY_FN(lambda ctx, e: int(bool(busy(e))))
        _lib.check(self.lib.tf_region_enter(self.handle, int(tag), cb, None,
                                            C.byref(res)), "tf_region_enter")
        return res

    def stream_idle(self, executor: int) -> list[int]:
        # sized by the core's own watcher count: every closed team's id is
        # returned (the core never closes a team it could not report)
        cap = self.lib.tf_region_watch_count(self.handle, executor)
        if cap < 0:
            _lib.check(-cap, "tf_region_watch_count")
        if cap == 0:
            return []
        buf = (C.c_int64 * cap)()
        n = self.lib.tf_region_stream_idle(self.handle, executor, buf, cap)
        if n < 0:
            _lib.check(-n, "tf_region_stream_idle")
        return list(buf[:n])

    def members(self, team: int) -> list[int]:
        size = self.lib.tf_region_team_size(self.handle, team)
        buf = (C.c_int64 * max(size, 1))()
        self.lib.tf_region_team_members(self.handle, team, buf, size)
        return list(buf[:size])

    def team_parent(self, team: int) -> int:
        return self.lib.tf_region_team_parent(self.handle, team)

    def release(self, team: int) -> None:
        _lib.check(self.lib.tf_region_release_team(self.handle, team),
                   "tf_region_release_team")

    def stats(self) -> dict:
        tf, solo = C.c_int64(), C.c_int64()
        hist = (C.c_int64 * 129)()
        self.lib.tf_region_stats(self.handle, C.byref(tf), C.byref(solo), hist)
        return {"teams_formed": tf.value, "solo_fast_path": solo.value,
                "size_histogram": {k: hist[k] for k in range(129) if hist[k]}}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.tf_region_destroy(h)
            self.handle = None


@dataclass
class Team:
    executor: int
    parent: int
    ids: list
    reason: str


def form_teams(arrivals, max_team: int, executors: int = 1,
               parents: int | None = None, name: str = "reconstruct",
               busy=lambda executor: True) -> list[Team]:
    """Run the formation core over an arrival sequence and return the closed
    teams in closure order.  `busy(executor)` answers the starvation query;
    the default models a saturated device.  Teams still forming when the
    arrivals end close as their streams drain (in executor order)."""
    arrivals = [int(a) for a in arrivals]
    if parents is None:
        parents = default_parents(len(arrivals), max_team)
    core = FormationCore(name, max_team, parents, executors)
    teams = []

    def take(team_id, reason):
        teams.append(Team(core.parent_executor(core.team_parent(team_id)),
                          core.team_parent(team_id), core.members(team_id),
                          reason))
        core.release(team_id)

    for tag in arrivals:
        res = core.enter(tag, busy)
        if res.closed:
            take(res.team, _CLOSE[res.closed])
    for e in range(executors):
        for team_id in core.stream_idle(e):
            take(team_id, "drain")
    return teams


class TeamPlan:
    """One iteration's teams captured as a CUDA graph (tf_plan)."""

    def __init__(self, teams, pool, n, velocity, um, up, F, executors,
                 amax=None, flux_form=0, overlap=True, team_buffers=False,
                 geometry="tma"):
        """team_buffers: write each team's outputs into its lease of the
        iteration's packed team buffers (slot = flat slice index in closure
        order, `self.order`) instead of per-sub-grid slots.
        geometry: "tma" — one CTA per slice, the stencil box staged by TMA
        (the product kernel); "reference" — the reference's blocks_for
        launch geometry, ceil((n+2)^3/128) CTAs of 128 threads per slice
        (the strategy-1 baseline)."""
        if geometry not in ("tma", "reference"):
            raise ValidationError(f"unknown geometry {geometry!r}")
        self.lib = _lib.load()
        ids = np.concatenate([np.asarray(t.ids, dtype=np.int32)
                              for t in teams]) if teams else \
            np.zeros(0, np.int32)
        offs = np.zeros(len(teams) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(t.ids) for t in teams])
        exe = np.asarray([t.executor for t in teams], dtype=np.int32)
        self._keep = (ids, offs, exe, pool, um, up, F, amax)
        # per-sub-grid slots, or (team buffers) one slot per flat slice
        S = _check_recon_args(pool, n, um, up, F, amax,
                              slots=int(ids.size) if team_buffers else None)
        if ids.size and (ids.min() < 0 or ids.max() >= S):
            raise ValidationError("team id outside the pool")
        ax, ay, az = (float(v) for v in velocity)
        h = C.c_void_p()
        rc = self.lib.tf_plan_capture_recon_flux(
            ids.ctypes.data_as(C.POINTER(C.c_int32)),
            offs.ctypes.data_as(C.POINTER(C.c_int64)),
            exe.ctypes.data_as(C.POINTER(C.c_int32)), len(teams), executors,
            pool.data_ptr(), S, n, ax, ay, az, um.data_ptr(), up.data_ptr(),
            F.data_ptr(), None if amax is None else amax.data_ptr(),
            int(flux_form),
            (_lib.TF_LAUNCH_OVERLAP_PREV if overlap else 0)
            | (_lib.TF_PLAN_TEAM_BUFFERS if team_buffers else 0)
            | (_lib.TF_PLAN_REFGEO if geometry == "reference" else 0),
            C.byref(h))
        self.order = ids      # flat slice index -> sub-grid id
        _lib.check(rc, "tf_plan_capture_recon_flux")
        self.handle = h
        self.kernels = self.lib.tf_plan_kernels(h)
        self.slices = int(ids.size)

    def launch(self, stream=None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream()
        _lib.check(self.lib.tf_plan_launch(self.handle, s.cuda_stream),
                   "tf_plan_launch")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.tf_plan_destroy(h)
            self.handle = None


class RealtimeExecutor:
    """tf_executor: real-time strategy-3 formation over `executors` streams."""

    def __init__(self, name: str, max_team: int, executors: int,
                 parents: int, overlap: bool = False):
        self.core = FormationCore(name, max_team, parents, executors)
        self.lib = self.core.lib
        h = C.c_void_p()
        _lib.check(self.lib.tf_executor_create(self.core.handle, executors,
                                               C.byref(h)),
                   "tf_executor_create")
        self.handle = h
        _lib.check(self.lib.tf_executor_set_flags(
            h, _lib.TF_LAUNCH_OVERLAP_PREV if overlap else 0),
            "tf_executor_set_flags")
        self.executors = executors

    def run(self, pool, n, velocity, ids, um, up, F, amax=None,
            flux_form=0, join_stream=None) -> int:
        """Submit the arrivals; returns the number of team launches.  The
        current torch stream (or join_stream) is made to wait for them."""
        arr = np.ascontiguousarray(np.asarray(ids, dtype=np.int32))
        S = _check_recon_args(pool, n, um, up, F, amax)
        if arr.size and (arr.min() < 0 or arr.max() >= S):
            raise ValidationError("arrival id outside the pool")
        launches = C.c_int64()
        ax, ay, az = (float(v) for v in velocity)
        s = join_stream if join_stream is not None else \
            torch.cuda.current_stream()
        _lib.check(self.lib.tf_executor_fork(self.handle, s.cuda_stream),
                   "tf_executor_fork")
        rc = self.lib.tf_executor_run_recon_flux(
            self.handle, pool.data_ptr(), S,
            arr.ctypes.data_as(C.POINTER(C.c_int32)), arr.size, n, ax, ay, az,
            um.data_ptr(), up.data_ptr(), F.data_ptr(),
            None if amax is None else amax.data_ptr(), int(flux_form),
            C.byref(launches))
        _lib.check(rc, "tf_executor_run_recon_flux")
        _lib.check(self.lib.tf_executor_join(self.handle, s.cuda_stream),
                   "tf_executor_join")
        return launches.value

    def stats(self) -> dict:
        return self.core.stats()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.tf_executor_destroy(h)
            self.handle = None


class QueueExecutor:
    """Strategy 3 with a device-side work queue (tf_qexec): the formation
    core's closed teams are PUBLISHED to a resident consumer grid instead of
    launched — a team closure costs a few host stores; the starvation
    signal is 'every published slice completed'."""

    def __init__(self, name: str, max_team: int, parents: int, n: int = 8,
                 early_loads: bool = False, sorted_dispatch: bool = False):
        """early_loads: a run's first stencil boxes may load while the
        previous kernel on the stream still runs — valid only when that
        kernel does not produce the pool (TF_LAUNCH_OVERLAP_PREV).
        sorted_dispatch: the device works through each mirrored batch of
        published slices in sub-grid id order (TF_QUEUE_SORTED)."""
        self.core = FormationCore(name, max_team, parents, 1)
        self.lib = self.core.lib
        h = C.c_void_p()
        _lib.check(self.lib.tf_qexec_create(self.core.handle, n, C.byref(h)),
                   "tf_qexec_create")
        self.handle = h
        qflags = (_lib.TF_LAUNCH_OVERLAP_PREV if early_loads else 0) | \
            (_lib.TF_QUEUE_SORTED if sorted_dispatch else 0)
        if qflags:
            _lib.check(self.lib.tf_qexec_set_flags(h, qflags),
                       "tf_qexec_set_flags")
        self.n = n
        self.runs = 0
        self._vcache = {}
        self._teams = C.c_int64()
        self._teams_ref = C.addressof(self._teams)

    def _validated(self, pool, um, up, F, amax):
        """Pointers of validated arguments.  A step loop passes the same
        tensors run after run: they are checked once (shape, dtype, device,
        capacity) and then recognised by identity and data pointer — the
        ids themselves are range-checked in C on every run."""
        key = (id(pool), id(um), id(up), id(F), id(amax))
        ptrs = (pool.data_ptr(), um.data_ptr(), up.data_ptr(), F.data_ptr(),
                None if amax is None else amax.data_ptr())
        hit = self._vcache.get(key)
        if hit is not None and hit[0] == ptrs and all(
                r() is t for r, t in zip(hit[2], (pool, um, up, F))):
            return ptrs, hit[1]
        S = _check_recon_args(pool, self.n, um, up, F, amax)
        if len(self._vcache) >= 8:
            self._vcache.pop(next(iter(self._vcache)))
        self._vcache[key] = (ptrs, S, tuple(
            weakref.ref(t) for t in (pool, um, up, F)))
        return ptrs, S

    def run(self, pool, velocity, ids, um, up, F, amax=None, flux_form=0,
            stream=None) -> int:
        """Publish the arrivals; returns teams published.  The consumer runs
        on `stream` (default: the current stream)."""
        if isinstance(ids, np.ndarray) and ids.dtype == np.int32 and \
                ids.flags.c_contiguous:
            arr = ids
        else:
            arr = np.ascontiguousarray(np.asarray(ids, dtype=np.int32))
        (pp, pum, pup, pF, pam), S = self._validated(pool, um, up, F, amax)
        s = stream if stream is not None else torch.cuda.current_stream()
        ax, ay, az = (float(v) for v in velocity)
        self._keep = arr
        rc = self.lib.tf_qexec_run_recon_flux(
            self.handle, pp, S, arr.ctypes.data, arr.size, ax, ay, az, pum,
            pup, pF, pam, int(flux_form), s.cuda_stream, self._teams_ref)
        if rc == _lib.TF_E_INVALID:
            raise ValidationError("tf_qexec_run_recon_flux: an arrival id "
                                  "lies outside the pool")
        _lib.check(rc, "tf_qexec_run_recon_flux")
        self.runs += 1
        return self._teams.value

    def bind(self, pool, velocity, ids, um, up, F, amax=None, flux_form=0,
             stream=None):
        """`run` with its arguments checked and converted once: returns a
        callable that publishes the same arrivals of the same pool into the
        same outputs on the same stream at each call (the ids array is kept
        and must not change).  For a step loop: a call costs one C call and
        none of `run`'s per-call argument handling."""
        arr = np.ascontiguousarray(np.asarray(ids, dtype=np.int32)).copy()
        (pp, pum, pup, pF, pam), S = self._validated(pool, um, up, F, amax)
        if arr.size and (int(arr.min()) < 0 or int(arr.max()) >= S):
            raise ValidationError("arrival id outside the pool")
        s = stream if stream is not None else torch.cuda.current_stream()
        keep = (pool, um, up, F, amax, arr)  # alive while the call lives
        fn = self.lib.tf_qexec_run_recon_flux
        args = (self.handle, C.c_void_p(pp), C.c_int64(S),
                C.c_void_p(arr.ctypes.data), C.c_int64(arr.size),
                *(C.c_double(float(v)) for v in velocity), C.c_void_p(pum),
                C.c_void_p(pup), C.c_void_p(pF), C.c_void_p(pam),
                C.c_int32(int(flux_form)), C.c_void_p(s.cuda_stream),
                C.c_void_p(self._teams_ref))

        def call() -> int:
            rc = fn(*args)
            if rc:
                _lib.check(rc, "tf_qexec_run_recon_flux")
            self.runs += 1
            return self._teams.value
        call.keep = keep
        return call

    def completed(self) -> int:
        return self.lib.tf_qexec_completed(self.handle)

    def host_times(self) -> dict:
        """Mean host microseconds per run: waiting for a queue slot's
        previous run, the launch, the formation + publish loop."""
        out = (C.c_int64 * 4)()
        _lib.check(self.lib.tf_qexec_host_times(self.handle, out),
                   "tf_qexec_host_times")
        runs = max(1, out[0])
        return {"runs": out[0], "wait_us": out[1] / runs / 1e3,
                "launch_us": out[2] / runs / 1e3,
                "publish_us": out[3] / runs / 1e3}

    def wait(self) -> None:
        """Block until every run has drained; raises TaskfuseCudaError if a
        consumer grid timed out with slices unprocessed."""
        _lib.check(self.lib.tf_qexec_wait(self.handle), "tf_qexec_wait")

    def stats(self) -> dict:
        return self.core.stats()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.tf_qexec_destroy(h)
            self.handle = None


class DeviceLaunchExecutor:
    """Strategy 3 with DEVICE-side team launches (tf_dlexec): the formation
    core's closed teams are published to a one-CTA launcher kernel that
    launches each team as its own T-CTA grid of the fused kernel from the
    GPU (dynamic parallelism) — one aggregated kernel per team as in the
    reference (aggregator.py:157-165), with no host launch per team."""

    def __init__(self, name: str, max_team: int, parents: int, n: int = 8):
        if n != 8:
            raise ValidationError("the device-launch executor supports n = 8")
        self.core = FormationCore(name, max_team, parents, 1)
        self.lib = self.core.lib
        h = C.c_void_p()
        _lib.check(self.lib.tf_dlexec_create(self.core.handle, n, C.byref(h)),
                   "tf_dlexec_create")
        self.handle = h
        self.n = n
        self.runs = 0

    def run(self, pool, velocity, ids, um, up, F, amax=None, flux_form=0,
            stream=None) -> int:
        """Publish the arrivals; returns teams published.  The launcher and
        its team grids complete on `stream` (default: the current one)."""
        arr = np.ascontiguousarray(np.asarray(ids, dtype=np.int32))
        S = _check_recon_args(pool, self.n, um, up, F, amax)
        if arr.size and (arr.min() < 0 or arr.max() >= S):
            raise ValidationError("arrival id outside the pool")
        s = stream if stream is not None else torch.cuda.current_stream()
        teams = C.c_int64()
        ax, ay, az = (float(v) for v in velocity)
        self._keep = arr
        _lib.check(self.lib.tf_dlexec_run_recon_flux(
            self.handle, pool.data_ptr(), S,
            arr.ctypes.data_as(C.POINTER(C.c_int32)), arr.size, ax, ay, az,
            um.data_ptr(), up.data_ptr(), F.data_ptr(),
            None if amax is None else amax.data_ptr(), int(flux_form),
            s.cuda_stream, C.byref(teams)), "tf_dlexec_run_recon_flux")
        self.runs += 1
        return teams.value

    def wait(self) -> None:
        _lib.check(self.lib.tf_dlexec_wait(self.handle), "tf_dlexec_wait")

    def stats(self) -> dict:
        return self.core.stats()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.tf_dlexec_destroy(h)
            self.handle = None


_COPY_STREAMS: dict = {}


def copy_split(dst: torch.Tensor, src: torch.Tensor, parts: int = 4) -> None:
    """Host<->device copy (one side pinned host memory) split along dim 0
    over `parts` side streams, ordered after the current stream's work and
    before what follows on it.  One copy engine moved config 2's 16.8 MB
    field at 17-49 GB/s from box to box; split over streams it ran at
    49 GB/s (2 or 4 streams) on a healthy host link and 25 GB/s (4) vs
    17 GB/s (1) on a slow one (scripts/probe_h2d_streams.py)."""
    dev = dst.device if dst.is_cuda else src.device
    cur = torch.cuda.current_stream(dev)
    key = (dev.index, parts)
    side = _COPY_STREAMS.get(key)
    if side is None:
        side = _COPY_STREAMS[key] = [torch.cuda.Stream(device=dev)
                                     for _ in range(parts)]
    rows = dst.shape[0]
    step = (rows + parts - 1) // parts
    for i, st in enumerate(side):
        lo, hi = i * step, min(rows, (i + 1) * step)
        if lo >= hi:
            continue
        st.wait_stream(cur)
        with torch.cuda.stream(st):
            dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
        cur.wait_stream(st)



class AggregatedIteration:
    """One device-resident hydro iteration with strategy-3 team launches:
    ghost fill -> reconstruct+flux (captured team plan) -> update -> swap.

    `run_host(field_in, field_out)` is the end-to-end call with HOST
    buffers: the global field (grid^3, the reference's `assemble` layout)
    goes host->device, one iteration runs, the updated field comes back —
    exactly what `reference_step(u, iterations=1)` computes on the CPU
    (reference.py:42-48), bit for bit.
    """

    def __init__(self, grid_n: int, n: int, velocity=(1.0, 1.0, 1.0),
                 max_team: int = 128, executors: int = 4, device=None,
                 overlap: bool = True, formation: str = "plan"):
        """formation: "plan" — the teams a saturated device forms, captured
        once as a CUDA graph (one kernel per team); "queue" — formed on the
        fly every iteration by the formation core and published to the
        device queue (QueueExecutor; one consumer grid per iteration)."""
        from . import ops
        if formation not in ("plan", "queue"):
            raise ValidationError(f"formation must be 'plan' or 'queue', "
                                  f"got {formation!r}")
        from .hydro.scenario import dt_over_dx
        self.ops = ops
        dev = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.n, self.grid_n = n, grid_n
        self.m = grid_n // n
        S = self.m ** 3
        self.S = S
        self.velocity = tuple(float(v) for v in velocity)
        self.dt_dx = dt_over_dx(velocity)
        e, c = n + 6, n + 2
        f64 = dict(dtype=torch.float64, device=dev)
        self.pools = [torch.full((S, e, e, e), float("nan"), **f64)
                      for _ in range(2)]
        self.um = torch.empty((S, 3, c, c, c), **f64)
        self.up = torch.empty_like(self.um)
        self.F = torch.empty_like(self.um)
        self.amax = torch.empty(S, **f64)
        self.field_dev = torch.empty((grid_n,) * 3, **f64)
        self.formation = formation
        self.teams = form_teams(range(S), max_team, executors)
        if formation == "plan":
            # one captured plan per pool (the pools swap every iteration)
            self.plans = [TeamPlan(self.teams, p, n, self.velocity, self.um,
                                   self.up, self.F, executors,
                                   amax=self.amax, overlap=overlap)
                          for p in self.pools]
        else:
            # the ghost fill before each run produces its pool: the queue's
            # boxes load after it (no early loads)
            self.queue = QueueExecutor("reconstruct", max_team,
                                       default_parents(S, max_team), n,
                                       sorted_dispatch=True)
            self.arrivals = np.arange(S, dtype=np.int32)
        self.cur = 0

    def _recon_flux(self) -> None:
        if self.formation == "plan":
            self.plans[self.cur].launch()
        else:
            self.queue.run(self.pool, self.velocity, self.arrivals, self.um,
                           self.up, self.F, amax=self.amax)

    @property
    def pool(self):
        return self.pools[self.cur]

    def load(self, field_dev) -> None:
        self.ops.field_to_pool(field_dev, self.n, self.pool)

    def step(self) -> None:
        """One iteration on the device-resident current pool."""
        ops, n = self.ops, self.n
        cur, nxt = self.pools[self.cur], self.pools[1 - self.cur]
        ops.ghost_fill(cur, n, self.m)
        self._recon_flux()
        ops.update(cur, n, self.F, self.dt_dx, nxt)
        self.cur = 1 - self.cur

    def store(self, field_dev) -> None:
        self.ops.pool_to_field(self.pool, self.n, field_dev)

    def run_host(self, field_in, field_out, iterations: int = 1) -> None:
        """Host (pinned) field in -> `iterations` iterations -> host out."""
        copy_split(self.field_dev, field_in)
        self.load(self.field_dev)
        for _ in range(iterations):
            self.step()
        self.store(self.field_dev)
        copy_split(field_out, self.field_dev)

    def recon_flux_host(self, field_in, amax_out) -> None:
        """End-to-end aggregated reconstruct+flux from a HOST field: the
        pinned (grid^3) field goes host->device, is scattered into the
        current sub-grid pool and ghost-filled (make_state +
        exchange_ghosts, scenario.py:83-142), the region's captured team
        plan runs (reconstruct_body + flux_body per slice, um / up / F
        materialised in HBM), and the per-sub-grid max signal speed — the
        reduce stage's result (kernels.py:96-97) — comes back to the pinned
        `amax_out` (S doubles).  Stream-ordered on the current stream."""
        if not (field_in.is_pinned() and amax_out.is_pinned()):
            raise ValidationError("recon_flux_host needs pinned host buffers")
        if amax_out.numel() < self.S:
            raise ValidationError(f"amax_out must hold {self.S} values")
        copy_split(self.field_dev, field_in.view(self.field_dev.shape))
        self.load(self.field_dev)
        self.ops.ghost_fill(self.pool, self.n, self.m)
        self._recon_flux()
        amax_out[:self.S].copy_(self.amax, non_blocking=True)

    @property
    def recon_flux_launches(self) -> int:
        """Kernels per recon_flux_host call: scatter, ghost fill, teams (or
        the one consumer grid)."""
        return 2 + (len(self.teams) if self.formation == "plan" else 1)

    @property
    def launches_per_step(self) -> int:
        return 2 + (len(self.teams) if self.formation == "plan" else 1)


class ReconFluxHostPipeline:
    """`AggregatedIteration.recon_flux_host` with the upload overlapped,
    captured once as a CUDA graph for FIXED pinned buffers.

    The host field moves in x-chunks of sub-grid layers on a copy stream,
    the LAST layer first (it is layer 0's periodic neighbour), then layers
    0, 1, ...; each chunk is scattered into the pool as soon as it lands,
    and every layer whose two neighbours have landed too is ghost-filled
    (exchange_ghosts reads the neighbours' OWNED cells) and run through its
    own captured team plans (teams formed over those arrivals with the
    iteration's cap) at once — so after the last chunk lands only two
    layers remain.  Their per-sub-grid max signal speeds return to
    `amax_out` group by group on a second copy stream.  Pure function of
    `field_in`: every replay rewrites the whole current pool."""

    def __init__(self, it: "AggregatedIteration", field_in, amax_out,
                 layers=(1, 4, 4, 4, 2, 1), executors: int = 2,
                 copy_streams: int = 2):
        from . import ops
        if not (field_in.is_pinned() and amax_out.is_pinned()):
            raise ValidationError("the pipeline needs pinned host buffers")
        m, n = it.m, it.n
        layers = [int(k) for k in layers]
        if sum(layers) != m:    # scale the taper to the lattice
            base = max(1, m // len(layers))
            layers = [base] * (m // base)
            layers[-1] += m - sum(layers)
        order = [m - 1] + list(range(m - 1)) if m > 1 else [0]
        chunks, pos = [], 0
        for k in layers:
            chunks.append(order[pos:pos + k])
            pos += k
        # compute groups: after chunk c lands, the layers whose neighbours
        # (periodic) have all landed and that have not run yet
        landed, done, groups = set(), set(), []
        for ch in chunks:
            landed.update(ch)
            ready = [l for l in range(m) if l not in done and
                     all((l + d) % m in landed for d in (-1, 0, 1))]
            done.update(ready)
            groups.append(ready)
        nch = len(chunks)
        self.it, self.bufs = it, (field_in, amax_out)
        dev = it.pool.device
        mm = m * m

        def runs(ls):
            """maximal runs of consecutive layers: (first, count)"""
            out = []
            for l in sorted(ls):
                if out and out[-1][0] + out[-1][1] == l:
                    out[-1][1] += 1
                else:
                    out.append([l, 1])
            return out
        self.group_runs = [runs(g) for g in groups]
        self.chunk_runs = [runs(c) for c in chunks]
        self.ids = [torch.cat([torch.arange(a * mm, (a + k) * mm,
                                            dtype=torch.int32, device=dev)
                               for a, k in r]) if r else None
                    for r in self.group_runs]
        cap = max(len(t.ids) for t in it.teams)
        # each group's arrivals formed into teams with the iteration's cap;
        # a team is one launch with its ids in the kernel parameters
        self.teams = [[np.asarray(t.ids, dtype=np.int32)
                       for t in form_teams(
                           [i for a, k in r
                            for i in range(a * mm, (a + k) * mm)], cap)]
                      for r in self.group_runs]
        lib = _lib.load()
        ax, ay, az = it.velocity
        self.launches = 0
        # each chunk's upload may be split over two copy streams (two copy
        # engines: one alone ran at 17-49 GB/s from box to box), chunks in
        # order on both — rotating whole chunks over the streams instead let
        # every chunk land at about the same time, which undid the overlap
        ups = [torch.cuda.Stream(device=dev)
               for _ in range(max(1, min(2, copy_streams)))]
        down = torch.cuda.Stream(device=dev)
        comp_side = torch.cuda.Stream(device=dev)
        fin = field_in.view(it.grid_n, it.grid_n, it.grid_n)
        dev_f, pool = it.field_dev, it.pool

        def group_compute(g):
            ops.ghost_fill(pool, n, m, ids=self.ids[g])
            st = torch.cuda.current_stream().cuda_stream
            for k, ids in enumerate(self.teams[g]):
                # teams after the first overlap their predecessor (PDL):
                # same region, independent slices
                _lib.check(lib.tf_recon_flux_team_ex_f64(
                    pool.data_ptr(), it.S,
                    ids.ctypes.data_as(C.POINTER(C.c_int32)), ids.size, n,
                    ax, ay, az, it.um.data_ptr(), it.up.data_ptr(),
                    it.F.data_ptr(), 1, it.amax.data_ptr(), 0,
                    _lib.TF_LAUNCH_OVERLAP_PREV if k else 0, st),
                    "tf_recon_flux_team_ex_f64")
            self.launches += 1 + len(self.teams[g])
            # this group's max signal speeds go home while the rest runs
            ev = torch.cuda.Event()
            ev.record()
            down.wait_event(ev)
            with torch.cuda.stream(down):
                for a, k in self.group_runs[g]:
                    amax_out[a * mm:(a + k) * mm].copy_(
                        it.amax[a * mm:(a + k) * mm], non_blocking=True)

        def run():
            self.launches = 0
            comp = torch.cuda.current_stream()
            evs = []
            for up in ups + [down]:
                up.wait_stream(comp)
            for c in range(nch):
                pair = []
                for a, k in self.chunk_runs[c]:
                    lo, hi = a * n, (a + k) * n
                    mid = (lo + hi) // 2 if len(ups) == 2 else hi
                    for up, (x0, x1) in zip(ups, ((lo, mid), (mid, hi))):
                        if x0 >= x1:
                            continue
                        with torch.cuda.stream(up):
                            dev_f[x0:x1].copy_(fin[x0:x1], non_blocking=True)
                            ev = torch.cuda.Event()
                            ev.record(up)
                            pair.append(ev)
                evs.append(pair)
            for c in range(nch):
                for ev in evs[c]:
                    comp.wait_event(ev)
                for a, k in self.chunk_runs[c]:
                    ops.field_to_pool_layers(dev_f, n, pool, a, k)
                    self.launches += 1
                if self.group_runs[c]:
                    group_compute(c)
            comp.wait_stream(down)

        run()                       # warm-up (also sizes the TMA maps)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        comp_side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(self.graph, stream=comp_side):
            run()
        torch.cuda.synchronize()
        self.chunks = nch

    def run(self) -> None:
        self.graph.replay()


def recon_flux_all(pool, n, velocity, um, up, F, amax=None, flux_form=0,
                   stream=None) -> None:
    """Aggregation limit: every slice of the pool in one launch."""
    from . import ops
    ops.recon_flux(pool, n, velocity, um, up, F, out_mode=1, amax=amax,
                   flux_form=flux_form, stream=stream)
