"""The native HydroSim engine (csrc/hydro_engine.cpp) behind the reference
API: `HydroSim(..., engine="native")` runs every iteration's per-sub-grid
tasks (step.py:83-123, five region visits each) in C++ under the same
formation and member rules as the Python task path (tf_region / tf_team),
on the executor pool's own CUDA streams, with real pinned/device staging
leases, one aggregated copy per team copy step and ONE batched kernel per
team launch.  The Python driver stays the caller (step.py:126-143)."""

from __future__ import annotations

import ctypes as C

from .. import _lib
from ..aggregator import RegionStats
from ..errors import OrderingViolationError, TaskfuseCudaError
from .kernels import KERNEL_ORDER


class NativeRegion:
    """Read-only view of one engine region (AggregationRegion.stats())."""

    def __init__(self, engine, k: int, name: str, max_team: int):
        self._engine = engine
        self.name = name
        self.max_team = max_team
        h = C.c_void_p()
        _lib.check(engine.lib.tf_hydro_region(engine.handle, k, C.byref(h)),
                   "tf_hydro_region")
        self.handle = h

    def stats(self) -> RegionStats:
        lib = self._engine.lib
        tf, solo = C.c_int64(), C.c_int64()
        hist = (C.c_int64 * 129)()
        lib.tf_region_stats(self.handle, C.byref(tf), C.byref(solo), hist)
        return RegionStats(
            name=self.name, max_team=self.max_team, teams_formed=tf.value,
            violations=int(lib.tf_region_violations(self.handle)),
            solo_fast_path=solo.value,
            size_histogram={k: hist[k] for k in range(129) if hist[k]})


class HydroEngine:
    COUNTERS = ("kernels", "copies", "bytes", "raw_device", "raw_pinned",
                "outstanding", "allocated", "polls")

    def __init__(self, state, scratch, executors, max_team: int, velocity,
                 dt_dx: float, device):
        self.lib = _lib.load()
        E = len(executors.executors)
        streams = (C.c_void_p * E)(*[
            device.stream(e.stream_id).cuda_stream
            for e in executors.executors])
        self._streams = streams
        ax, ay, az = (float(v) for v in velocity)
        h = C.c_void_p()
        _lib.check(self.lib.tf_hydro_create(
            state.n, state.per_axis, max_team, E, streams, ax, ay, az,
            float(dt_dx), scratch.w.data_ptr(), scratch.um.data_ptr(),
            scratch.up.data_ptr(), scratch.F.data_ptr(),
            scratch.reduce_out.data_ptr(), C.byref(h)), "tf_hydro_create")
        self.handle = h
        self._keep = (scratch,)
        self.regions = {k: NativeRegion(self, i, k, max_team)
                        for i, k in enumerate(KERNEL_ORDER)}

    def presize(self) -> None:
        _lib.check(self.lib.tf_hydro_presize(self.handle), "tf_hydro_presize")

    def iteration(self, u_pool, u_next_pool, stream) -> None:
        rc = self.lib.tf_hydro_iteration(self.handle, u_pool.data_ptr(),
                                         u_next_pool.data_ptr(),
                                         stream.cuda_stream)
        if rc == _lib.TF_E_ORDERING:
            for r in self.regions.values():
                err = self.lib.tf_region_error(r.handle).decode()
                if err:
                    exp, got = err.split("\n", 1)
                    raise OrderingViolationError(r.name, -1, exp, got)
            raise TaskfuseCudaError("native HydroSim engine deadlocked: "
                                    "parked tasks and no device work")
        _lib.check(rc, "tf_hydro_iteration")

    def counters(self) -> dict:
        buf = (C.c_int64 * 8)()
        _lib.check(self.lib.tf_hydro_counters(self.handle, buf),
                   "tf_hydro_counters")
        return dict(zip(self.COUNTERS, buf))

    def host_times(self) -> dict:
        """Cumulative host ns: issuing device ops, idle polling, iterations."""
        buf = (C.c_int64 * 3)()
        _lib.check(self.lib.tf_hydro_host_times(self.handle, buf),
                   "tf_hydro_host_times")
        return dict(zip(("issue_ns", "idle_poll_ns", "iteration_ns"), buf))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            self.lib.tf_hydro_destroy(h)
            self.handle = None
