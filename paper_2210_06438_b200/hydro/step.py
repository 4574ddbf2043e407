"""Task bodies and the driver loop — taskfuse/hydro/step.py on a B200.

Same structure as the reference (step.py:38-143): one task per sub-grid per
iteration, five region visits per task (prep, reconstruct, flux, reduce,
update), each visit = enter -> slice_alloc x4 -> h2d -> slice_launch -> d2h
-> await -> leave.  Differences, all B200-first:

* every visit's slice_launch names a batched sm_100a kernel; the LAST member
  of a team issues ONE launch for the whole team over the members' sub-grid
  ids (the kernel registry of each region), writing the per-sub-grid
  ScratchPool (the reference's HydroSim.scratch);
* the field lives on the device (HydroState pools); the staging allocs and
  copies keep the reference's transfer structure (ext^3 up, n^3 down per
  slice, one aggregated copy per team) with real pinned/device buffers;
* ghost exchange for all sub-grids is one device launch at the start of an
  iteration (each task's exchange reads only current owned cells, which no
  task writes during the iteration — scenario.py:127-129 — so doing them
  together is equivalent);
* there is no CPU path: executors == 0 raises UsageError;
* engine="native" (the default on a real CudaDevice) runs the iteration's
  tasks in C++ (hydro/engine.py) under the same formation and member rules,
  so arrivals keep up with the device and teams form; engine="python" runs
  each task as a Python generator through the mirrored AggregationRegion
  API (the same path user task bodies take).
"""

from __future__ import annotations

from fractions import Fraction
from functools import partial

import torch

from .. import ops
from ..aggregator import AggregationRegion
from ..bufferpool import BufferPool
from ..errors import UsageError
from ..executorpool import ExecutorPool
from ..sched import Scheduler, await_all, charge
from .kernels import KERNEL_ORDER, ScratchPool, blocks_for, check_reduce
from .scenario import (ITERATIONS_PER_STEP, VELOCITY, HydroState, dt_over_dx,
                       exchange_ghosts, ghost_cells)

ITEM_BYTES = 8


class _IdRing:
    """Team id lists for the stage kernels in a pinned host ring, read by
    the kernels zero-copy (no per-launch tensor, pin or copy).  Reuse is
    fenced per half ring: crossing into a half waits for events recorded on
    every executor stream when that half was last left, i.e. for launches
    issued a half ring ago (in practice long finished)."""

    def __init__(self, streams, size: int = 1 << 16):
        self.buf = torch.empty(size, dtype=torch.int32).pin_memory()
        self.np = self.buf.numpy()
        self.size, self.half = size, size // 2
        self.pos = 0
        self.cur = 0                  # the half being written
        self.streams = streams
        self.fence = [None, None]     # per half: events from when we left it

    def put(self, args) -> torch.Tensor:
        T = len(args)
        if self.pos + T > self.size:
            self._cross(0)
            self.pos = 0
        elif self.cur == 0 and self.pos + T > self.half:
            self._cross(1)
            self.pos = self.half
        a = self.pos
        self.np[a:a + T] = args
        self.pos = a + T
        return self.buf[a:a + T]

    def _cross(self, into: int) -> None:
        self.cur = into
        for ev in self.fence[into] or ():
            ev.synchronize()
        left = []
        for st in self.streams:
            ev = torch.cuda.Event()
            ev.record(st)
            left.append(ev)
        self.fence[1 - into] = left


class HydroSim:
    def __init__(self, sched: Scheduler, state: HydroState,
                 executors: ExecutorPool, buffers: BufferPool | None = None,
                 work_factors: dict | None = None, max_team: int = 1,
                 velocity=VELOCITY, engine: str = "auto"):
        if executors.cpu_only:
            raise UsageError("HydroSim on the B200 needs >= 1 executor; "
                             "there is no CPU path")
        self.sched = sched
        self.state = state
        self.executors = executors
        self.velocity = tuple(float(v) for v in velocity)
        self.dt_dx = dt_over_dx(velocity)
        self.work_factors = work_factors or {k: Fraction(1)
                                             for k in KERNEL_ORDER}
        S = len(state.blocks)
        self.scratch_pool = ScratchPool(S, state.n, state.device)
        self.max_team = max_team
        if engine == "auto":
            # the native engine needs real streams; a test double (or custom
            # work factors, which only the Python path's launch specs carry)
            # keeps the Python task path
            from ..device import CudaDevice
            engine = "native" if isinstance(executors.device, CudaDevice) \
                and work_factors is None else "python"
        if engine not in ("native", "python"):
            raise UsageError(f"unknown engine {engine!r}")
        self.native = None
        if engine == "native":
            from .engine import HydroEngine
            self.buffers = buffers
            self.native = HydroEngine(state, self.scratch_pool, executors,
                                      max_team, self.velocity, self.dt_dx,
                                      executors.device)
            self.regions = self.native.regions
            self._seen = self.native.counters()
            return
        self.buffers = buffers or BufferPool(executors.device)
        parents = max(1, S // max_team)          # step.py:59-61
        self.regions = {
            k: AggregationRegion(sched, executors, self.buffers, name=k,
                                 max_team=max_team, parent_count=parents)
            for k in KERNEL_ORDER}
        for k, region in self.regions.items():
            region.register_kernel(k, partial(self._launch, k))
        dev = executors.device
        self._ids_ring = _IdRing([dev.stream(e.stream_id)
                                  for e in executors.executors])

    @property
    def scratch(self):
        """Reference-style {block: scratch dict} view."""
        return {b: self.scratch_pool.view(self.state.block_id(b))
                for b in self.state.blocks}

    def native_iteration(self) -> None:
        """Every sub-grid's task for one iteration in the native engine;
        its device work is folded into the CudaDevice counters."""
        st = self.state
        self.native.iteration(st.u_pool, st.u_next_pool,
                              torch.cuda.current_stream())
        now = self.native.counters()
        dev = self.executors.device
        dev.kernels_enqueued += now["kernels"] - self._seen["kernels"]
        dev.copies_enqueued += now["copies"] - self._seen["copies"]
        dev.bytes_copied += now["bytes"] - self._seen["bytes"]
        dev.raw_allocations["device"] += (now["raw_device"]
                                          - self._seen["raw_device"])
        dev.raw_allocations["pinned_host"] += (now["raw_pinned"]
                                               - self._seen["raw_pinned"])
        self._seen = now

    def presize(self) -> None:
        """bench.py:142-153 for the native engine's staging pool."""
        if self.native is not None:
            self.native.presize()
            self.native_iteration_counters_only()

    def native_iteration_counters_only(self) -> None:
        now = self.native.counters()
        dev = self.executors.device
        dev.raw_allocations["device"] += (now["raw_device"]
                                          - self._seen["raw_device"])
        dev.raw_allocations["pinned_host"] += (now["raw_pinned"]
                                               - self._seen["raw_pinned"])
        self._seen = now

    def _ids(self, args) -> torch.Tensor:
        return self._ids_ring.put(args)

    def _launch(self, kernel: str, stream, args) -> None:
        """One batched launch for a whole team (slice order = args order)."""
        st, sp, n = self.state, self.scratch_pool, self.state.n
        ids = self._ids(args)
        if kernel == "prep":
            ops.prep(st.u_pool, n, sp.w, ids=ids, stream=stream)
        elif kernel == "reconstruct":
            ops.reconstruct(sp.w, n, sp.um, sp.up, ids=ids, stream=stream)
        elif kernel == "flux":
            ops.flux(n, self.velocity, sp.um, sp.up, sp.F, ids=ids,
                     stream=stream)
        elif kernel == "reduce":
            ops.reduce(self.velocity, sp.reduce_out, ids=ids, stream=stream)
        else:
            ops.update(st.u_pool, n, sp.F, self.dt_dx, st.u_next_pool,
                       ids=ids, stream=stream)

    def task_iteration(self, block):
        """Task body: one sub-grid through one iteration (step.py:83-123)."""
        state, sched, n = self.state, self.sched, self.state.n
        g = state.block_id(block)
        yield charge(sched.cost("ghost_per_cell", 25) * ghost_cells(n))
        ext3, n3 = state.ext ** 3, n ** 3
        for kernel in KERNEL_ORDER:
            member = yield self.regions[kernel].enter()
            member.slice_alloc("pinned_host", "f8", ext3)
            member.slice_alloc("device", "f8", ext3)
            member.slice_alloc("pinned_host", "f8", n3)
            member.slice_alloc("device", "f8", n3)
            member.slice_copy("h2d", ext3 * ITEM_BYTES)
            member.slice_launch(kernel, blocks_for(kernel, n),
                                self.work_factors[kernel], slice_args=g)
            landed = member.slice_copy("d2h", n3 * ITEM_BYTES)
            yield await_all(landed)
            member.leave()


def driver(sim: HydroSim, steps: int, step_hook=None):
    """Root task body (step.py:126-143)."""
    sched, state = sim.sched, sim.state
    dt = sim.dt_dx / state.grid_n
    for _ in range(steps):
        for _ in range(ITERATIONS_PER_STEP):
            exchange_ghosts(state)
            if sim.native is not None:
                sim.native_iteration()
                yield charge(0)
            else:
                torch.cuda.current_stream().synchronize()
                tokens = [sched.spawn(partial(sim.task_iteration, b),
                                      label=f"hydro{b}")[1]
                          for b in state.blocks]
                yield await_all(*tokens)
            check_reduce(sim.scratch_pool, sim.velocity)
            state.swap()
            state.time += dt
        state.steps_taken += 1
        if step_hook is not None:
            step_hook(state.steps_taken)
