"""Timed CPU baseline — TEST/BENCH INFRASTRUCTURE ONLY.

Times the reference's own per-sub-grid task bodies, restated in
oracle/hydro_oracle.py, exactly as a HydroSim task runs them on the CPU
path (reference hydro/step.py:93-97), on the host cores: a multiprocessing
*spawn* pool, each worker holding private inputs (
fork-shared inputs did not scale).  Step time = the slowest worker's time
for its share of the sub-grids.

bodies="recon_flux": prep_body + reconstruct_body + flux_body + reduce_body
  (kernels.py:69-97) on ghost-filled sub-grids — the recon+flux metric.
bodies="iteration": the whole CPU task iteration — exchange_ghosts
  (scenario.py:124-142) then prep, reconstruct, flux, reduce, update
  (kernels.py:69-111) — the config-5 full-iteration metric.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

_STATE = {}


def _init(field_name, grid, n, velocity, ids, bodies):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import hydro_oracle as HO
    field = {"sod": HO.sod_field, "blast": HO.initial_field,
             "stress": HO.stress_field}[field_name](grid)
    pool = HO.make_pool(field, n)
    if bodies == "recon_flux":
        HO.exchange_ghosts_pool(pool, n, grid // n, ids=ids)
    _STATE.update(pool=pool, nxt=pool.copy(), n=n, m=grid // n,
                  velocity=tuple(velocity), ids=list(ids), bodies=bodies,
                  scratch=HO.make_scratch(n), HO=HO,
                  dt_dx=HO.dt_over_dx(velocity))


def _pass(_):
    HO = _STATE["HO"]
    pool, n, vel, sc = (_STATE["pool"], _STATE["n"], _STATE["velocity"],
                        _STATE["scratch"])
    t0 = time.perf_counter()
    if _STATE["bodies"] == "recon_flux":
        for g in _STATE["ids"]:
            HO.prep_body(pool[g], sc)
            HO.reconstruct_body(sc, n)
            HO.flux_body(sc, n, vel)
            HO.reduce_body(sc, vel)
    else:
        m, nxt, dt_dx = _STATE["m"], _STATE["nxt"], _STATE["dt_dx"]
        for g in _STATE["ids"]:
            HO.exchange_ghosts_pool(pool, n, m, ids=(g,))
            HO.prep_body(pool[g], sc)
            HO.reconstruct_body(sc, n)
            HO.flux_body(sc, n, vel)
            HO.reduce_body(sc, vel)
            HO.update_body(pool[g], nxt[g], sc, n, dt_dx)
    return time.perf_counter() - t0


def _worker_main(conn, field_name, grid, n, velocity, ids, bodies):
    _init(field_name, grid, n, velocity, ids, bodies)
    conn.send("ready")
    while True:
        msg = conn.recv()
        if msg is None:
            break
        conn.send(_pass(None))


class CpuBaseline:
    """Persistent spawn workers, each owning a contiguous share of ids."""

    def __init__(self, field_name, grid, n, velocity, ids, workers=None,
                 bodies="recon_flux"):
        if bodies not in ("recon_flux", "iteration"):
            raise ValueError(f"unknown bodies {bodies!r}")
        self.bodies = bodies
        ids = list(ids)
        workers = workers or os.cpu_count() or 1
        workers = max(1, min(workers, len(ids)))
        self.workers = workers
        self.count = len(ids)
        ctx = mp.get_context("spawn")
        chunks = np.array_split(np.asarray(ids), workers)
        self.procs, self.conns = [], []
        for chunk in chunks:
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker_main,
                            args=(b, field_name, grid, n, velocity,
                                  [int(x) for x in chunk], bodies),
                            daemon=True)
            p.start()
            self.procs.append(p)
            self.conns.append(a)
        for c in self.conns:
            assert c.recv() == "ready"

    def step(self) -> float:
        """One pass over all ids; returns the slowest worker's seconds."""
        for c in self.conns:
            c.send(1)
        return max(c.recv() for c in self.conns)

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=5)
            if p.is_alive():
                p.kill()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
