"""Wall-clock mirror of the reference benchmark matrix (taskfuse/bench.py).

The reference sweeps executors x max_team on its VIRTUAL device and reports
virtual ms/step (bench.py:156-245).  This module runs the same sweep on the
real B200 through the device-resident HydroSim mirror (one Python task per
sub-grid per iteration, five aggregated region visits each, real streams,
real pinned/device staging buffers, one batched kernel per team), and
reports the same columns (bench.py:248-249) measured with the wall clock:

    cores subgrid executors max_team ms_per_step kernels transfers
    raw_allocs syncs

plus the team-size histogram and the raw allocations / device syncs inside
the measured window (acceptance criterion 4: zero after warm-up).  This is
the per-task API path — its ms/step is dominated by Python task dispatch
(SURVEY F7); the throughput path is strategy3.TeamPlan / bench.py.
"""

from __future__ import annotations

import argparse
import csv
import io
import math
import time
from dataclasses import dataclass, field

import torch

from .bufferpool import BufferPool
from .device import CudaDevice
from .errors import UsageError, ValidationError
from .executorpool import ExecutorPool
from .hydro import HydroSim, driver, make_state
from .sched import Scheduler, SchedulerConfig

GRID_N = 64
COLUMNS = ("cores", "subgrid", "executors", "max_team", "ms_per_step",
           "kernels", "transfers", "raw_allocs", "syncs")
_SECTIONS = (
    ("Strategy 1: larger sub-grids",
     lambda r: r.executors == 1 and r.max_team == 1),
    ("Strategy 2: more executors",
     lambda r: r.executors >= 1 and r.max_team == 1),
    ("Strategy 3: on-the-fly aggregation", lambda r: r.executors == 1),
    ("Combined strategies", lambda r: r.executors > 1 and r.max_team > 1),
)


@dataclass(frozen=True)
class Row:
    cores: int
    subgrid: int
    executors: int
    max_team: int
    ms_per_step: float
    kernels: int
    transfers: int
    raw_allocs: int
    syncs: int
    team_sizes: dict = field(default_factory=dict, compare=False)
    measured_raw_allocs: int = field(default=0, compare=False)
    measured_syncs: int = field(default=0, compare=False)
    pinned_raw_allocs: int = field(default=0, compare=False)


@dataclass(frozen=True)
class BenchConfig:
    subgrid_n: int = 8
    executors: tuple = (1,)
    max_team: tuple = (1,)
    steps: int = 2
    fmt: str = "csv"

    def __post_init__(self):
        if self.steps < 1:
            raise ValidationError(f"steps must be >= 1, got {self.steps}")
        if self.fmt not in ("csv", "markdown"):
            raise ValidationError(f"unknown format {self.fmt!r}")


@dataclass(frozen=True)
class Report:
    rows: tuple
    steps: int = 0


def _presize_pools(buffers: BufferPool, subgrid_n: int, grid_n: int,
                   max_team: int) -> None:
    """bench.py:142-153: every (shape, team size) bucket the run can touch,
    so the steady state never raw-allocates."""
    tasks = (grid_n // subgrid_n) ** 3
    ext3 = (subgrid_n + 6) ** 3
    n3 = subgrid_n ** 3
    for size in range(1, min(max_team, tasks) + 1):
        count = math.ceil(tasks / size)
        for kind in ("device", "pinned_host"):
            for length in (ext3, n3):
                buffers.ensure(kind, "f8", length * size, count)
    buffers.materialise_all()


def run_cell(subgrid_n: int, executors: int, max_team: int, steps: int,
             policy: str = "round_robin", grid_n: int = GRID_N,
             field=None, engine: str = "native"):
    """Warm-up step + `steps` measured steps; returns (Row, sim, device).
    engine: "native" — the HydroSim tasks run in the C++ engine (the
    throughput path of the reference API); "python" — one Python generator
    per task through the mirrored AggregationRegion."""
    if executors < 1:
        raise UsageError("the B200 matrix has no host-only cell")
    sched = Scheduler(SchedulerConfig(worker_count=32))
    state = make_state(subgrid_n, grid_n, field=field)
    device = CudaDevice(sched)
    pool = ExecutorPool(sched, device, executors, policy)
    buffers = BufferPool(device) if engine == "python" else None
    sim = HydroSim(sched, state, pool, buffers, max_team=max_team,
                   engine=engine)
    if sim.native is not None:
        sim.presize()
    else:
        _presize_pools(buffers, subgrid_n, grid_n, max_team)
    marks = []

    def on_step(_index):
        torch.cuda.synchronize()
        marks.append((time.perf_counter(), device.kernels_enqueued,
                      device.copies_enqueued,
                      device.raw_allocations["device"],
                      device.sync_count,
                      device.raw_allocations["pinned_host"],
                      # native engine: real cudaMalloc / cudaHostAlloc
                      # calls past its reserved staging arenas (chunks are
                      # carved from the arenas lazily, by size class)
                      sim.native.counters()["allocated"]
                      if sim.native is not None else 0))

    sched.spawn(lambda: driver(sim, steps + 1, on_step), label="bench")
    sched.run()
    warm, last = marks[0], marks[-1]
    ms = (last[0] - warm[0]) * 1e3 / steps

    def per_step(a, b):
        d = a - b
        return d // steps if d % steps == 0 else d / steps

    sizes: dict[int, int] = {}
    for region in sim.regions.values():
        for size, count in region.stats().size_histogram.items():
            sizes[size] = sizes.get(size, 0) + count
    return Row(
        cores=1, subgrid=subgrid_n, executors=executors, max_team=max_team,
        ms_per_step=round(ms, 3),
        kernels=per_step(last[1], warm[1]),
        transfers=per_step(last[2], warm[2]),
        # the reference's column counts device allocations only
        # (bench.py:212); pinned staging allocations are reported beside it
        raw_allocs=last[3], syncs=last[4],
        team_sizes=dict(sorted(sizes.items())),
        measured_raw_allocs=(last[3] - warm[3]) + (last[5] - warm[5])
        + (last[6] - warm[6]),
        measured_syncs=last[4] - warm[4],
        pinned_raw_allocs=last[5],
    ), sim, device


def run_matrix(cfg: BenchConfig, grid_n: int = GRID_N,
               engine: str = "native") -> Report:
    """The executors x max_team sweep (bench.py:220-245).  The reference's
    extra (0, 1) host-only row is not produced: this framework has no CPU
    compute path; bench.py times the reference's CPU task
    iteration separately as the config-1 baseline."""
    cells = [(e, c) for e in sorted(set(cfg.executors))
             for c in sorted(set(cfg.max_team))]
    rows = [run_cell(cfg.subgrid_n, e, c, cfg.steps, grid_n=grid_n,
                     engine=engine)[0]
            for e, c in cells]
    return Report(rows=tuple(rows), steps=cfg.steps)


def _cells(row: Row) -> list[str]:
    return [str(getattr(row, col)) for col in COLUMNS]


def emit(report: Report, fmt: str = "csv") -> str:
    """bench.py:266-291 format (csv or sectioned markdown)."""
    if fmt == "csv":
        out = io.StringIO()
        w = csv.writer(out, lineterminator="\n")
        w.writerow(COLUMNS)
        for row in report.rows:
            w.writerow(_cells(row))
        return out.getvalue()
    if fmt != "markdown":
        raise ValidationError(f"unknown format {fmt!r}")
    lines = [f"# Work aggregation benchmark: B200 wall clock, "
             f"{report.steps} measured steps", ""]
    header = "| " + " | ".join(COLUMNS) + " |"
    rule = "|" + "|".join(" --- " for _ in COLUMNS) + "|"
    for title, belongs in _SECTIONS:
        rows = [r for r in report.rows if belongs(r)]
        if not rows:
            continue
        lines += [f"## {title}", "", header, rule]
        lines += ["| " + " | ".join(_cells(r)) + " |" for r in rows]
        lines.append("")
    return "\n".join(lines)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="bench_matrix")
    ap.add_argument("--subgrid-n", type=int, default=8, choices=(8, 16))
    ap.add_argument("--executors", type=int, nargs="+", default=[1])
    ap.add_argument("--max-team", type=int, nargs="+", default=[1])
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--grid-n", type=int, default=GRID_N)
    ap.add_argument("--format", choices=("csv", "markdown"), default="csv")
    ap.add_argument("--engine", choices=("native", "python"),
                    default="native")
    a = ap.parse_args(argv)
    cfg = BenchConfig(a.subgrid_n, tuple(a.executors), tuple(a.max_team),
                      a.steps, a.format)
    print(emit(run_matrix(cfg, a.grid_n, a.engine), a.format))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
