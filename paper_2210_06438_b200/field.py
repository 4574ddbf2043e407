"""Fused full iteration on a padded global field — SURVEY §8(f) rank 2.

The materialising path (ghost-filled per-sub-grid pools, um/up/F written to
HBM, separate update) moves ~150 KB per 8^3 sub-grid-iteration.  Here the
field is stored once, padded by the stencil's halo (csrc/field_step.cu), and
one fused kernel per team does reconstruct + flux + update for its
sub-grids: ~22.5 KB per sub-grid-iteration.  Strategy 3 is unchanged on
top: teams formed by the same formation core, one launch per team, the
iteration's team launches captured as a CUDA graph over the executor
branches with PDL between consecutive teams.  Bit-identical to
reference_step (tests/test_gpu_field.py).

`FieldIteration` — one GPU.  `SlabFieldIteration` — one rank of an x-slab
partition: the x halo layers are contiguous slices of the padded array, so
the ring exchange sends/receives them in place (no pack kernel), and the
interior sub-grid layers are stepped while the planes are in flight.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import TaskfuseCudaError, ValidationError
from .parallel_halo import SlabPartition, exchange_halos
from .strategy3 import Team, form_teams

HX, HY, HZ = 2, 2, 4


def padded_shape(X: int, G: int) -> tuple[int, int, int]:
    return (X + 2 * HX, G + 2 * HY, G + 2 * HZ)


def taper_layers(L: int) -> list[int]:
    """Sub-grid layers per upload chunk for the host pipeline: small first
    and last chunks shorten the pipeline's fill (nothing to step before the
    first upload lands) and drain (the last chunk's step + download after
    the last upload); measured best at L = 16: [1, 3, 4, 4, 3, 1]."""
    base = [1, 3, 4, 4, 3, 1]
    if L < 2 * len(base):
        return [1] * L if L < 4 else [1] + [L - 2] + [1]
    w = [max(1, round(b * L / 16)) for b in base]
    k = 2
    while sum(w) != L:          # fix rounding in the middle chunks
        w[k] += 1 if sum(w) < L else -1
        k = 3 if k == 2 else 2
    return w


def interior(P: torch.Tensor) -> torch.Tensor:
    return P[HX:-HX, HY:-HY, HZ:-HZ]


class _FieldBase:
    def __init__(self, X: int, G: int, n: int, velocity, dt_dx, device):
        from .hydro.scenario import dt_over_dx
        if n not in (8, 16) or X % n or G % n:
            raise ValidationError("sub-grid edge must be 8 or 16 and divide "
                                  "the field extents")
        self.lib = _lib.load()
        self.X, self.G, self.n = X, G, n
        self.m = G // n
        self.mx = X // n
        self.S = self.mx * self.m * self.m
        self.velocity = tuple(float(v) for v in velocity)
        self.dt_dx = dt_over_dx(velocity) if dt_dx is None else float(dt_dx)
        dev = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.P = [torch.full(padded_shape(X, G), float("nan"),
                             dtype=torch.float64, device=dev)
                  for _ in range(2)]
        self.cur = 0

    @property
    def field(self) -> torch.Tensor:
        return self.P[self.cur]

    def _s(self, stream=None) -> int:
        return (stream or torch.cuda.current_stream()).cuda_stream

    def load(self, field_dev: torch.Tensor, stream=None) -> None:
        """(X, G, G) device field -> current padded interior."""
        _lib.check(self.lib.tf_field_pad_f64(
            field_dev.data_ptr(), self.X, self.G, self.G,
            self.field.data_ptr(), self._s(stream)), "tf_field_pad_f64")

    def store(self, field_dev: torch.Tensor, stream=None) -> None:
        _lib.check(self.lib.tf_field_unpad_f64(
            self.field.data_ptr(), self.X, self.G, self.G,
            field_dev.data_ptr(), self._s(stream)), "tf_field_unpad_f64")

    def halo(self, periodic_x: bool, stream=None) -> None:
        _lib.check(self.lib.tf_field_halo_f64(
            self.field.data_ptr(), self.X, self.G, self.G, int(periodic_x),
            self._s(stream)), "tf_field_halo_f64")

    def step_ids(self, ids: torch.Tensor | None, T: int, stream=None) -> None:
        """One fused step for T sub-grids (device ids, or the first T)."""
        cur, nxt = self.P[self.cur], self.P[1 - self.cur]
        ax, ay, az = self.velocity
        _lib.check(self.lib.tf_field_step_f64(
            cur.data_ptr(), self.X, self.G, self.G, self.n,
            None if ids is None else ids.data_ptr(), None, T, ax, ay, az,
            self.dt_dx, nxt.data_ptr(), 0, self._s(stream)),
            "tf_field_step_f64")

    def march_ok(self) -> bool:
        """The whole-slab march kernel tiles the field by 8-row x 32-cell
        warp columns (csrc/field_march.cu)."""
        return self.G % 32 == 0

    def march(self, flags: int = 0, peer_lo: int | None = None,
              peer_hi: int | None = None, xc: int = 0, stream=None) -> None:
        """One fused iteration over EVERY sub-grid of the field in one launch
        (tf_field_march_f64): current -> next padded field.  flags:
        TF_STEP_HALO_YZ / TF_STEP_HALO_X (also write the next field's
        periodic halos), TF_MARCH_ROWS4; peer_lo / peer_hi: device pointers
        of the ring neighbours' next fields (their x halos)."""
        cur, nxt = self.P[self.cur], self.P[1 - self.cur]
        ax, ay, az = self.velocity
        work = getattr(self, "_march_work", None)
        if work is None:
            # the launch's item counters (the kernel leaves them zeroed);
            # one pair per object: concurrent iterations must not share
            work = self._march_work = torch.zeros(
                2, dtype=torch.int32, device=self.device)
        _lib.check(self.lib.tf_field_march_f64(
            cur.data_ptr(), self.X, self.G, self.G, ax, ay, az, self.dt_dx,
            nxt.data_ptr(), peer_lo, peer_hi, flags, xc,
            work.data_ptr() if getattr(self, "march_dynamic", True) else None,
            self._s(stream)), "tf_field_march_f64")

    def swap(self) -> None:
        self.cur = 1 - self.cur

    def owned(self) -> torch.Tensor:
        return interior(self.field).contiguous()


class FieldPlan:
    """A formed team plan of the fused step captured as a CUDA graph.
    halo_flags: TF_STEP_HALO_YZ / TF_STEP_HALO_X (n = 8) — the team kernels
    also write the next field's periodic halos."""

    def __init__(self, teams: list[Team], fi: _FieldBase, src: int,
                 executors: int, overlap: bool = True, halo_flags: int = 0):
        lib = fi.lib
        ids = np.concatenate([np.asarray(t.ids, np.int32) for t in teams])
        offs = np.zeros(len(teams) + 1, np.int64)
        offs[1:] = np.cumsum([len(t.ids) for t in teams])
        exe = np.asarray([t.executor for t in teams], np.int32)
        self._keep = (ids, offs, exe)
        ax, ay, az = fi.velocity
        h = C.c_void_p()
        _lib.check(lib.tf_plan_capture_field_step(
            ids.ctypes.data_as(C.POINTER(C.c_int32)),
            offs.ctypes.data_as(C.POINTER(C.c_int64)),
            exe.ctypes.data_as(C.POINTER(C.c_int32)), len(teams), executors,
            fi.P[src].data_ptr(), fi.X, fi.G, fi.G, fi.n, ax, ay, az,
            fi.dt_dx, fi.P[1 - src].data_ptr(),
            (_lib.TF_LAUNCH_OVERLAP_PREV if overlap else 0) | halo_flags,
            C.byref(h)),
            "tf_plan_capture_field_step")
        self.lib, self.handle = lib, h
        self.kernels = lib.tf_plan_kernels(h)

    def launch(self, stream=None) -> None:
        s = stream or torch.cuda.current_stream()
        _lib.check(self.lib.tf_plan_launch(self.handle, s.cuda_stream),
                   "tf_plan_launch")

    def __del__(self):
        if getattr(self, "handle", None):
            self.lib.tf_plan_destroy(self.handle)
            self.handle = None


class FieldIteration(_FieldBase):
    """One-GPU fused iteration with strategy-3 team launches."""

    def __init__(self, grid_n: int, n: int, velocity=(1.0, 1.0, 1.0),
                 max_team: int = 128, executors: int = 4, dt_dx=None,
                 device=None, overlap: bool = True):
        super().__init__(grid_n, grid_n, n, velocity, dt_dx, device)
        self.teams = form_teams(range(self.S), max_team, executors)
        # n = 8: the team kernels write the next field's periodic halos
        # themselves (every sub-grid is in some team), so only a freshly
        # loaded field needs the halo kernels
        self.kernel_halo = n == 8
        hf = _lib.TF_STEP_HALO_YZ | _lib.TF_STEP_HALO_X \
            if self.kernel_halo else 0
        self.plans = [FieldPlan(self.teams, self, src, executors, overlap,
                                halo_flags=hf)
                      for src in (0, 1)]
        self.halo_fresh = False
        self.field_dev = torch.empty((grid_n,) * 3, dtype=torch.float64,
                                     device=self.device)

    def load(self, field_dev: torch.Tensor, stream=None) -> None:
        super().load(field_dev, stream)
        self.halo_fresh = False

    def step(self, stream=None) -> None:
        if not self.halo_fresh:
            self.halo(True, stream)
        self.plans[self.cur].launch(stream)
        self.swap()
        self.halo_fresh = self.kernel_halo

    def run_host(self, field_in, field_out, iterations: int = 1) -> None:
        """Host field (pinned) in -> iterations -> host field out."""
        from .strategy3 import copy_split
        copy_split(self.field_dev, field_in)   # two copy engines
        self.load(self.field_dev)
        for _ in range(iterations):
            self.step()
        self.store(self.field_dev)
        copy_split(field_out, self.field_dev)

    @property
    def launches_per_step(self) -> int:
        # one kernel per team (+ 2 halo kernels when n = 16)
        return len(self.teams) + (0 if self.kernel_halo else 2)

    def run_host_pipelined(self, field_in, field_out, chunks="taper",
                           down_ctas: int = 16,
                           down_stream: bool = True) -> int:
        """One iteration from a pinned host field to a pinned host field with
        the transfers overlapped.  The field moves in x-chunks on an upload
        stream (copy engine), each chunk's range shifted by the x halo
        (HX planes) so that chunk i can be stepped as soon as ITS upload
        lands: upload 0 also carries the field's last HX planes (the
        periodic low x halo) and every upload i carries chunk i+1's first HX
        planes.  Each landed range is scattered into the padded field and
        its y/z halos refreshed, chunk i is stepped (one fused launch over
        its sub-grids), and its updated owned cells go straight into the
        pinned output by a zero-copy kernel on a download stream (the copy
        engines serve only the upload).  The tail after the last upload is
        one chunk's step and download.  Returns kernel launches."""
        G, n, m = self.G, self.n, self.m
        L = self.mx
        if chunks == "taper":
            chunks = taper_layers(L)
        if isinstance(chunks, int):
            c = max(d for d in range(1, min(chunks, L) + 1) if L % d == 0)
            layers = [L // c] * c
        else:   # explicit sub-grid layers per chunk (e.g. small first/last)
            layers = [int(k) for k in chunks]
            if sum(layers) != L or min(layers) < 1:
                raise ValidationError(f"chunk layers must be positive and "
                                      f"sum to {L}")
        chunks = len(layers)
        if chunks < 2 or n <= 2 * HX:
            self.run_host(field_in, field_out)
            return self.launches_per_step + 2
        start = [0]
        for k in layers:
            start.append(start[-1] + k)     # chunk i = layers [start[i], start[i+1])
        if not (field_in.is_pinned() and field_out.is_pinned()):
            raise ValidationError("run_host_pipelined needs pinned host "
                                  "fields (torch pin_memory)")
        lib, X, H = self.lib, self.X, HX
        py, pz = G + 2 * HY, G + 2 * HZ
        lay_elems = py * pz
        plane = G * G
        P, Pn = self.P[self.cur], self.P[1 - self.cur]
        if not hasattr(self, "_pipe"):
            self._pipe = dict(up=torch.cuda.Stream(device=self.device),
                              down=torch.cuda.Stream(device=self.device),
                              ids={})
        pipe = self._pipe
        up, down = pipe["up"], pipe["down"]
        comp = torch.cuda.current_stream()
        dev_in = self.field_dev
        ranges = []
        for i in range(chunks):
            lo = start[i] * n + H if i else 0
            hi = start[i + 1] * n + H if i < chunks - 1 else X - H
            ranges.append(([(X - H, X)] if i == 0 else []) + [(lo, hi)])
        ev_up = [torch.cuda.Event() for _ in range(chunks)]
        ev_done = [torch.cuda.Event() for _ in range(chunks)]
        up.wait_stream(comp)
        down.wait_stream(comp)
        fin = field_in.view(G, G, G)
        with torch.cuda.stream(up):
            for i, rs in enumerate(ranges):
                for lo, hi in rs:
                    dev_in[lo:hi].copy_(fin[lo:hi], non_blocking=True)
                ev_up[i].record(up)
        cs, ds = comp.cuda_stream, down.cuda_stream
        ax, ay, az = self.velocity
        launches = 0
        for i, rs in enumerate(ranges):
            comp.wait_event(ev_up[i])
            # the chunk's padded layers in full (interior, periodic y/z
            # halos, and for chunk 0 both periodic x halos: their sources,
            # the first and last HX planes, landed with upload 0)
            lo, hi = rs[-1]
            spans = [(0, hi + HX), (X, 2 * HX)] if i == 0 else \
                [(lo + HX, hi - lo)]
            for first, count in spans:
                _lib.check(lib.tf_field_pad_halo_f64(
                    dev_in.data_ptr(), X, G, G, P.data_ptr(), first, count,
                    cs), "tf_field_pad_halo_f64")
                launches += 1
            a, b = start[i], start[i + 1]
            ids = pipe["ids"].get((a, b))
            if ids is None:
                ids = torch.arange(a * m * m, b * m * m, dtype=torch.int32,
                                   device=self.device)
                pipe["ids"][(a, b)] = ids
            _lib.check(lib.tf_field_step_f64(
                P.data_ptr(), X, G, G, n, ids.data_ptr(), None, ids.numel(),
                ax, ay, az, self.dt_dx, Pn.data_ptr(), 0, cs),
                "tf_field_step_f64")
            if down_stream and down_ctas > 0:
                ev_done[i].record(comp)
                down.wait_event(ev_done[i])
            if down_ctas > 0:
                _lib.check(lib.tf_field_unpad_host_f64(
                    Pn.data_ptr() + 8 * a * n * lay_elems, (b - a) * n, G, G,
                    field_out.data_ptr() + 8 * a * n * plane, down_ctas,
                    ds if down_stream else cs),
                    "tf_field_unpad_host_f64")
            else:   # copy-engine download through a device staging field
                out = pipe.setdefault("out", torch.empty_like(dev_in))
                _lib.check(lib.tf_field_unpad_f64(
                    Pn.data_ptr() + 8 * a * n * lay_elems, (b - a) * n, G, G,
                    out.data_ptr() + 8 * a * n * plane, cs),
                    "tf_field_unpad_f64")
                ev_done[i].record(comp)
                down.wait_event(ev_done[i])
                with torch.cuda.stream(down):
                    field_out.view(G, G, G)[a * n:b * n].copy_(
                        out[a * n:b * n], non_blocking=True)
            launches += 2
        comp.wait_stream(down)
        self.swap()
        self.halo_fresh = False     # the chunk steps write no halos
        return launches


class MarchFieldIteration(_FieldBase):
    """One-GPU fused iteration of the whole field in ONE launch per step:
    the march kernel (csrc/field_march.cu) also writes the next field's
    periodic y/z and x halos, so after the first step no halo kernel runs.
    The config-5 iteration at N = 1 (one team = every sub-grid)."""

    def __init__(self, grid_n: int, n: int = 8, velocity=(1.0, 1.0, 1.0),
                 dt_dx=None, device=None, xc: int = 0, rows4: bool = False,
                 along_y: bool = False):
        super().__init__(grid_n, grid_n, n, velocity, dt_dx, device)
        if not self.march_ok():
            raise ValidationError("the march kernel needs grid_n % 32 == 0")
        self.xc = xc
        self.flags = _lib.TF_STEP_HALO_YZ | _lib.TF_STEP_HALO_X | \
            (_lib.TF_MARCH_ROWS4 if rows4 else 0) | \
            (_lib.TF_MARCH_ALONG_Y if along_y else 0)
        self.halo_fresh = False

    def load(self, field_dev: torch.Tensor, stream=None) -> None:
        super().load(field_dev, stream)
        self.halo_fresh = False

    def step(self, stream=None) -> None:
        if not self.halo_fresh:
            self.halo(True, stream)
        self.march(self.flags, xc=self.xc, stream=stream)
        self.swap()
        self.halo_fresh = True

    launches_per_step = 1


class HostPipeline:
    """`FieldIteration.run_host_pipelined` for FIXED pinned host buffers,
    captured once as a CUDA graph (copies, per-chunk kernels and the
    cross-stream dependencies): one host->host iteration per replay, with no
    per-chunk host submission cost.  Pure function of `field_in` (the
    iteration's state is the host field), so every replay reads P[0] and
    writes P[1]."""

    def __init__(self, fi: "FieldIteration", field_in, field_out,
                 chunks="taper", down_ctas: int = 16,
                 down_stream: bool = True):
        self.fi = fi
        self.bufs = (field_in, field_out)
        fi.cur = 0
        fi.run_host_pipelined(field_in, field_out, chunks, down_ctas,
                              down_stream)  # warm-up
        fi.cur = 0
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=fi.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(self.graph, stream=s):
            self.launches = fi.run_host_pipelined(field_in, field_out, chunks,
                                                  down_ctas, down_stream)
        fi.cur = 0
        fi.halo_fresh = False
        torch.cuda.synchronize()

    def run(self) -> None:
        self.graph.replay()


class PeerSlabFieldIteration(_FieldBase):
    """x-slab rank with the exchange FUSED into the compute: the fused step
    stores the slab's boundary layers straight into the ring neighbours'
    next padded fields through CUDA-IPC peer pointers (NVLink on a
    multi-GPU node), then a device-side peer barrier (release/acquire flags
    in each rank's memory, written by the neighbours) orders the iterations.
    No NCCL call and no pack/unpack on the data path; NCCL/gloo is used once,
    at setup, to swap the IPC handles."""

    def __init__(self, part: SlabPartition, slab_field=None,
                 velocity=(1.0, 1.0, 1.0), dt_dx=None, device=None,
                 group=None, timeout_s: float = 10.0, kernel: str = "auto",
                 xc: int = 0, overlap_barrier: bool | None = None,
                 march_axis: str = "auto"):
        super().__init__(part.mx * part.n, part.grid_n, part.n, velocity,
                         dt_dx, device)
        self.part = part
        # "march": the whole-slab march kernel (also writes the next
        # field's y/z halos: no halo kernel per iteration); "cols": one CTA
        # per sub-grid (k_step_cols8s) + the halo kernels
        if kernel == "auto":
            kernel = "march" if self.march_ok() else "cols"
        if kernel not in ("march", "cols") or \
                (kernel == "march" and not self.march_ok()):
            raise ValidationError(f"kernel {kernel!r} not usable here")
        self.kernel, self.xc = kernel, xc
        # march axis: x (planes of the slab), or y for a thin slab (a rank's
        # share at N >= 4: columns of x rows marching the long y extent;
        # config 5 at 128 planes 143 vs 152 us, at 64 planes even, at 256
        # x ahead, 236 vs 260 us — DESIGN §9); "auto" picks y for a slab of
        # at most 128 planes and a quarter of the y extent
        if march_axis == "auto":
            march_axis = "y" if self.X <= 128 and self.X % 8 == 0 and \
                self.G >= 4 * self.X else "x"
        if march_axis not in ("x", "y") or \
                (march_axis == "y" and self.X % 8):
            raise ValidationError(f"march axis {march_axis!r} not usable here")
        self.march_axis = march_axis
        # march kernel: overlap the ring barrier with the next iteration's
        # interior (programmatic dependent launches; x-edge items wait).
        # Default: with real neighbours only — on one rank the barrier is a
        # self-handshake and the waiting variant's register pressure costs
        # as much as the overlap saves (457 vs 461 us at config 5)
        self.overlap_barrier = (part.world > 1 if overlap_barrier is None
                                else bool(overlap_barrier))
        self.timeout_ns = int(timeout_s * 1e9)
        dev = self.device
        self.flags = torch.zeros(2, dtype=torch.int64, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.epoch = 0
        if slab_field is not None:
            if isinstance(slab_field, np.ndarray):
                slab_field = torch.from_numpy(np.ascontiguousarray(slab_field))
            self.load(slab_field.to(dev, torch.float64))
        if part.world == 1:
            mine = {"P": self.P, "flags": self.flags}
            self.left = self.right = mine
        else:
            import torch.distributed as dist
            from torch.multiprocessing.reductions import reduce_tensor
            handles = {"P": [reduce_tensor(p) for p in self.P],
                       "flags": reduce_tensor(self.flags)}
            every = [None] * part.world
            dist.all_gather_object(every, handles, group=group)

            def open_(h):
                fn, args = h
                return fn(*args)

            def peer(r):
                return {"P": [open_(h) for h in every[r]["P"]],
                        "flags": open_(every[r]["flags"])}
            self.left = peer(part.left)
            self.right = self.left if part.right == part.left else \
                peer(part.right)
        self._prime()

    def _barrier(self, stream=None, pdl: bool = False) -> None:
        self.epoch += 1
        _lib.check(self.lib.tf_peer_barrier_ex(
            self.flags.data_ptr(), self.left["flags"].data_ptr(),
            self.right["flags"].data_ptr(), self.epoch, self.timeout_ns,
            self.err.data_ptr(), _lib.TF_BARRIER_PDL if pdl else 0,
            self._s(stream)), "tf_peer_barrier_ex")

    def _prime(self) -> None:
        """Initial x halo of the current field: copy my boundary layers into
        the neighbours' halos over the peer mapping, then barrier."""
        X, c = self.X, self.cur
        self.halo(False)
        self.left["P"][c][X + HX:X + 2 * HX].copy_(self.P[c][HX:2 * HX])
        self.right["P"][c][0:HX].copy_(self.P[c][X:X + HX])
        self._barrier()

    def iteration(self) -> None:
        cur, nxt = self.cur, 1 - self.cur
        if self.kernel == "march":
            # y/z halos of the current field: written by the previous
            # iteration's kernel (or _prime); the x halo by the neighbours.
            # overlap: this march is a programmatic dependent of the
            # previous barrier — its interior runs while the epochs are
            # exchanged, only its x-edge items wait for the barrier — and
            # the barrier a programmatic dependent of this march
            ov = self.overlap_barrier
            self.march(_lib.TF_STEP_HALO_YZ |
                       (_lib.TF_MARCH_PDL_EDGE if ov else 0) |
                       (_lib.TF_MARCH_ALONG_Y if self.march_axis == "y"
                        else 0),
                       self.left["P"][nxt].data_ptr(),
                       self.right["P"][nxt].data_ptr(), self.xc)
            self._barrier(pdl=self.overlap_barrier)
            self.swap()
            return
        self.halo(False)          # y/z halos incl. the received x layers
        ax, ay, az = self.velocity
        _lib.check(self.lib.tf_field_step_peer_f64(
            self.P[cur].data_ptr(), self.X, self.G, self.G, self.n, None,
            self.S, ax, ay, az, self.dt_dx, self.P[nxt].data_ptr(),
            self.left["P"][nxt].data_ptr(), self.right["P"][nxt].data_ptr(),
            self._s()), "tf_field_step_peer_f64")
        self._barrier()
        self.swap()

    def run_host(self, slab_in, slab_out) -> None:
        """End-to-end iteration of this rank's slab through HOST buffers:
        the pinned (mx*n, G, G) slab goes host->device and is padded, its
        boundary layers are primed into the neighbours' halos (peer copies
        + device barrier), one fused iteration runs with the exchange fused
        into the step, and the updated slab comes back to the pinned
        `slab_out`.  Every rank calls it once per step."""
        if not (slab_in.is_pinned() and slab_out.is_pinned()):
            raise ValidationError("run_host needs pinned host slabs")
        dev = getattr(self, "_host_dev", None)
        if dev is None:
            dev = self._host_dev = torch.empty(
                (self.X, self.G, self.G), dtype=torch.float64,
                device=self.device)
        from .strategy3 import copy_split
        copy_split(dev, slab_in)       # two copy engines (strategy3)
        self.load(dev)
        self._prime()
        self.iteration()
        self.store(dev)
        copy_split(slab_out, dev)

    def check(self) -> None:
        """Raise if a peer barrier timed out."""
        if int(self.err.item()):
            raise TaskfuseCudaError("peer barrier timed out: a neighbour "
                                    "rank did not arrive")


class SlabFieldIteration(_FieldBase):
    """One rank's x-slab of a padded global field (multi-GPU)."""

    def __init__(self, part: SlabPartition, slab_field=None,
                 velocity=(1.0, 1.0, 1.0), dt_dx=None, device=None):
        super().__init__(part.mx * part.n, part.grid_n, part.n, velocity,
                         dt_dx, device)
        self.part = part
        mm = self.m * self.m
        self.comm_stream = torch.cuda.Stream(device=self.device)
        ar = lambda a, b: torch.arange(a, b, dtype=torch.int32,  # noqa: E731
                                       device=self.device)
        self.interior_ids = ar(mm, self.S - mm) if self.mx > 2 else None
        self.boundary_ids = torch.cat([ar(0, mm), ar(self.S - mm, self.S)]) \
            if self.mx > 1 else ar(0, self.S)
        if slab_field is not None:
            if isinstance(slab_field, np.ndarray):
                slab_field = torch.from_numpy(np.ascontiguousarray(slab_field))
            self.load(slab_field.to(self.device, torch.float64))

    def _planes(self):
        P, X = self.field, self.X
        # lo = my lowest 2 owned x layers, hi = my highest; halos in place
        return (P[HX:2 * HX], P[X:X + HX], P[0:HX], P[X + HX:X + 2 * HX])

    def iteration(self, exchange=None, overlap: bool = True) -> None:
        exchange = exchange or exchange_halos
        cur = torch.cuda.current_stream()
        self.halo(False, cur)                      # y/z halos, own layers
        lo, hi, halo_lo, halo_hi = self._planes()
        if not overlap or self.interior_ids is None:
            exchange(self.part, lo, hi, halo_lo, halo_hi)
            self.step_ids(None, self.S, cur)
        else:
            self.comm_stream.wait_stream(cur)
            with torch.cuda.stream(self.comm_stream):
                exchange(self.part, lo, hi, halo_lo, halo_hi)
            self.step_ids(self.interior_ids, self.interior_ids.numel(), cur)
            cur.wait_stream(self.comm_stream)
            self.step_ids(self.boundary_ids, self.boundary_ids.numel(), cur)
        self.swap()
