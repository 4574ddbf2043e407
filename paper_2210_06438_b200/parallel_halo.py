"""Multi-GPU slab partition of the sub-grid lattice with a ghost-layer
exchange — SURVEY §8(e).

The reference runs one process on one (virtual) device and fills ghosts
from the 26 periodic neighbours in memory (scenario.py:124-142); multi-GPU
is a non-goal there.  Here the m^3 lattice of sub-grids is
cut into x-slabs of mx = m / world sub-grid layers, one slab per rank (one
process per GPU).  Because x is the slowest lattice axis, a slab is a
contiguous range of sub-grid ids.  Within an iteration sub-grids are
independent (each reads only the current field, scenario.py:9-11), so the
only cross-rank traffic is, per iteration, each rank's 3 lowest and 3
highest owned x cell layers (3 x G x G FP64 each, G = m*n) to its two ring
neighbours (periodic wrap).  There is no global reduction: dt is fixed
(SURVEY F11).

Overlap: interior sub-grid layers (1 .. mx-2) need no halo, so they are
ghost-filled and computed while the planes are in flight on a separate
stream; the two boundary layers follow once the planes land.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, ops
from .errors import ValidationError

GHOST = 3


@dataclass(frozen=True)
class SlabPartition:
    grid_n: int
    n: int
    world: int
    rank: int

    def __post_init__(self):
        if self.grid_n % self.n:
            raise ValidationError("sub-grid edge must divide the grid")
        if self.m % self.world:
            raise ValidationError(
                f"{self.m} sub-grid layers do not split over {self.world} "
                "ranks")
        if not 0 <= self.rank < self.world:
            raise ValidationError("rank out of range")

    @property
    def m(self) -> int:
        return self.grid_n // self.n

    @property
    def mx(self) -> int:
        return self.m // self.world

    @property
    def x0(self) -> int:
        """First sub-grid x layer of this rank's slab."""
        return self.rank * self.mx

    @property
    def left(self) -> int:
        return (self.rank - 1) % self.world

    @property
    def right(self) -> int:
        return (self.rank + 1) % self.world

    @property
    def subgrids(self) -> int:
        return self.mx * self.m * self.m

    @property
    def id_range(self) -> tuple[int, int]:
        """Global lexicographic ids owned by this rank (contiguous)."""
        lo = self.x0 * self.m * self.m
        return lo, lo + self.subgrids

    @property
    def plane_shape(self) -> tuple[int, int, int]:
        return (GHOST, self.grid_n, self.grid_n)

    @property
    def plane_bytes(self) -> int:
        return 8 * GHOST * self.grid_n * self.grid_n

    def slab(self, field):
        """This rank's (mx*n, G, G) part of a global (G, G, G) field."""
        a = self.x0 * self.n
        return field[a:a + self.mx * self.n]


def exchange_halos(part: SlabPartition, lo, hi, halo_lo, halo_hi,
                   group=None) -> None:
    """Send my hi plane right and my lo plane left; receive the left
    neighbour's hi into halo_lo and the right neighbour's lo into halo_hi.
    Tags (and, for NCCL, the fixed per-peer order) keep the two planes apart
    when left == right (world 2)."""
    if part.world == 1:
        halo_lo.copy_(hi)
        halo_hi.copy_(lo)
        return
    import torch.distributed as dist
    if lo.is_cuda and dist.get_backend(group) == "gloo":
        # gloo moves host tensors only (ranks sharing one GPU in tests):
        # stage the planes through host memory
        h = [t.cpu() for t in (lo, hi, halo_lo, halo_hi)]
        exchange_halos(part, *h, group=group)
        halo_lo.copy_(h[2])
        halo_hi.copy_(h[3])
        return
    ops_ = [dist.P2POp(dist.isend, hi, part.right, group, tag=1),
            dist.P2POp(dist.isend, lo, part.left, group, tag=2),
            dist.P2POp(dist.irecv, halo_lo, part.left, group, tag=1),
            dist.P2POp(dist.irecv, halo_hi, part.right, group, tag=2)]
    for req in dist.batch_isend_irecv(ops_):
        req.wait()


def pool_from_slab(slab: torch.Tensor, n: int, m: int) -> torch.Tensor:
    """(mx*n, G, G) owned cells -> (mx*m*m, E, E, E) pool, ghosts NaN."""
    X = slab.shape[0]
    mx = X // n
    e = n + 2 * GHOST
    pool = torch.full((mx * m * m, e, e, e), float("nan"),
                      dtype=torch.float64, device=slab.device)
    blocks = slab.reshape(mx, n, m, n, m, n).permute(0, 2, 4, 1, 3, 5)
    pool[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n] = \
        blocks.reshape(mx * m * m, n, n, n)
    return pool


def slab_from_pool(pool: torch.Tensor, n: int, m: int) -> torch.Tensor:
    mx = pool.shape[0] // (m * m)
    own = pool[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n]
    return own.reshape(mx, m, m, n, n, n).permute(0, 3, 1, 4, 2, 5) \
        .reshape(mx * n, m * n, m * n).contiguous()


class SlabHydro:
    """One rank's device-resident slab: ghost exchange + aggregated
    reconstruct+flux + update per iteration."""

    def __init__(self, part: SlabPartition, slab_field, velocity=(1., 1., 1.),
                 dt_dx=None, device=None):
        from .hydro.scenario import dt_over_dx
        self.part = part
        self.n = part.n
        self.velocity = tuple(float(v) for v in velocity)
        self.dt_dx = dt_over_dx(velocity) if dt_dx is None else dt_dx
        dev = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        if isinstance(slab_field, np.ndarray):
            slab_field = torch.from_numpy(np.ascontiguousarray(slab_field))
        slab_field = slab_field.to(dev, torch.float64)
        self.u = pool_from_slab(slab_field, self.n, part.m)
        self.u_next = torch.full_like(self.u, float("nan"))
        c = self.n + 2
        S = part.subgrids
        self.um = torch.empty((S, 3, c, c, c), dtype=torch.float64, device=dev)
        self.up = torch.empty_like(self.um)
        self.F = torch.empty_like(self.um)
        shp = part.plane_shape
        self.lo, self.hi, self.halo_lo, self.halo_hi = (
            torch.empty(shp, dtype=torch.float64, device=dev)
            for _ in range(4))
        self.comm_stream = torch.cuda.Stream(device=dev)
        self.lib = _lib.load()

    # -- stages ---------------------------------------------------------------
    def pack(self, stream=None) -> None:
        p = self.part
        s = (stream or torch.cuda.current_stream()).cuda_stream
        _lib.check(self.lib.tf_halo_pack_f64(
            self.u.data_ptr(), self.n, p.mx, p.m, self.lo.data_ptr(),
            self.hi.data_ptr(), s), "tf_halo_pack_f64")

    def fill(self, first: int, count: int, stream=None) -> None:
        p = self.part
        s = (stream or torch.cuda.current_stream()).cuda_stream
        _lib.check(self.lib.tf_ghost_fill_slab_f64(
            self.u.data_ptr(), self.n, p.mx, p.m, self.halo_lo.data_ptr(),
            self.halo_hi.data_ptr(), first, count, s),
            "tf_ghost_fill_slab_f64")

    def compute(self, first: int, count: int, stream=None) -> None:
        """recon+flux then update for local ids [first, first+count)."""
        if count == 0:
            return
        ids = self._ids(first, count)
        ops.recon_flux(self.u, self.n, self.velocity, self.um, self.up,
                       self.F, ids=ids, out_mode=1, stream=stream)
        ops.update(self.u, self.n, self.F, self.dt_dx, self.u_next, ids=ids,
                   out_mode=1, stream=stream)

    def _ids(self, first, count):
        key = (first, count)
        cache = self.__dict__.setdefault("_id_cache", {})
        if key not in cache:
            cache[key] = torch.arange(first, first + count, dtype=torch.int32,
                                      device=self.u.device)
        return cache[key]

    def swap(self) -> None:
        self.u, self.u_next = self.u_next, self.u

    # -- one iteration ----------------------------------------------------------
    def iteration(self, exchange=None, overlap=True) -> None:
        """exchange(part, lo, hi, halo_lo, halo_hi) defaults to the
        torch.distributed ring exchange."""
        exchange = exchange or exchange_halos
        p = self.part
        mm = p.m * p.m
        cur = torch.cuda.current_stream()
        self.pack(cur)
        if not overlap or p.mx <= 2:
            exchange(p, self.lo, self.hi, self.halo_lo, self.halo_hi)
            self.fill(0, p.subgrids, cur)
            self.compute(0, p.subgrids, cur)
        else:
            self.comm_stream.wait_stream(cur)
            with torch.cuda.stream(self.comm_stream):
                exchange(p, self.lo, self.hi, self.halo_lo, self.halo_hi)
            # interior layers: no halo needed
            self.fill(mm, p.subgrids - 2 * mm, cur)
            self.compute(mm, p.subgrids - 2 * mm, cur)
            cur.wait_stream(self.comm_stream)
            self.fill(0, mm, cur)
            self.fill(p.subgrids - mm, mm, cur)
            self.compute(0, mm, cur)
            self.compute(p.subgrids - mm, mm, cur)
        self.swap()

    def owned(self) -> torch.Tensor:
        """(mx*n, G, G) owned field of the current pool."""
        return slab_from_pool(self.u, self.n, self.part.m)
