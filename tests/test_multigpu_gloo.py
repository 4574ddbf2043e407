"""Multi-process (gloo, world 2 and 4) test of the slab partition and the
ring halo exchange of paper_2210_06438_b200.parallel_halo, on CPU.

Each rank owns an x-slab of the sub-grid lattice, packs its boundary layers
(oracle restatement), exchanges them with the PRODUCT's exchange_halos over
a real torch.distributed process group, fills its ghosts and advances its
slab with the oracle numerics.  The gathered field must be bit-identical to
the whole-grid reference iteration (decomposition invariance,
test_hydro.py:139-142)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import hydro_oracle as HO


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _slab_pool(slab, n, m):
    mx = slab.shape[0] // n
    e = n + 6
    pool = np.full((mx * m * m, e, e, e), np.nan)
    blocks = slab.reshape(mx, n, m, n, m, n).transpose(0, 2, 4, 1, 3, 5)
    pool[:, 3:3 + n, 3:3 + n, 3:3 + n] = blocks.reshape(mx * m * m, n, n, n)
    return pool


def _worker(rank, world, port, grid, n, iters, velocity, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2210_06438_b200.parallel_halo import (SlabPartition,
                                                     exchange_halos)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = SlabPartition(grid, n, world, rank)
        field = HO.stress_field(grid)
        pool = _slab_pool(part.slab(field), n, part.m)
        for _ in range(iters):
            lo, hi = HO.slab_pack(pool, n, part.mx, part.m)
            t = [torch.from_numpy(a) for a in (lo, hi)]
            halo_lo = torch.empty(part.plane_shape, dtype=torch.float64)
            halo_hi = torch.empty(part.plane_shape, dtype=torch.float64)
            exchange_halos(part, t[0], t[1], halo_lo, halo_hi)
            HO.slab_fill(pool, n, part.mx, part.m, halo_lo.numpy(),
                         halo_hi.numpy())
            _, _, F = HO.recon_flux_batch(pool, n, velocity)
            nxt = np.full_like(pool, np.nan)
            nxt[:, 3:3 + n, 3:3 + n, 3:3 + n] = HO.update_batch(
                pool, F, n, HO.dt_over_dx(velocity))
            pool = nxt
        lo, hi = HO.slab_pack(pool, n, part.mx, part.m)  # not used: shape
        own = pool[:, 3:3 + n, 3:3 + n, 3:3 + n]
        slab = own.reshape(part.mx, part.m, part.m, n, n, n) \
            .transpose(0, 3, 1, 4, 2, 5).reshape(part.mx * n, grid, grid)
        gathered = [torch.empty_like(torch.from_numpy(slab))
                    for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(np.ascontiguousarray(slab)))
        if rank == 0:
            out_q.put(np.concatenate([g.numpy() for g in gathered], axis=0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,velocity", [
    (2, (1.0, 1.0, 1.0)), (2, (-1.0, 0.5, -0.25)), (4, (0.7, -1.3, 0.0))])
def test_slab_partition_matches_whole_grid(world, velocity):
    grid, n, iters = 32, 8, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, grid, n, iters, velocity, q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        got = q.get(timeout=120)
    finally:
        for p in procs:
            p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    ref = HO.stress_field(grid)
    for _ in range(iters):
        ref = HO.advect_once(ref, velocity)
    assert np.array_equal(got, ref)


def test_partition_geometry():
    from paper_2210_06438_b200.errors import ValidationError
    from paper_2210_06438_b200.parallel_halo import SlabPartition
    p = SlabPartition(512, 8, 8, 3)
    assert (p.m, p.mx, p.x0, p.left, p.right) == (64, 8, 24, 2, 4)
    assert p.subgrids == 32768 and p.id_range == (98304, 131072)
    assert p.plane_bytes == 3 * 512 * 512 * 8
    assert SlabPartition(512, 8, 8, 0).left == 7
    with pytest.raises(ValidationError):
        SlabPartition(512, 8, 3, 0)      # 64 layers do not split over 3
    with pytest.raises(ValidationError):
        SlabPartition(100, 8, 1, 0)
