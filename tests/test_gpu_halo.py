"""CUDA halo pack / slab ghost fill / SlabHydro on one GPU with virtual
ranks: W slabs on the same device, planes handed to the ring neighbours by
the same pairing exchange_halos uses.  The partitioned iteration must be
bit-identical to the whole-grid reference (decomposition invariance), for
the sequential and the interior/boundary-overlapped schedule."""

import numpy as np
import pytest

from oracle import hydro_oracle as HO

pytestmark = pytest.mark.gpu


def _ranks(grid, n, world, field, velocity, dev):
    from paper_2210_06438_b200.parallel_halo import SlabHydro, SlabPartition
    return [SlabHydro(SlabPartition(grid, n, world, r),
                      SlabPartition(grid, n, world, r).slab(field), velocity,
                      device=dev) for r in range(world)]


def _virtual_iteration(ranks):
    import torch
    for r in ranks:
        r.pack()
    for r in ranks:
        p = r.part
        r.halo_lo.copy_(ranks[p.left].hi)
        r.halo_hi.copy_(ranks[p.right].lo)
    for r in ranks:
        r.fill(0, r.part.subgrids)
        r.compute(0, r.part.subgrids)
        r.swap()
    torch.cuda.synchronize()


@pytest.mark.parametrize("world,n,grid,velocity", [
    (1, 8, 32, (1.0, 1.0, 1.0)), (2, 8, 32, (-1.0, 0.5, -0.25)),
    (4, 8, 64, (0.7, -1.3, 0.0)), (2, 16, 64, (1.0, 1.0, 1.0))])
def test_virtual_ranks_match_whole_grid(cuda, world, n, grid, velocity):
    import torch
    field = HO.stress_field(grid)
    ranks = _ranks(grid, n, world, field, velocity, cuda)
    iters = 3
    for _ in range(iters):
        _virtual_iteration(ranks)
    got = torch.cat([r.owned() for r in ranks]).cpu().numpy()
    ref = field
    for _ in range(iters):
        ref = HO.advect_once(ref, velocity)
    assert np.array_equal(got, ref)


def test_pack_and_fill_match_oracle(cuda):
    from paper_2210_06438_b200 import ops
    import torch
    grid, n = 32, 8
    field = HO.initial_field(grid)
    (r,) = _ranks(grid, n, 1, field, (1.0, 1.0, 1.0), cuda)
    r.pack()
    hp = HO.make_pool(field, n)
    lo, hi = HO.slab_pack(hp, n, 4, 4)
    assert np.array_equal(r.lo.cpu().numpy(), lo)
    assert np.array_equal(r.hi.cpu().numpy(), hi)
    r.halo_lo.copy_(r.hi)
    r.halo_hi.copy_(r.lo)
    r.fill(0, r.part.subgrids)
    ref = torch.from_numpy(HO.make_pool(field, n)).to(cuda)
    ops.ghost_fill(ref, n, 4)
    assert torch.equal(r.u, ref)


def test_single_rank_overlapped_iteration(cuda):
    """world 1 through SlabHydro.iteration (interior/boundary schedule on two
    streams; the exchange is the periodic self-copy)."""
    import torch
    grid, n = 64, 8
    field = HO.initial_field(grid)
    (r,) = _ranks(grid, n, 1, field, (1.0, 1.0, 1.0), cuda)
    for _ in range(3):
        r.iteration(overlap=True)
    torch.cuda.synchronize()
    assert np.array_equal(r.owned().cpu().numpy(),
                          HO.reference_step(field, (1.0, 1.0, 1.0)))
