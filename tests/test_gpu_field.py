"""The fused full iteration on a padded global field (SURVEY §8 f #2) is
bit-identical to the reference's whole-grid integrator, through team plans,
the host round trip, and slab partitions (virtual ranks on one GPU)."""

import numpy as np
import pytest

from oracle import hydro_oracle as HO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("grid,n,vel,A,E", [
    (16, 8, (1.0, 1.0, 1.0), 1, 1),
    (32, 8, (-1.0, 0.5, -0.25), 16, 4),
    (64, 8, (0.7, -1.3, 0.0), 128, 4),
    (64, 16, (1.0, 1.0, 1.0), 8, 2),
    (64, 16, (-0.3, -0.2, 0.9), 64, 4)])
def test_field_iteration_matches_reference(cuda, grid, n, vel, A, E):
    import torch
    from paper_2210_06438_b200.field import FieldIteration
    f = HO.stress_field(grid)
    it = FieldIteration(grid, n, vel, max_team=A, executors=E)
    it.load(torch.from_numpy(f).to(cuda))
    for _ in range(3):
        it.step()
    torch.cuda.synchronize()
    assert np.array_equal(it.owned().cpu().numpy(), HO.reference_step(f, vel))


SIGNED_VELOCITIES = [(1.0, 1.0, 1.0), (-1.0, 0.5, -0.25), (0.7, -1.3, 0.0),
                     (-0.2, -0.9, 1.1), (0.6, 0.8, -1.0), (-0.5, -0.4, -0.3),
                     (0.9, -0.1, -0.7), (-0.0, 1.2, 0.5)]


@pytest.mark.parametrize("vel", SIGNED_VELOCITIES)
def test_field_step_one_large_launch(cuda, vel):
    """One launch over >= 4096 sub-grids takes the one-thread-per-column
    kernel shape (k_step_cols8s<8>); team-sized launches take <4>.  Both
    bit-identical, every sign combination of the velocity (the swizzled box
    origin shifts against the flow)."""
    import torch
    from paper_2210_06438_b200.field import FieldIteration
    f = HO.stress_field(128)
    it = FieldIteration(128, 8, vel, max_team=128, executors=1)
    it.load(torch.from_numpy(f).to(cuda))
    for _ in range(3):
        it.halo(True)
        it.step_ids(None, it.S)      # one launch, 4096 sub-grids
        it.swap()
    torch.cuda.synchronize()
    assert np.array_equal(it.owned().cpu().numpy(), HO.reference_step(f, vel))


@pytest.mark.parametrize("vel", SIGNED_VELOCITIES)
def test_field_step_team_launches_every_sign(cuda, vel):
    """Team-sized launches (two threads per column) for all eight velocity
    sign combinations; strided teams so warps see scattered sub-grids."""
    import torch
    from paper_2210_06438_b200.field import FieldIteration
    f = HO.stress_field(64)
    it = FieldIteration(64, 8, vel, max_team=64, executors=3)
    it.load(torch.from_numpy(f).to(cuda))
    for _ in range(3):
        it.step()
    torch.cuda.synchronize()
    assert np.array_equal(it.owned().cpu().numpy(), HO.reference_step(f, vel))


def test_field_iteration_golden(cuda, hydro_golden):
    import torch
    from paper_2210_06438_b200.field import FieldIteration
    case = next(c for c in hydro_golden["cases"]
                if c["name"] == "blast16_n8_v111")
    it = FieldIteration(16, 8, (1.0, 1.0, 1.0), max_team=4, executors=2)
    it.load(torch.from_numpy(HO.initial_field(16)).to(cuda))
    for _ in range(6):
        it.step()
    torch.cuda.synchronize()
    assert HO.digest(it.owned().cpu().numpy()) == case["reference_step_2"]


def test_field_host_roundtrip(cuda):
    import torch
    from paper_2210_06438_b200.field import FieldIteration
    f = HO.initial_field(64)
    it = FieldIteration(64, 8, (1.0, 1.0, 1.0))
    hin = torch.from_numpy(f).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    it.run_host(hin, hout)
    torch.cuda.synchronize()
    assert np.array_equal(hout.numpy(), HO.advect_once(f))


@pytest.mark.parametrize("grid,n,chunks,vel", [
    (64, 8, 8, (1.0, 1.0, 1.0)), (128, 8, 8, (-1.0, 0.5, -0.25)),
    (128, 8, 4, (0.7, -1.3, 0.0)), (128, 16, 8, (1.0, 1.0, 1.0)),
    (32, 8, 8, (1.0, 1.0, 1.0)), (128, 8, 2, (-0.3, 1.0, 0.9)),
    (128, 8, 16, (-1.0, -1.0, 1.0)), (128, 8, [1, 2, 4, 5, 3, 1], (1.0, -0.5, 0.25)),
    (64, 16, [1, 3], (0.5, 1.0, -1.0)), (128, 8, "taper", (1.0, 1.0, 1.0))])
def test_field_host_pipelined(cuda, grid, n, chunks, vel):
    """Chunked, transfer-overlapped host round trip == one reference
    iteration; repeated calls chain correctly."""
    import torch
    from paper_2210_06438_b200.field import FieldIteration
    f = HO.stress_field(grid)
    it = FieldIteration(grid, n, vel, max_team=32, executors=2)
    hin = torch.from_numpy(f).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    it.run_host_pipelined(hin, hout, chunks=chunks)
    torch.cuda.synchronize()
    assert np.array_equal(hout.numpy(), HO.advect_once(f, vel))
    h2 = torch.empty_like(hin).pin_memory()
    it.run_host_pipelined(hout, h2, chunks=chunks)
    torch.cuda.synchronize()
    assert np.array_equal(h2.numpy(),
                          HO.advect_once(HO.advect_once(f, vel), vel))


def test_host_pipeline_graph(cuda):
    import torch
    from paper_2210_06438_b200.field import FieldIteration, HostPipeline
    f = HO.stress_field(128)
    it = FieldIteration(128, 8, (1.0, 1.0, 1.0))
    hin = torch.from_numpy(f).pin_memory()
    hout = torch.full_like(hin, float("nan")).pin_memory()
    pipe = HostPipeline(it, hin, hout, chunks=8)
    hout.fill_(float("nan"))
    pipe.run()
    torch.cuda.synchronize()
    assert np.array_equal(hout.numpy(), HO.advect_once(f))
    hin.copy_(torch.from_numpy(HO.initial_field(128)))   # new input, replay
    pipe.run()
    torch.cuda.synchronize()
    assert np.array_equal(hout.numpy(), HO.advect_once(HO.initial_field(128)))


@pytest.mark.parametrize("world,n,grid,vel", [
    (2, 8, 32, (1.0, 1.0, 1.0)), (4, 8, 64, (-1.0, 0.5, -0.25)),
    (2, 16, 64, (0.7, -1.3, 0.0)), (8, 8, 64, (1.0, 1.0, 1.0))])
def test_slab_field_virtual_ranks(cuda, world, n, grid, vel):
    import torch
    from paper_2210_06438_b200.field import SlabFieldIteration
    from paper_2210_06438_b200.parallel_halo import SlabPartition
    f = HO.stress_field(grid)
    ranks = []
    for r in range(world):
        p = SlabPartition(grid, n, world, r)
        ranks.append(SlabFieldIteration(p, p.slab(f), vel, device=cuda))
    for _ in range(3):
        for r in ranks:
            r.halo(False)
        planes = [r._planes() for r in ranks]
        for k, r in enumerate(ranks):
            p = r.part
            planes[k][2].copy_(planes[p.left][1])    # halo_lo <- left's hi
            planes[k][3].copy_(planes[p.right][0])   # halo_hi <- right's lo
        for r in ranks:
            r.step_ids(None, r.S)
            r.swap()
    torch.cuda.synchronize()
    got = torch.cat([r.owned() for r in ranks]).cpu().numpy()
    assert np.array_equal(got, HO.reference_step(f, vel))


def test_slab_field_single_rank_overlap(cuda):
    import torch
    from paper_2210_06438_b200.field import SlabFieldIteration
    from paper_2210_06438_b200.parallel_halo import SlabPartition
    f = HO.initial_field(64)
    p = SlabPartition(64, 8, 1, 0)
    r = SlabFieldIteration(p, f, (1.0, 1.0, 1.0), device=cuda)
    for _ in range(3):
        r.iteration(overlap=True)
    torch.cuda.synchronize()
    assert np.array_equal(r.owned().cpu().numpy(), HO.reference_step(f))


@pytest.mark.parametrize("vel", [(1.0, 1.0, 1.0), (-0.6, 1.1, -0.9)])
def test_step_kernel_writes_the_periodic_halos(cuda, vel):
    """TF_STEP_HALO_YZ | TF_STEP_HALO_X: a team plan over every sub-grid
    leaves the next field's periodic halo faces exactly as the halo kernels
    would (edges and corners — never read by the 6-point stencil — are
    excluded), and chained steps without halo kernels match the reference."""
    import torch
    from paper_2210_06438_b200.field import HX, HY, HZ, FieldIteration
    f = HO.stress_field(32)
    it = FieldIteration(32, 8, vel, max_team=8, executors=2)
    it.load(torch.from_numpy(f).to(cuda))
    it.step()                     # halo kernels (fresh load), then the plan
    assert it.halo_fresh
    got = it.field.clone()
    it.halo(True)                 # what the halo kernels make of it
    want = it.field.clone()
    torch.cuda.synchronize()
    px, py, pz = got.shape
    ix = np.arange(px)
    iy = np.arange(py)
    iz = np.arange(pz)
    hx = (ix < HX) | (ix >= px - HX)
    hy = (iy < HY) | (iy >= py - HY)
    hz = (iz < HZ) | (iz >= pz - HZ)
    nh = hx[:, None, None].astype(int) + hy[None, :, None] + hz[None, None, :]
    face = nh <= 1                # interior or exactly one halo coordinate
    assert (nh == 1).sum() > 0
    assert np.array_equal(got.cpu().numpy()[face], want.cpu().numpy()[face])
    for _ in range(2):
        it.step()
    torch.cuda.synchronize()
    assert np.array_equal(it.owned().cpu().numpy(),
                          HO.reference_step(f, vel))
