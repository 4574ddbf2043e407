"""The whole-slab march kernel (tf_field_march_f64, csrc/field_march.cu):
one launch per iteration over every sub-grid, warps marching x through
plane boxes, the next field's periodic halos written by the kernel itself.
Bit-identical to the reference's whole-grid integrator (reference.py:24-48
via the oracle's advect_once / reference_step) for every velocity sign
pattern, both column heights, chunk lengths that do and do not divide the
slab, and the peer (multi-GPU) form."""

import numpy as np
import pytest

from oracle import hydro_oracle as HO

pytestmark = pytest.mark.gpu

SIGNED_VELOCITIES = [(1.0, 1.0, 1.0), (-1.0, 0.5, -0.25), (0.7, -1.3, 0.0),
                     (-0.2, -0.9, 1.1), (0.6, 0.8, -1.0), (-0.5, -0.4, -0.3),
                     (0.9, -0.1, -0.7), (-0.0, 1.2, 0.5)]


@pytest.mark.parametrize("vel", SIGNED_VELOCITIES)
@pytest.mark.parametrize("rows4,along_y", [(False, False), (True, False),
                                           (False, True), (True, True)])
def test_march_every_sign(cuda, vel, rows4, along_y):
    """along_y: the warps march y with x rows (TF_MARCH_ALONG_Y)."""
    import torch
    from paper_2210_06438_b200.field import MarchFieldIteration
    f = HO.stress_field(64)
    it = MarchFieldIteration(64, 8, vel, device=cuda, rows4=rows4,
                             along_y=along_y)
    it.load(torch.from_numpy(f).to(cuda))
    for _ in range(3):          # steps 2, 3 read the halos step 1 wrote
        it.step()
    torch.cuda.synchronize()
    assert np.array_equal(it.owned().cpu().numpy(), HO.reference_step(f, vel))


@pytest.mark.parametrize("grid,xc,along_y", [
    (32, 0, False), (32, 5, False), (64, 1, False), (64, 7, False),
    (64, 64, False), (96, 40, False), (128, 0, False),
    (32, 5, True), (64, 1, True), (96, 40, True), (128, 0, True)])
def test_march_chunk_lengths(cuda, grid, xc, along_y):
    """Work items of xc planes (0 = the default: 16, or 8 for few items);
    a last chunk shorter than xc, one-plane chunks, one chunk for the whole
    slab; both march axes."""
    import torch
    from paper_2210_06438_b200.field import MarchFieldIteration
    vel = (-0.6, 1.1, -0.9)
    f = HO.stress_field(grid)
    it = MarchFieldIteration(grid, 8, vel, device=cuda, xc=xc,
                             along_y=along_y)
    it.load(torch.from_numpy(f).to(cuda))
    for _ in range(2):
        it.step()
    torch.cuda.synchronize()
    assert np.array_equal(it.owned().cpu().numpy(),
                          HO.reference_step(f, vel, iterations=2))


@pytest.mark.parametrize("vel", [(1.0, 1.0, 1.0), (-0.6, 1.1, -0.9)])
@pytest.mark.parametrize("along_y", [False, True])
def test_march_writes_the_periodic_halos(cuda, vel, along_y):
    """After one march step the next field's halo faces (one halo
    coordinate: what the 6-point stencil reads) equal what the halo kernels
    make of its owned cells."""
    import torch
    from paper_2210_06438_b200.field import HX, HY, HZ, MarchFieldIteration
    f = HO.stress_field(64)
    it = MarchFieldIteration(64, 8, vel, device=cuda, along_y=along_y)
    it.load(torch.from_numpy(f).to(cuda))
    it.step()
    got = it.field.clone()
    it.halo(True)
    want = it.field.clone()
    torch.cuda.synchronize()
    px, py, pz = got.shape
    hx = (np.arange(px) < HX) | (np.arange(px) >= px - HX)
    hy = (np.arange(py) < HY) | (np.arange(py) >= py - HY)
    hz = (np.arange(pz) < HZ) | (np.arange(pz) >= pz - HZ)
    nh = hx[:, None, None].astype(int) + hy[None, :, None] + hz[None, None, :]
    face = nh <= 1
    assert np.array_equal(got.cpu().numpy()[face], want.cpu().numpy()[face])


def test_march_sod_and_blast(cuda):
    import torch
    from paper_2210_06438_b200.field import MarchFieldIteration
    for f in (HO.sod_field(64), HO.initial_field(64)):
        it = MarchFieldIteration(64, 8, device=cuda)
        it.load(torch.from_numpy(f).to(cuda))
        for _ in range(3):
            it.step()
        torch.cuda.synchronize()
        assert np.array_equal(it.owned().cpu().numpy(), HO.reference_step(f))


@pytest.mark.parametrize("kernel,overlap,axis", [
    ("march", False, "x"), ("march", True, "x"), ("march", False, "y"),
    ("march", True, "y"), ("cols", None, "x")])
@pytest.mark.parametrize("vel", [(-1.0, 0.5, -0.25), (1.0, 1.0, 1.0)])
def test_peer_single_rank_both_kernels(cuda, kernel, overlap, axis, vel):
    """The peer path on one rank (its own ring neighbour), both kernels;
    the march along x and along y, with and without the barrier overlap
    (the march a programmatic dependent of the barrier, the items on the
    x faces waiting for it)."""
    import torch
    from paper_2210_06438_b200.field import PeerSlabFieldIteration
    from paper_2210_06438_b200.parallel_halo import SlabPartition
    f = HO.stress_field(64)
    r = PeerSlabFieldIteration(SlabPartition(64, 8, 1, 0), f, vel,
                               device=cuda, kernel=kernel,
                               overlap_barrier=overlap, march_axis=axis)
    assert r.kernel == kernel and r.march_axis == axis
    for _ in range(3):
        r.iteration()
    torch.cuda.synchronize()
    r.check()
    assert np.array_equal(r.owned().cpu().numpy(), HO.reference_step(f, vel))


def test_march_rejects_bad_shapes(cuda, native_lib):
    import torch
    from paper_2210_06438_b200 import _lib
    P = torch.zeros((12, 20, 24), dtype=torch.float64, device=cuda)
    Q = torch.zeros_like(P)
    s = torch.cuda.current_stream().cuda_stream
    # Gz = 16 is not a multiple of the 32-lane column
    assert native_lib.tf_field_march_f64(P.data_ptr(), 8, 16, 16, 1.0, 1.0,
                                         1.0, 0.1, Q.data_ptr(), None, None, 0,
                                         0, None, s) == _lib.TF_E_INVALID
    # in == out
    assert native_lib.tf_field_march_f64(P.data_ptr(), 8, 32, 32, 1.0, 1.0,
                                         1.0, 0.1, P.data_ptr(), None, None, 0,
                                         0, None, s) == _lib.TF_E_INVALID
    # HALO_X together with peer pointers
    assert native_lib.tf_field_march_f64(
        P.data_ptr(), 8, 32, 32, 1.0, 1.0, 1.0, 0.1, Q.data_ptr(),
        Q.data_ptr(), None, _lib.TF_STEP_HALO_X, 0, None, s) == _lib.TF_E_INVALID
    # along y: needs the y/z halos and both x halo destinations, X % R == 0
    ym = _lib.TF_MARCH_ALONG_Y
    assert native_lib.tf_field_march_f64(
        P.data_ptr(), 8, 32, 32, 1.0, 1.0, 1.0, 0.1, Q.data_ptr(), None,
        None, ym | _lib.TF_STEP_HALO_X, 0, None, s) == _lib.TF_E_INVALID
    assert native_lib.tf_field_march_f64(
        P.data_ptr(), 8, 32, 32, 1.0, 1.0, 1.0, 0.1, Q.data_ptr(),
        Q.data_ptr(), None, ym | _lib.TF_STEP_HALO_YZ, 0, None,
        s) == _lib.TF_E_INVALID
    assert native_lib.tf_field_march_f64(
        P.data_ptr(), 6, 32, 32, 1.0, 1.0, 1.0, 0.1, Q.data_ptr(), None,
        None, ym | _lib.TF_STEP_HALO_YZ | _lib.TF_STEP_HALO_X, 0, None,
        s) == _lib.TF_E_INVALID
