"""PPM reconstruction (north_star's scheme; UNPINNED — the reference has
minmod only).  CPU: the oracle satisfies the method's defining
properties.  GPU: the sm_100a kernel equals the oracle bit for bit."""

import numpy as np
import pytest

from oracle import hydro_oracle as HO
from oracle import ppm_oracle as PO


def _pool(field, n):
    p = HO.make_pool(field, n)
    HO.exchange_ghosts_pool(p, n, field.shape[0] // n)
    return p


def test_constant_field_preserved():
    p = _pool(np.full((16, 16, 16), 2.5), 8)
    um, up = PO.reconstruct_ppm_batch(p, 8)
    assert bool((um == 2.5).all()) and bool((up == 2.5).all())


def test_linear_profile_reproduced():
    """PPM is exact for linear data away from the periodic kink: interior
    faces equal the interface midpoints to rounding."""
    g, n = 32, 8
    x = np.arange(g, dtype=float)
    field = np.broadcast_to((1.0 + 0.01 * x)[:, None, None], (g, g, g)).copy()
    p = _pool(field, n)
    um, up = PO.reconstruct_ppm_batch(p, n)
    # sub-grid (1,1,1) is far from the wrap in x; cube cells 1..n
    sid = (1 * 4 + 1) * 4 + 1
    xs = 8 + np.arange(-1, 9)            # global x of cube cells 0..9
    exp_up = 1.0 + 0.01 * (xs + 0.5)
    exp_um = 1.0 + 0.01 * (xs - 0.5)
    np.testing.assert_allclose(up[sid, 0, :, 3, 3], exp_up, rtol=1e-14)
    np.testing.assert_allclose(um[sid, 0, :, 3, 3], exp_um, rtol=1e-14)
    # y and z faces of an x-only profile are flat
    assert np.array_equal(up[sid, 1], um[sid, 1])


def test_states_bounded_by_neighbours():
    """CW84 limiting: face states never leave the range of the cell and its
    two neighbours (no new extrema)."""
    f = HO.stress_field(16)
    n = 8
    p = _pool(f, n)
    um, up = PO.reconstruct_ppm_batch(p, n)
    for axis in range(3):
        u = PO._shift(p, n, axis, 0)
        lo = np.minimum(np.minimum(PO._shift(p, n, axis, -1), u),
                        PO._shift(p, n, axis, 1))
        hi = np.maximum(np.maximum(PO._shift(p, n, axis, -1), u),
                        PO._shift(p, n, axis, 1))
        assert bool((um[:, axis] >= lo).all() and (um[:, axis] <= hi).all())
        assert bool((up[:, axis] >= lo).all() and (up[:, axis] <= hi).all())


def test_ppm_sharper_than_minmod_on_smooth_data():
    """On a smooth bump PPM's face states are closer to the exact interface
    values than minmod's (the point of the higher-order scheme)."""
    g, n = 32, 8
    x = (np.arange(g) + 0.5) / g
    f1 = np.sin(2 * np.pi * x)
    field = np.broadcast_to(f1[:, None, None], (g, g, g)).copy()
    p = _pool(field, n)
    um_p, up_p = PO.reconstruct_ppm_batch(p, n)
    um_m, up_m = HO.reconstruct_batch(p, n)
    # cube cell c of sub-grid bx=1 is global cell 7 + c; its +1/2 face
    exact = np.sin(2 * np.pi * ((np.arange(10) + 8.0) / g))
    sid = (1 * 4 + 1) * 4 + 1
    # away from the extremum at x = 1/4 (cube cells 0-1, where both limiters
    # flatten), PPM is about an order of magnitude more accurate
    err_p = np.abs(up_p[sid, 0, 2:, 3, 3] - exact[2:]).max()
    err_m = np.abs(up_m[sid, 0, 2:, 3, 3] - exact[2:]).max()
    assert err_p < 0.2 * err_m


@pytest.mark.gpu
@pytest.mark.parametrize("grid,n,field,vel,form", [
    (16, 8, "stress", (1.0, 1.0, 1.0), 0),
    (32, 8, "blast", (-1.0, 0.5, -0.25), 0),
    (32, 8, "sod", (0.7, -1.3, 0.0), 1),
    (32, 16, "stress", (-0.3, 0.2, 0.9), 0),
    (32, 16, "blast", (1.0, 1.0, 1.0), 1),
    (16, 8, "stress", (-0.4, -0.9, -1.2), 1),
    (16, 8, "stress", (0.5, 0.0, 1.5), 1)])
def test_gpu_ppm_matches_oracle(cuda, grid, n, field, vel, form):
    import torch
    from paper_2210_06438_b200 import ops
    f = {"stress": HO.stress_field, "blast": HO.initial_field,
         "sod": HO.sod_field}[field](grid)
    hp = _pool(f, n)
    pool = torch.from_numpy(hp).to(cuda)
    S, c = pool.shape[0], n + 2
    um, up, F = (torch.full((S, 3, c, c, c), float("nan"),
                            dtype=torch.float64, device=cuda)
                 for _ in range(3))
    ops.recon_flux(pool, n, vel, um, up, F, flux_form=form,
                   reconstruction="ppm")
    oum, oup = PO.reconstruct_ppm_batch(hp, n)
    oF = HO.flux_kt_batch(oum, oup, vel) if form else \
        HO.flux_batch(oum, oup, vel)
    assert np.array_equal(um.cpu().numpy(), oum)
    assert np.array_equal(up.cpu().numpy(), oup)
    assert np.array_equal(F.cpu().numpy(), oF)
