"""GPU parity: the sm_100a kernels, called through the C ABI, against the
golden vectors recorded from the reference and against the CPU oracle.

Bar: bit-exact (sha256 of the FP64 bytes) for reconstruct / flux / update /
ghost fill / prep / reduce; the optional Kurganov-Tadmor flux form within
1e-12 relative of the reference upwind flux (north_star tolerance).
"""

import numpy as np
import pytest

from oracle import hydro_oracle as HO

pytestmark = pytest.mark.gpu

FIELDS = {"blast": HO.initial_field, "sod": HO.sod_field,
          "stress": HO.stress_field}


def _torch():
    import torch
    return torch


def device_pool(field, n, dev):
    torch = _torch()
    return torch.from_numpy(HO.make_pool(field, n)).to(dev)


def faces(S, n, dev, fill=np.nan):
    torch = _torch()
    c = n + 2
    return torch.full((S, 3, c, c, c), fill, dtype=torch.float64, device=dev)


def per_digests(t):
    a = t.cpu().numpy()
    return [HO.digest(a[i]) for i in range(a.shape[0])]


@pytest.fixture(scope="module")
def cases(hydro_golden):
    return hydro_golden["cases"]


def test_ghost_fill_bit_exact(cuda, cases):
    from paper_2210_06438_b200 import ops
    for case in cases:
        n, g = case["n"], case["grid"]
        pool = device_pool(FIELDS[case["field"]](g), n, cuda)
        ops.ghost_fill(pool, n, g // n)
        assert per_digests(pool) == case["per_subgrid"]["w"], case["name"]


def test_recon_flux_bit_exact_all_cases(cuda, cases):
    """Fused kernel == reconstruct_body + flux_body of the reference."""
    from paper_2210_06438_b200 import ops
    torch = _torch()
    for case in cases:
        n, g = case["n"], case["grid"]
        vel = tuple(case["velocity"])
        pool = device_pool(FIELDS[case["field"]](g), n, cuda)
        ops.ghost_fill(pool, n, g // n)
        S = pool.shape[0]
        um, up, F = faces(S, n, cuda), faces(S, n, cuda), faces(S, n, cuda)
        amax = torch.full((S,), np.nan, dtype=torch.float64, device=cuda)
        ops.recon_flux(pool, n, vel, um, up, F, out_mode=1, amax=amax)
        torch.cuda.synchronize()
        per = case["per_subgrid"]
        assert per_digests(um) == per["um"], case["name"]
        assert per_digests(up) == per["up"], case["name"]
        assert per_digests(F) == per["F"], case["name"]
        assert amax.cpu().tolist() == per["reduce"]


def test_team_launch_strided_members(cuda, cases):
    """A strided team through by-value kernel-parameter ids, into
    the team buffer layout (slice s owns [s*len, (s+1)*len))."""
    from paper_2210_06438_b200 import ops
    for case in cases:
        n, g = case["n"], case["grid"]
        pool = device_pool(FIELDS[case["field"]](g), n, cuda)
        ops.ghost_fill(pool, n, g // n)
        S = pool.shape[0]
        ids = list(range(S - 1, -1, -3)) + [0, 0]   # strided, duplicates ok
        T = len(ids)
        um, up, F = faces(T, n, cuda), faces(T, n, cuda), faces(T, n, cuda)
        ops.recon_flux_team(pool, n, tuple(case["velocity"]), ids, um, up, F,
                            out_mode=0)
        per = case["per_subgrid"]
        assert per_digests(F) == [per["F"][i] for i in ids], case["name"]
        assert per_digests(um) == [per["um"][i] for i in ids], case["name"]
        assert per_digests(up) == [per["up"][i] for i in ids], case["name"]


def test_device_ids_gather(cuda, cases):
    from paper_2210_06438_b200 import ops
    torch = _torch()
    case = cases[4]
    n, g = case["n"], case["grid"]
    pool = device_pool(FIELDS[case["field"]](g), n, cuda)
    ops.ghost_fill(pool, n, g // n)
    S = pool.shape[0]
    perm = np.random.default_rng(7).permutation(S).astype(np.int32)
    ids = torch.from_numpy(perm).to(cuda)
    um, up, F = faces(S, n, cuda), faces(S, n, cuda), faces(S, n, cuda)
    ops.recon_flux(pool, n, tuple(case["velocity"]), um, up, F, ids=ids,
                   out_mode=0)
    assert per_digests(F) == [case["per_subgrid"]["F"][i] for i in perm]


def test_two_kernel_mode_bit_exact(cuda, cases):
    """reconstruct_body and flux_body as separate batched kernels."""
    from paper_2210_06438_b200 import ops
    for case in cases:
        n, g = case["n"], case["grid"]
        pool = device_pool(FIELDS[case["field"]](g), n, cuda)
        ops.ghost_fill(pool, n, g // n)
        S = pool.shape[0]
        um, up, F = faces(S, n, cuda), faces(S, n, cuda), faces(S, n, cuda)
        ops.reconstruct(pool, n, um, up)
        ops.flux(n, tuple(case["velocity"]), um, up, F)
        per = case["per_subgrid"]
        assert per_digests(um) == per["um"], case["name"]
        assert per_digests(F) == per["F"], case["name"]


def test_prep_reduce_update_bit_exact(cuda, cases):
    from paper_2210_06438_b200 import ops
    torch = _torch()
    for case in cases:
        n, g = case["n"], case["grid"]
        vel = tuple(case["velocity"])
        pool = device_pool(FIELDS[case["field"]](g), n, cuda)
        ops.ghost_fill(pool, n, g // n)
        S = pool.shape[0]
        w = torch.full_like(pool, np.nan)
        ops.prep(pool, n, w)
        assert per_digests(w) == case["per_subgrid"]["w"]
        red = torch.full((S,), np.nan, dtype=torch.float64, device=cuda)
        ops.reduce(vel, red)
        assert red.cpu().tolist() == case["per_subgrid"]["reduce"]
        um, up, F = faces(S, n, cuda), faces(S, n, cuda), faces(S, n, cuda)
        ops.recon_flux(pool, n, vel, um, up, F)
        nxt = torch.full_like(pool, np.nan)
        ops.update(pool, n, F, case["dt_dx"], nxt)
        own = nxt[:, 3:3 + n, 3:3 + n, 3:3 + n].contiguous()
        assert per_digests(own) == case["per_subgrid"]["next"], case["name"]
        # update writes the owned region only (kernels.py:102)
        ghost = nxt.clone()
        ghost[:, 3:3 + n, 3:3 + n, 3:3 + n] = 0.0
        assert torch.isnan(ghost).sum().item() == S * HO.ghost_cells(n)


def test_kt_flux_form_within_tolerance(cuda, cases):
    from paper_2210_06438_b200 import ops
    for case in cases:
        n, g = case["n"], case["grid"]
        vel = tuple(case["velocity"])
        field = FIELDS[case["field"]](g)
        pool = device_pool(field, n, cuda)
        ops.ghost_fill(pool, n, g // n)
        S = pool.shape[0]
        um, up, F = faces(S, n, cuda), faces(S, n, cuda), faces(S, n, cuda)
        ops.recon_flux(pool, n, vel, um, up, F, flux_form=1)
        hp = HO.make_pool(field, n)
        HO.exchange_ghosts_pool(hp, n, g // n)
        oum, oup, oF = HO.recon_flux_batch(hp, n, vel)
        got = F.cpu().numpy()
        # identical op order to the numpy KT restatement -> bit-exact
        assert np.array_equal(got, HO.flux_kt_batch(oum, oup, vel))
        # and within the north_star tolerance of the reference upwind flux
        np.testing.assert_allclose(got, oF, rtol=1e-12, atol=1e-300)


def test_outputs_fully_overwritten_on_poisoned_buffers(cuda, cases):
    """test_hydro.py:145-150: recycled buffers are never read stale."""
    from paper_2210_06438_b200 import ops
    torch = _torch()
    case = cases[1]
    n, g = case["n"], case["grid"]
    pool = device_pool(FIELDS[case["field"]](g), n, cuda)
    ops.ghost_fill(pool, n, g // n)
    S = pool.shape[0]
    for fill in (np.nan, np.inf, -1e300):
        um, up, F = (faces(S, n, cuda, fill) for _ in range(3))
        ops.recon_flux(pool, n, tuple(case["velocity"]), um, up, F)
        assert per_digests(F) == case["per_subgrid"]["F"]
        assert torch.isfinite(um).all() and torch.isfinite(up).all()


def test_empty_and_invalid_launches(cuda):
    from paper_2210_06438_b200 import ops
    from paper_2210_06438_b200.errors import ValidationError
    torch = _torch()
    pool = torch.zeros((2, 14, 14, 14), dtype=torch.float64, device=cuda)
    um = faces(2, 8, cuda)
    ops.recon_flux(pool, 8, (1, 1, 1), um, um.clone(), um.clone(),
                   ids=torch.zeros(0, dtype=torch.int32, device=cuda))
    with pytest.raises(ValidationError):
        ops.recon_flux(pool, 10, (1, 1, 1), um, um, um)
    with pytest.raises(Exception):
        ops.recon_flux_team(pool, 8, (1, 1, 1), [5], um, um, um)  # id >= S
    with pytest.raises(ValidationError):
        ops.recon_flux_team(pool, 8, (1, 1, 1), [0] * 129, um, um, um)


@pytest.mark.parametrize("grid,field", [(128, "sod"), (128, "stress")])
def test_config2_full_size_against_oracle(cuda, grid, field):
    """BASELINE config 2 (4096 8^3 sub-grids) at full size, bit-exact."""
    from paper_2210_06438_b200 import ops
    torch = _torch()
    n = 8
    f = FIELDS[field](grid)
    hp = HO.make_pool(f, n)
    HO.exchange_ghosts_pool(hp, n, grid // n)
    pool = torch.from_numpy(HO.make_pool(f, n)).to(cuda)
    ops.ghost_fill(pool, n, grid // n)
    assert HO.digest(pool.cpu().numpy()) == HO.digest(hp)
    S = pool.shape[0]
    for vel in ((1.0, 1.0, 1.0), (-1.0, 0.5, -0.25)):
        um, up, F = faces(S, n, cuda), faces(S, n, cuda), faces(S, n, cuda)
        ops.recon_flux(pool, n, vel, um, up, F)
        oum, oup, oF = HO.recon_flux_batch(hp, n, vel)
        assert np.array_equal(F.cpu().numpy(), oF)
        assert np.array_equal(um.cpu().numpy(), oum)
        assert np.array_equal(up.cpu().numpy(), oup)


def test_config3_size_independent_properties(cuda):
    """32768 sub-grids (config 3): uniform field is a fixed point of the
    faces (sigma = 0 -> um = up = u, F = a u), the per-sub-grid digest of a
    deterministic stride sample matches the oracle, and translation
    covariance: shifting the field by one sub-grid permutes the outputs."""
    from paper_2210_06438_b200 import ops
    torch = _torch()
    n, grid = 8, 256
    m = grid // n
    S = m ** 3
    pool = torch.full((S, 14, 14, 14), 2.5, dtype=torch.float64, device=cuda)
    um, up, F = faces(S, n, cuda), faces(S, n, cuda), faces(S, n, cuda)
    ops.recon_flux(pool, n, (1.0, 1.0, 1.0), um, up, F)
    assert bool((um == 2.5).all()) and bool((up == 2.5).all())
    assert bool((F == 2.5).all())
    f = HO.initial_field(grid)
    pool = torch.from_numpy(HO.make_pool(f, n)).to(cuda)
    ops.ghost_fill(pool, n, m)
    ops.recon_flux(pool, n, (1.0, 1.0, 1.0), um, up, F)
    sample = np.arange(0, S, 97)
    hp = HO.make_pool(f, n)
    HO.exchange_ghosts_pool(hp, n, m, ids=sample)
    _, _, oF = HO.recon_flux_batch(hp, n, (1.0, 1.0, 1.0), ids=sample)
    got = F[torch.from_numpy(sample).to(cuda)].cpu().numpy()
    assert np.array_equal(got, oF)
    # translation by one sub-grid along x
    f2 = np.roll(f, -n, axis=0)
    pool2 = torch.from_numpy(HO.make_pool(f2, n)).to(cuda)
    ops.ghost_fill(pool2, n, m)
    F2 = faces(S, n, cuda)
    ops.recon_flux(pool2, n, (1.0, 1.0, 1.0), um, up, F2)
    shift = torch.arange(S, device=cuda).reshape(m, m, m).roll(-1, 0) \
        .reshape(-1)
    assert torch.equal(F2, F[shift])
