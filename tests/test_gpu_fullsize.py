"""Whole-grid parity at the benchmarked sizes (GPU).

The reference pins whole-grid equality with `reference_step`
(/root/reference/pkg/tests/test_hydro.py:116-136, test_acceptance.py:
119-132); these tests do the same for the paths the bench times, at the
size it times them:

* config 5 (262 144 8^3 sub-grids, grid 512, blast): the peer-fused step
  (`PeerSlabFieldIteration`, the cfg5 bench leg), the fused team plan
  (`FieldIteration`) and the materialising pool path (`SlabHydro`: ghost
  fill, recon+flux to HBM, update) — one iteration each, compared bit for
  bit with the oracle's `advect_once` on the whole 512^3 grid;
* config 3 (32 768 sub-grids, grid 256, blast): the A = 128 captured team
  plan writing packed team leases (the config-3 bench leg) — every um / up /
  F value of every sub-grid against the oracle's per-sub-grid bodies, for
  an upwind (a > 0) and a mixed-sign velocity.
"""

import gc

import numpy as np
import pytest

from oracle import hydro_oracle as HO

pytestmark = pytest.mark.gpu

VEL = (1.0, 1.0, 1.0)


def _free():
    import torch
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def cfg5():
    """The config-5 field and its one-iteration oracle result (~20 s)."""
    f = HO.initial_field(512)
    return f, HO.advect_once(f, VEL)


@pytest.mark.parametrize("kernel", ["march", "cols"])
def test_cfg5_peer_fused_step_whole_grid(cuda, cfg5, kernel):
    """The bench's config-5 iteration: the whole-slab march kernel (the
    headline) and the one-CTA-per-sub-grid kernel."""
    import torch
    from paper_2210_06438_b200.field import PeerSlabFieldIteration
    from paper_2210_06438_b200.parallel_halo import SlabPartition
    f, want = cfg5
    r = PeerSlabFieldIteration(SlabPartition(512, 8, 1, 0), f, VEL,
                               device=cuda, kernel=kernel)
    r.iteration()
    torch.cuda.synchronize()
    r.check()
    got = r.owned().cpu().numpy()
    del r
    _free()
    assert np.array_equal(got, want)


def test_cfg5_fused_team_plan_whole_grid(cuda, cfg5):
    import torch
    from paper_2210_06438_b200.field import FieldIteration
    f, want = cfg5
    it = FieldIteration(512, 8, VEL, max_team=128, executors=2, device=cuda)
    it.load(torch.from_numpy(f).to(cuda))
    it.step()
    torch.cuda.synchronize()
    got = it.owned().cpu().numpy()
    del it
    _free()
    assert np.array_equal(got, want)


def test_cfg5_materialising_pool_path_whole_grid(cuda, cfg5):
    """Ghost-filled sub-grid pool, faces materialised in HBM (19 GB), then
    the update: the config-5 `materialising_path` bench leg."""
    import torch
    from paper_2210_06438_b200.parallel_halo import SlabHydro, SlabPartition
    f, want = cfg5
    h = SlabHydro(SlabPartition(512, 8, 1, 0), f, VEL, device=cuda)
    h.iteration(overlap=True)
    torch.cuda.synchronize()
    got = h.owned().cpu().numpy()
    del h
    _free()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("vel", [(1.0, 1.0, 1.0), (-1.0, 0.5, -0.25)])
def test_cfg3_team_plan_every_subgrid(cuda, vel):
    """Config 3 as benchmarked: A = 128, 2 executor branches, outputs in the
    packed team leases (slice order = plan.order); every sub-grid's faces
    and fluxes equal the oracle's."""
    import torch
    from paper_2210_06438_b200 import ops
    from paper_2210_06438_b200.strategy3 import TeamPlan, form_teams
    n, grid = 8, 256
    m = grid // n
    f = HO.initial_field(grid)
    hp = HO.make_pool(f, n)
    HO.exchange_ghosts_pool(hp, n, m)
    pool = torch.from_numpy(HO.make_pool(f, n)).to(cuda)
    ops.ghost_fill(pool, n, m)
    S, c = pool.shape[0], n + 2
    um, up, F = (torch.full((S, 3, c, c, c), float("nan"),
                            dtype=torch.float64, device=cuda)
                 for _ in range(3))
    amax = torch.full((S,), float("nan"), dtype=torch.float64, device=cuda)
    teams = form_teams(range(S), 128, 2)
    plan = TeamPlan(teams, pool, n, vel, um, up, F, 2, amax=amax,
                    team_buffers=True)
    plan.launch()
    torch.cuda.synchronize()
    assert bool((pool.cpu() == torch.from_numpy(hp)).all())
    order = torch.from_numpy(plan.order.astype(np.int64))
    del pool
    oum, oup, oF = HO.recon_flux_batch(hp, n, vel)
    del hp
    # slice i of the packed leases holds sub-grid order[i]
    for got, want in ((um, oum), (up, oup), (F, oF)):
        g = got.cpu()
        w = torch.from_numpy(want)[order]
        assert torch.equal(g, w)
    assert bool((amax.cpu() == max(abs(v) for v in vel)).all())
    del um, up, F, plan
    _free()
