"""The reference's mini-app tests (test_hydro.py:102-199) against the
device-resident HydroSim mirror: every execution path (serial visits, fused
teams over several executors, any decomposition) must reproduce the
reference's whole-grid result bit for bit (golden digests recorded from the
reference's reference_step)."""

import numpy as np
import pytest

from oracle import hydro_oracle as HO

pytestmark = pytest.mark.gpu


def run_sim(n, grid, steps, executors=1, max_team=1, field=None,
            velocity=(1.0, 1.0, 1.0), poison=False, id_ring=None,
            engine="python"):
    from paper_2210_06438_b200.device import CudaDevice
    from paper_2210_06438_b200.executorpool import ExecutorPool
    from paper_2210_06438_b200.hydro import HydroSim, driver, make_state
    from paper_2210_06438_b200.sched import Scheduler, SchedulerConfig
    sched = Scheduler(SchedulerConfig(worker_count=32))
    if field is None:
        field = HO.initial_field(grid)
    state = make_state(n, grid, field=field)
    device = CudaDevice(sched)
    pool = ExecutorPool(sched, device, executors)
    sim = HydroSim(sched, state, pool, max_team=max_team, velocity=velocity,
                   engine=engine)
    if poison:
        sim.scratch_pool.poison()
    if id_ring is not None:   # a tiny ring: wraps every few launches
        from paper_2210_06438_b200.hydro.step import _IdRing
        sim._ids_ring = _IdRing([device.stream(e.stream_id)
                                 for e in pool.executors], size=id_ring)
    sched.spawn(lambda: driver(sim, steps), label="driver")
    sched.run()
    return state, sim, device


def _golden(hydro_golden, name):
    return next(c for c in hydro_golden["cases"] if c["name"] == name)


def test_device_path_matches_reference(cuda, hydro_golden):
    from paper_2210_06438_b200.hydro import assemble
    case = _golden(hydro_golden, "blast16_n8_v111")
    state, sim, device = run_sim(8, 16, steps=2, executors=1, max_team=1)
    assert HO.digest(assemble(state)) == case["reference_step_2"]
    # test_hydro.py:153-160 accounting: 8 tasks x 3 iterations x 5 visits
    visits = len(state.blocks) * 3 * 5
    assert visits == 120
    assert device.kernels_enqueued == 2 * visits
    assert device.copies_enqueued == 2 * 2 * visits
    assert sim.buffers.stats().outstanding == 0


def test_fused_teams_match_reference(cuda, hydro_golden):
    from paper_2210_06438_b200.hydro import assemble
    case = _golden(hydro_golden, "blast16_n8_v111")
    state, sim, device = run_sim(8, 16, steps=2, executors=4, max_team=8)
    assert HO.digest(assemble(state)) == case["reference_step_2"]
    assert all(r.stats().violations == 0 for r in sim.regions.values())
    total = sum(sz * c for r in sim.regions.values()
                for sz, c in r.stats().size_histogram.items())
    assert total == 8 * 3 * 2 * 5


def test_negative_velocity_path(cuda, hydro_golden):
    from paper_2210_06438_b200.hydro import assemble
    case = _golden(hydro_golden, "stress16_n8_vneg")
    state, _, _ = run_sim(8, 16, steps=1, executors=2, max_team=4,
                          field=HO.stress_field(16),
                          velocity=tuple(case["velocity"]))
    assert HO.digest(assemble(state)) == case["reference_step_1"]


def test_decomposition_invariance(cuda):
    from paper_2210_06438_b200.hydro import assemble
    coarse, _, _ = run_sim(16, 16, steps=2, executors=1)
    fine, _, _ = run_sim(8, 16, steps=2, executors=2, max_team=4)
    assert np.array_equal(assemble(coarse), assemble(fine))


def test_poisoned_scratch_is_harmless(cuda, hydro_golden):
    from paper_2210_06438_b200.hydro import assemble
    case = _golden(hydro_golden, "blast16_n8_v111")
    state, _, _ = run_sim(8, 16, steps=1, executors=1, poison=True)
    assert HO.digest(assemble(state)) == case["reference_step_1"]


def test_uniform_field_is_fixed_point_and_mass(cuda):
    from paper_2210_06438_b200.hydro import assemble
    field = np.full((16, 16, 16), 2.5)
    state, _, _ = run_sim(8, 16, steps=2, field=field)
    assert np.array_equal(assemble(state), field)
    f = HO.initial_field(16)
    state, _, _ = run_sim(8, 16, steps=2, executors=2, max_team=2, field=f)
    assert abs(assemble(state).sum() - f.sum()) <= 1e-12 * f.sum()


def test_reduction_reports_advection_speed(cuda):
    _, sim, _ = run_sim(8, 8, steps=1)
    assert float(sim.scratch[(0, 0, 0)]["reduce_out"][0]) == 1.0


def test_dump_and_load_roundtrip(cuda, tmp_path):
    from paper_2210_06438_b200.hydro import assemble, dump_state, load_state
    state, _, _ = run_sim(8, 16, steps=1)
    path = str(tmp_path / "checkpoint.npz")
    dump_state(state, path)
    loaded = load_state(path)
    assert (loaded.n, loaded.grid_n, loaded.steps_taken, loaded.time) == \
        (state.n, state.grid_n, state.steps_taken, state.time)
    assert np.array_equal(assemble(loaded), assemble(state))


def test_per_subgrid_bodies_match_reference(cuda, hydro_golden):
    """The per-block body API (kernels.py signatures) on device tensors."""
    import torch
    from paper_2210_06438_b200.hydro import (exchange_ghosts, flux_body,
                                             make_scratch, make_state,
                                             prep_body, reconstruct_body,
                                             reduce_body, update_body)
    case = _golden(hydro_golden, "stress16_n8_vmix")
    vel = tuple(case["velocity"])
    state = make_state(8, 16, field=HO.stress_field(16))
    for b in state.blocks:
        exchange_ghosts(state, b)
    for g, b in enumerate(state.blocks):
        sc = make_scratch(8)
        prep_body(state.u[b], sc)
        reconstruct_body(sc, 8)
        flux_body(sc, 8, vel)
        reduce_body(sc, vel)
        update_body(state.u[b], state.u_next[b], sc, 8, case["dt_dx"])
        torch.cuda.synchronize()
        per = case["per_subgrid"]
        assert HO.digest(sc["w"].cpu().numpy()) == per["w"][g]
        assert HO.digest(sc["um"].cpu().numpy()) == per["um"][g]
        assert HO.digest(sc["F"].cpu().numpy()) == per["F"][g]
        own = state.u_next[b][3:11, 3:11, 3:11].cpu().numpy()
        assert HO.digest(own) == per["next"][g]
        assert float(sc["reduce_out"][0]) == per["reduce"][g]


def test_ghost_exchange_matches_periodic_window(cuda):
    from paper_2210_06438_b200.hydro import exchange_ghosts, make_state
    field = HO.initial_field(16)
    state = make_state(8, 16, field=field)
    assert np.isnan(float(state.u[(0, 0, 0)][0, 0, 0]))
    exchange_ghosts(state, (0, 0, 0))
    idx = np.arange(-3, 8 + 3) % 16
    assert np.array_equal(state.u[(0, 0, 0)].cpu().numpy(),
                          field[np.ix_(idx, idx, idx)])


def test_team_id_ring_wraps(cuda, hydro_golden):
    """Team ids go to the kernels through a pinned ring read zero-copy;
    a 64-entry ring wraps every few teams and must stay fenced."""
    from paper_2210_06438_b200.hydro import assemble
    case = _golden(hydro_golden, "blast16_n8_v111")
    state, sim, _ = run_sim(8, 16, steps=2, executors=4, max_team=8,
                            id_ring=64)
    assert HO.digest(assemble(state)) == case["reference_step_2"]
    assert sim._ids_ring.size == 64


def test_bitwise_reproducibility_matrix(cuda):
    """The reference's acceptance criterion 2 (test_acceptance.py:119-132)
    on the B200: the field after the run is bit-identical to the whole-grid
    reference for every executors x cap x policy cell (16^3 sub-grids) and
    for the finer 8^3 decomposition.  3 steps instead of the reference's 15
    (the per-task path is host-bound; every cell still runs 9 iterations
    through real team formation, launches and copies).  executors = 0 (the
    reference's CPU path) does not exist here."""
    from paper_2210_06438_b200.device import CudaDevice
    from paper_2210_06438_b200.executorpool import ExecutorPool
    from paper_2210_06438_b200.hydro import HydroSim, assemble, driver, make_state
    from paper_2210_06438_b200.sched import Scheduler, SchedulerConfig
    grid, steps = 64, 3
    ref = HO.reference_step(HO.initial_field(grid), iterations=3 * steps)

    def field_after(n, executors, cap, policy):
        sched = Scheduler(SchedulerConfig(worker_count=32))
        state = make_state(n, grid)
        pool = ExecutorPool(sched, CudaDevice(sched), executors, policy)
        sim = HydroSim(sched, state, pool, max_team=cap)
        sched.spawn(lambda: driver(sim, steps), label="driver")
        sched.run()
        return assemble(state)

    bad = [(e, c, p) for e in (1, 4, 32, 128) for c in (1, 8, 128)
           for p in ("round_robin", "load_balanced")
           if not np.array_equal(field_after(16, e, c, p), ref)]
    if not np.array_equal(field_after(8, 32, 8, "load_balanced"), ref):
        bad.append((8, 32, 8, "load_balanced"))
    assert not bad, bad


# ---------------------------------------------------------------- native
# The same task iteration in the C++ engine (hydro/engine.py), under the
# same tf_region / tf_team rules: same whole-grid results, same counting
# identities, every lease back in the pool, and teams that actually form.

@pytest.mark.parametrize("executors,cap", [(1, 1), (4, 8), (2, 3)])
def test_native_engine_matches_reference(cuda, hydro_golden, executors, cap):
    from paper_2210_06438_b200.hydro import assemble
    case = _golden(hydro_golden, "blast16_n8_v111")
    state, sim, device = run_sim(8, 16, steps=2, executors=executors,
                                 max_team=cap, engine="native")
    assert sim.native is not None
    assert HO.digest(assemble(state)) == case["reference_step_2"]
    c = sim.native.counters()
    assert c["outstanding"] == 0
    hist = {}
    for r in sim.regions.values():
        st = r.stats()
        assert st.violations == 0 and max(st.size_histogram) <= cap
        for k, v in st.size_histogram.items():
            hist[k] = hist.get(k, 0) + v
    # every task visits every region once per iteration (test_hydro.py:
    # 153-160): 8 tasks x 3 iterations x 2 steps x 5 regions
    assert sum(k * v for k, v in hist.items()) == 8 * 3 * 2 * 5
    teams = sum(hist.values())
    assert device.kernels_enqueued == teams
    assert device.copies_enqueued == 2 * teams
    if cap == 1:
        assert device.kernels_enqueued == 2 * 120


def test_native_engine_negative_velocity(cuda, hydro_golden):
    from paper_2210_06438_b200.hydro import assemble
    case = _golden(hydro_golden, "stress16_n8_vneg")
    state, _, _ = run_sim(8, 16, steps=1, executors=2, max_team=4,
                          field=HO.stress_field(16),
                          velocity=tuple(case["velocity"]), engine="native")
    assert HO.digest(assemble(state)) == case["reference_step_1"]


def test_native_engine_forms_teams_config2(cuda):
    """Config 2 (4096 sub-grids) through HydroSim + driver at A = 64: the
    arrivals outpace the device, so most teams close at the cap (the Python
    per-task path closes nearly all of them solo).  The reference's own
    simulated A100 forms a mean team of 23.3 here (probe P4); the
    bar is that, and the field is still the whole-grid reference's."""
    from paper_2210_06438_b200.hydro import assemble
    f = HO.sod_field(128)
    state, sim, _ = run_sim(8, 128, steps=1, executors=1, max_team=64,
                            field=f, engine="native")
    hist = {}
    for r in sim.regions.values():
        for k, v in r.stats().size_histogram.items():
            hist[k] = hist.get(k, 0) + v
    members = sum(k * v for k, v in hist.items())
    assert members == 4096 * 3 * 5
    assert members / sum(hist.values()) >= 23.3, hist
    assert np.array_equal(assemble(state), HO.reference_step(f))
