"""Pin the CPU oracle to the reference: every golden vector recorded from the
unmodified reference (tests/golden/make_golden.py) must be reproduced bit
for bit by oracle/hydro_oracle.py and oracle/aggregation_oracle.py."""

import numpy as np
import pytest

from oracle import aggregation_oracle as AO
from oracle import hydro_oracle as HO

FIELDS = {"blast": HO.initial_field, "sod": HO.sod_field,
          "stress": HO.stress_field}


def _case_ids(golden):
    return [c["name"] for c in golden["cases"]]


def _pool_for(case):
    field = FIELDS[case["field"]](case["grid"])
    assert HO.digest(field) == case["field_digest"], "field generator drift"
    n = case["n"]
    pool = HO.make_pool(field, n)
    HO.exchange_ghosts_pool(pool, n, case["grid"] // n)
    return field, pool


def test_minmod_edge_vectors(hydro_golden):
    mm = hydro_golden["minmod"]
    a = np.array([float.fromhex(x) for x in mm["a"]])
    b = np.array([float.fromhex(x) for x in mm["b"]])
    out = HO.minmod(a, b)
    assert [float(x).hex() for x in out] == mm["out"]


def test_per_subgrid_bodies_match_reference(hydro_golden):
    """The per-sub-grid restated bodies (what the CPU baseline times)."""
    for case in hydro_golden["cases"]:
        field, pool = _pool_for(case)
        n, vel = case["n"], tuple(case["velocity"])
        per = case["per_subgrid"]
        nxt = np.full_like(pool[0], np.nan)
        for g in range(pool.shape[0]):
            sc = HO.make_scratch(n)
            HO.prep_body(pool[g], sc)
            HO.reconstruct_body(sc, n)
            HO.flux_body(sc, n, vel)
            HO.reduce_body(sc, vel)
            HO.update_body(pool[g], nxt, sc, n, case["dt_dx"])
            own = nxt[3:3 + n, 3:3 + n, 3:3 + n]
            assert HO.digest(sc["w"]) == per["w"][g], (case["name"], g)
            assert HO.digest(sc["um"]) == per["um"][g], (case["name"], g)
            assert HO.digest(sc["up"]) == per["up"][g], (case["name"], g)
            assert HO.digest(sc["F"]) == per["F"][g], (case["name"], g)
            assert HO.digest(own) == per["next"][g], (case["name"], g)
            assert sc["reduce_out"][0] == per["reduce"][g]


def test_batched_oracle_matches_reference(hydro_golden):
    for case in hydro_golden["cases"]:
        field, pool = _pool_for(case)
        n, vel = case["n"], tuple(case["velocity"])
        um, up, F = HO.recon_flux_batch(pool, n, vel)
        st = case["stacked"]
        assert HO.digest(pool) == st["w"], case["name"]
        assert HO.digest(um) == st["um"], case["name"]
        assert HO.digest(up) == st["up"], case["name"]
        assert HO.digest(F) == st["F"], case["name"]
        nxt = HO.update_batch(pool, F, n, case["dt_dx"])
        assert HO.digest(nxt) == st["next"], case["name"]


def test_whole_grid_reference_step(hydro_golden):
    for case in hydro_golden["cases"]:
        field = FIELDS[case["field"]](case["grid"])
        vel = tuple(case["velocity"])
        one = HO.reference_step(field, vel)
        assert HO.digest(one) == case["reference_step_1"], case["name"]
        assert HO.digest(HO.reference_step(one, vel)) == \
            case["reference_step_2"], case["name"]
        assert HO.digest(HO.reference_step(field, vel, iterations=1)) == \
            case["advect_once"]


def test_staged_iteration_equals_whole_grid(hydro_golden):
    """Staged sub-grid iteration == advect_once (reference.py:5-7)."""
    for case in hydro_golden["cases"]:
        field = FIELDS[case["field"]](case["grid"])
        n, g = case["n"], case["grid"]
        nxt = HO.staged_iteration(HO.make_pool(field, n), n, g // n,
                                  tuple(case["velocity"]))
        assert HO.digest(HO.assemble_pool(nxt, n, g)) == case["advect_once"]


def test_ghost_fill_matches_periodic_window():
    """test_hydro.py:89-99 known answer."""
    field = HO.initial_field(16)
    pool = HO.make_pool(field, 8)
    assert np.isnan(pool[0, 0, 0, 0])
    HO.exchange_ghosts_pool(pool, 8, 2)
    idx = np.arange(-3, 8 + 3) % 16
    assert np.array_equal(pool[0], field[np.ix_(idx, idx, idx)])


def test_geometry_kats():
    """test_hydro.py:59-86 / test_acceptance.py:103-116 counts."""
    assert HO.ghost_cells(8) == 2232 and HO.ghost_cells(16) == 6552
    assert {k: HO.blocks_for(k, 8) for k in HO.KERNEL_ORDER} == \
        {"prep": 22, "reconstruct": 8, "flux": 24, "reduce": 1, "update": 4}
    assert {k: HO.blocks_for(k, 16) for k in HO.KERNEL_ORDER} == \
        {"prep": 84, "reconstruct": 46, "flux": 138, "reduce": 1,
         "update": 32}
    assert HO.domain_cells("flux", 8) == 3000
    assert len(HO.lattice(64, 8)) == 512 and len(HO.lattice(64, 16)) == 64


def _trace_ids(traces):
    return [t["name"] for t in traces]


def test_aggregation_oracle_replays_reference_traces(traces_golden):
    for tr in traces_golden:
        got = AO.replay(tr)
        for name, closes in tr["closes"].items():
            exp = [(p, tags, reason) for p, tags, reason in closes]
            mine = [(p, tags, reason) for _, p, tags, reason in got[name]]
            assert mine == exp, (tr["name"], name)


def test_trace_stats_consistent(traces_golden):
    for tr in traces_golden:
        for name, st in tr["stats"].items():
            hist = {}
            for _, tags, _ in tr["closes"][name]:
                hist[len(tags)] = hist.get(len(tags), 0) + 1
            assert {str(k): v for k, v in sorted(hist.items())} == \
                st["histogram"]
            solo = sum(1 for _, _, r in tr["closes"][name] if r == "solo")
            assert solo == st["solo_fast_path"]


@pytest.mark.parametrize("name,lead", [
    ("prep", 1434529120), ("reconstruct", 1190910889), ("flux", 1917989178),
    ("reduce", 864850440), ("update", 2552575352)])
def test_crc32_leads(name, lead):
    """the region-name crc32 leads."""
    from zlib import crc32
    assert crc32(name.encode()) == lead
