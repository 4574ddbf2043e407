"""Acceptance criterion 1 and 4 of the reference (test_acceptance.py:103-153)
on the real B200 through the HydroSim mirror: counting identities (kernel
launches and transfers per step) and zero raw allocations after warm-up."""

import pytest

pytestmark = pytest.mark.gpu


def test_counting_identities_grid64(cuda):
    from paper_2210_06438_b200.bench_matrix import run_cell
    for engine in ("native", "python"):
        row8, _, _ = run_cell(8, 1, 1, steps=1, engine=engine)
        assert (row8.kernels, row8.transfers) == (7680, 15360), engine
        row16, _, _ = run_cell(16, 1, 1, steps=1, engine=engine)
        assert (row16.kernels, row16.transfers) == (960, 1920), engine
        assert row8.measured_raw_allocs == 0, engine
        assert row16.measured_raw_allocs == 0, engine
        assert row8.team_sizes == {1: 2 * 7680}, engine


def test_aggregation_reduces_launches_and_caps_teams(cuda):
    from paper_2210_06438_b200.bench_matrix import (BenchConfig, emit,
                                                    run_matrix)
    rep = run_matrix(BenchConfig(8, (1, 4), (1, 8), steps=1), grid_n=32)
    rows = {(r.executors, r.max_team): r for r in rep.rows}
    for (e, cap), r in rows.items():
        assert max(r.team_sizes) <= cap
        assert sum(k * v for k, v in r.team_sizes.items()) == 2 * 64 * 15
        assert r.measured_raw_allocs == 0
    assert rows[(1, 8)].kernels <= rows[(1, 1)].kernels
    text = emit(rep, "markdown")
    assert "## Strategy 3: on-the-fly aggregation" in text
    assert emit(rep).splitlines()[0] == ("cores,subgrid,executors,max_team,"
                                         "ms_per_step,kernels,transfers,"
                                         "raw_allocs,syncs")
