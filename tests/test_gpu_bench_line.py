"""The bench.py JSON line on a B200 carries every key of the contract:
device-timed value, roofline against the measured peak, e2e with host
buffers, kernel launch count, clocks sampled during the timed region."""

import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_line_contract(cuda):
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--steps", "5", "--warmup",
         "3", "--no-sweep", "--no-cpu-baseline"],
        capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup",
              "ms_per_step", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
              "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3
    assert d["higher_is_better"] is True and d["dtype"] == "f64"
    assert d["value"] > 0 and d["unit"] == "cell-updates/s"
    assert "workload" in d["config"] and "l2" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 \
        and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    # the timed outputs were checked against the oracle's digests
    assert d["self_check"]["bitexact_vs_oracle_digest"] is True
    assert e["result_check"] is True
    # the headline forms its teams on the fly inside the timed step; the
    # pre-formed plan rides along as a sub-key, equally checked
    assert d["run"]["mode"] == "queue" and d["gpu_launches"] == 5
    assert d["run"]["teams_per_step"] >= 1
    assert sum(int(k) * v for k, v in d["run"]["team_histogram"].items()) \
        >= 5 * 4096
    assert d["plan"]["self_check"]["bitexact_vs_oracle_digest"] is True


def test_bench_two_ranks_config5_gloo(cuda):
    """`--gpus 2` self-launches two ranks (here sharing the one GPU, gloo
    for the host-side collectives); the N > 1 line is config 5 strong
    scaling with the ghost exchange inside the step, printed once, with
    n_gpus = 2 and the three exchange paths cross-checked bit for bit."""
    import os
    env = dict(os.environ, TASKFUSE_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps",
         "3", "--warmup", "3", "--cfg5-grid", "256"],
        capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["workload"].startswith("config 5")
    assert d["run"]["halo_bytes_per_rank_per_step"] > 0
    assert all(d["self_check"].values()) and len(d["self_check"]) == 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0
