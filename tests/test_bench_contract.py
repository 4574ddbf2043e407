"""bench.py contract pieces that run without a GPU: the algorithmic byte
counts (SURVEY §8 d) and the --impl reference line (the reference's CPU path
timed on host cores)."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_algorithmic_bytes():
    sys.path.insert(0, str(ROOT))
    import bench
    assert bench.b_alg(8) == 84800          # 165.63 B per cell-update
    assert bench.b_alg(16) == 482112
    assert bench.b_step(8) == 16896         # 33.0 B per cell-update
    assert abs(bench.b_alg(8) / 512 - 165.625) < 1e-9


def test_reference_arm_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
         "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "cell-updates/s" and line["value"] > 0
    assert line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["cpu_baseline"]["cores"] >= 1
    assert line["warmup"] >= 3


def test_reference_arm_prints_our_config():
    """Both arms print the same `config` dict (the driver compares them)."""
    sys.path.insert(0, str(ROOT))
    import bench
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
         "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=600, env=env, cwd=str(ROOT))
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["config"] == json.loads(json.dumps(bench.cfg2_config()))
    assert bench.cfg5_config(4, 512)["subgrids"] == 262144


def test_gpus_n_self_launches_n_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two
    ranks; the reference arm's N > 1 line is config 5 (strong scaling),
    printed once (rank 0), with n_gpus = 2."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
         "--gpus", "2", "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["subgrids"] == 262144
    assert line["config"]["workload"].startswith("config 5")


def test_world_size_must_match_gpus():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="", WORLD_SIZE="1", RANK="0",
               LOCAL_RANK="0")
    out = subprocess.run(
        [sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
         "--gpus", "2", "--steps", "1", "--warmup", "0"],
        capture_output=True, text=True, timeout=300, env=env, cwd=str(ROOT))
    assert out.returncode != 0
    assert "WORLD_SIZE=1" in out.stderr
