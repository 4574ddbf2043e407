"""Writes tests/golden/bench_cfg2.json: sha256 digests of the oracle's
reconstruct+flux outputs (um, up, F in per-sub-grid order) for the bench
headline workload — BASELINE config 2, the Sod field on a 128^3 grid,
4096 8^3 sub-grids, velocity (1, 1, 1).

The Sod field (1.0 / 0.125) and every value derived from it are exactly
representable and computed without transcendental functions, so the digests
do not depend on the machine that produced them: bench.py compares the
bytes its timed team plan wrote against these (a fixture read, no oracle
code runs on the GPU box).  The oracle itself is pinned to the reference
by tests/test_oracle_golden.py.

    python tests/golden/make_bench_digests.py
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import hydro_oracle as HO  # noqa: E402

GRID, N, VEL = 128, 8, (1.0, 1.0, 1.0)


def main():
    f = HO.sod_field(GRID)
    pool = HO.make_pool(f, N)
    HO.exchange_ghosts_pool(pool, N, GRID // N)
    um, up, F = HO.recon_flux_batch(pool, N, VEL)
    out = {"workload": "config 2: sod, grid 128, n 8, velocity (1,1,1)",
           "grid": GRID, "subgrid_n": N, "velocity": list(VEL),
           "field_digest": HO.digest(f),
           "um": HO.digest(um), "up": HO.digest(up), "F": HO.digest(F),
           "amax": HO.max_speed(VEL)}
    path = ROOT / "tests" / "golden" / "bench_cfg2.json"
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(path, out)


if __name__ == "__main__":
    main()
