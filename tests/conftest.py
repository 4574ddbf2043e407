"""Shared test setup.

Markers: `gpu` — needs a B200 (run on a GPU box: pytest -m gpu).  Everything
else runs on the CPU build container (pytest -m "not gpu").  The oracle
(oracle/) is imported here as the checker only.
"""

import gzip
import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")


@pytest.fixture(scope="session")
def native_lib():
    from paper_2210_06438_b200 import _lib
    return _lib.load()


@pytest.fixture(scope="session")
def hydro_golden():
    with gzip.open(GOLDEN / "hydro.json.gz", "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def traces_golden():
    with gzip.open(GOLDEN / "traces.json.gz", "rt") as fh:
        return json.load(fh)["traces"]


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test on a box without CUDA")
    from paper_2210_06438_b200 import _lib
    lib = _lib.load(build_if_missing=os.environ.get("TASKFUSE_NO_BUILD") != "1")
    assert lib.tf_check_device(0) == 0, "device 0 is not sm_100 (B200)"
    return torch.device("cuda:0")
