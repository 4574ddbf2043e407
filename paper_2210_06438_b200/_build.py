"""Builds the in-tree C-ABI library `libtaskfuse_b200.so` for sm_100a.

Plain nvcc, no torch extension machinery: the product is a C ABI
(`include/taskfuse_b200.h`), bound from Python with ctypes.  The library
lands next to this file so it travels with the repo snapshot to GPU boxes.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libtaskfuse_b200.so"
SOURCES = ("hydro_kernels.cu", "aggregator.cpp", "halo.cu", "field_step.cu",
           "field_march.cu", "hydro_engine.cpp")
# relocatable device code (device-side kernel launches), device-linked
RDC_SOURCES = ("device_launch.cu",)
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found; cannot build libtaskfuse_b200.so")
    return cand


def _stale() -> bool:
    if not LIB.exists():
        return True
    built = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + RDC_SOURCES] + [
        ROOT / "include" / "taskfuse_b200.h", CSRC / "sm100_common.cuh",
        CSRC / "tf_nvtx.h", CSRC / "recon_flux.cuh", CSRC / "internal.h"]
    return any(p.stat().st_mtime > built for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile (if stale) and return the library path."""
    if not force and not _stale():
        return LIB
    tmp = PKG / "build"
    tmp.mkdir(exist_ok=True)
    objs = []
    log = []
    rdc_objs = []
    for src in SOURCES + RDC_SOURCES:
        obj = tmp / (src + ".o")
        # TASKFUSE_NVCC_EXTRA: extra -D tuning flags for experiment builds
        extra = os.environ.get("TASKFUSE_NVCC_EXTRA", "").split()
        rdc = ["-rdc=true"] if src in RDC_SOURCES else []
        cmd = [nvcc(), *NVCC_FLAGS, *rdc, *extra, "-x", "cu", "-c",
               str(CSRC / src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log.append(res.stdout + res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{res.stderr}")
        objs.append(str(obj))
        if rdc:
            rdc_objs.append(str(obj))
    gen = ["-gencode", "arch=compute_100a,code=sm_100a"]
    if rdc_objs:
        dlink = tmp / "device_link.o"
        cmd = [nvcc(), *gen, "-dlink", "-Xcompiler", "-fPIC", *rdc_objs,
               "-o", str(dlink), "-lcudadevrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc device link failed:\n{res.stderr}")
        objs.append(str(dlink))
    out = tmp / LIB.name
    cmd = [nvcc(), *gen, "-shared", "-Xcompiler", "-fPIC", *objs, "-o",
           str(out), "-lcudadevrt"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(out, LIB)
    (tmp / "ptxas.log").write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
