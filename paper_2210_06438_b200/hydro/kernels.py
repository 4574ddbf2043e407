"""Per-sub-grid stage bodies on the device — taskfuse/hydro/kernels.py.

Same names and signatures as the reference (kernels.py:22-111); the scratch
dict holds device tensors instead of numpy arrays, and each body is one
launch of the corresponding batched sm_100a kernel with a single slice.
`ScratchPool` is the batched form: the scratch of every sub-grid stacked
along a leading axis, addressed by sub-grid id — what the aggregated team
launches write into (HydroSim.scratch, step.py:53).
"""

from __future__ import annotations

import math

import torch

from .. import ops
from .scenario import GHOST, VELOCITY, max_speed

KERNEL_ORDER = ("prep", "reconstruct", "flux", "reduce", "update")
THREADS_PER_BLOCK = 128


def _dev(device):
    return torch.device(device) if device is not None else \
        torch.device("cuda", torch.cuda.current_device())


def make_scratch(n: int, device=None) -> dict:
    """kernels.py:27-36 on the device (NaN-initialised: outputs must be
    fully overwritten)."""
    d = _dev(device)
    ext, cube = n + 2 * GHOST, n + 2
    f = dict(dtype=torch.float64, device=d)
    nan = float("nan")
    return {
        "w": torch.full((ext, ext, ext), nan, **f),
        "up": torch.full((3, cube, cube, cube), nan, **f),
        "um": torch.full((3, cube, cube, cube), nan, **f),
        "F": torch.full((3, cube, cube, cube), nan, **f),
        "reduce_out": torch.full((1,), nan, **f),
    }


def domain_cells(kernel: str, n: int) -> int:
    ext, cube = n + 2 * GHOST, n + 2
    return {"prep": ext ** 3, "reconstruct": cube ** 3, "flux": 3 * cube ** 3,
            "reduce": 1, "update": n ** 3}[kernel]


def blocks_for(kernel: str, n: int) -> int:
    if kernel == "flux":
        return 3 * math.ceil((n + 2) ** 3 / THREADS_PER_BLOCK)
    return math.ceil(domain_cells(kernel, n) / THREADS_PER_BLOCK)


def _one(t: torch.Tensor) -> torch.Tensor:
    return t.unsqueeze(0)


def prep_body(u_ext, scratch: dict) -> None:
    n = u_ext.shape[0] - 2 * GHOST
    ops.prep(_one(u_ext), n, _one(scratch["w"]), out_mode=0)


def reconstruct_body(scratch: dict, n: int) -> None:
    ops.reconstruct(_one(scratch["w"]), n, _one(scratch["um"]),
                    _one(scratch["up"]), out_mode=0)


def flux_body(scratch: dict, n: int, velocity=VELOCITY) -> None:
    ops.flux(n, velocity, _one(scratch["um"]), _one(scratch["up"]),
             _one(scratch["F"]), out_mode=0)


def reduce_body(scratch: dict, velocity=VELOCITY) -> None:
    ops.reduce(velocity, scratch["reduce_out"], out_mode=0)


def update_body(u_ext, out_ext, scratch: dict, n: int, dt_dx: float) -> None:
    """Writes the owned region of `out_ext`; everything else untouched."""
    ops.update(_one(u_ext), n, _one(scratch["F"]), dt_dx, _one(out_ext),
               out_mode=0)


class ScratchPool:
    """make_scratch for S sub-grids, stacked (slot = sub-grid id)."""

    def __init__(self, S: int, n: int, device=None):
        d = _dev(device)
        ext, cube = n + 2 * GHOST, n + 2
        f = dict(dtype=torch.float64, device=d)
        nan = float("nan")
        self.n = n
        self.w = torch.full((S, ext, ext, ext), nan, **f)
        self.um = torch.full((S, 3, cube, cube, cube), nan, **f)
        self.up = torch.full_like(self.um, nan)
        self.F = torch.full_like(self.um, nan)
        self.reduce_out = torch.full((S,), nan, **f)

    def view(self, g: int) -> dict:
        """Reference-style scratch dict of sub-grid g (views)."""
        return {"w": self.w[g], "um": self.um[g], "up": self.up[g],
                "F": self.F[g], "reduce_out": self.reduce_out[g:g + 1]}

    def poison(self, value=float("nan")) -> None:
        for t in (self.w, self.um, self.up, self.F, self.reduce_out):
            t.fill_(value)


def check_reduce(pool: ScratchPool, velocity=VELOCITY) -> None:
    """step.py:121-123: the reduction must report the advection speed."""
    if not bool((pool.reduce_out == max_speed(velocity)).all()):
        raise AssertionError("reduce stage did not report max |v|")
