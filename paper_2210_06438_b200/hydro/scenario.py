"""Problem setup on the device — mirror of taskfuse/hydro/scenario.py.

Same constants, names and semantics as the reference (scenario.py:20-157),
but the sub-grid arrays live in ONE device pool per field, a float64 tensor
(S, E, E, E) with sub-grids in lexicographic (bx, by, bz) order — exactly
the stacking of the reference's per-block (E, E, E) arrays — so the batched
kernels can address any sub-grid by its id.  `state.u[block]` /
`state.u_next[block]` are views into the pools, so reference-style per-block
code keeps working.  Ghosts start as NaN (scenario.py:6-7, 91).
"""

from __future__ import annotations

import numpy as np
import torch

from ..errors import ValidationError
from .. import ops

GRID_N = 64
GHOST = 3
CENTER = (0.5, 0.5, 0.5)
WIDTH = 0.1
AMPLITUDE = 1.0
VELOCITY = (1.0, 1.0, 1.0)
CFL = 0.3
ITERATIONS_PER_STEP = 3


def _dev(device):
    return torch.device(device) if device is not None else \
        torch.device("cuda", torch.cuda.current_device())


def initial_field(grid_n: int = GRID_N, device=None) -> torch.Tensor:
    """scenario.py:30-37 (1 + Gaussian bump; the blast-wave stand-in).

    Setup, not hot path: evaluated with numpy on the host so the initial
    data are bit-identical to the reference's (a device exp() may differ in
    the last ulp), then moved to the device."""
    x = (np.arange(grid_n) + 0.5) / grid_n
    dx2 = (x - CENTER[0]) ** 2
    dy2 = (x - CENTER[1]) ** 2
    dz2 = (x - CENTER[2]) ** 2
    r2 = (dx2[:, None, None] + dy2[None, :, None] + dz2[None, None, :])
    field = 1.0 + AMPLITUDE * np.exp(-r2 / (2.0 * WIDTH ** 2))
    return torch.from_numpy(field).to(_dev(device))


def sod_field(grid_n: int, device=None) -> torch.Tensor:
    """Sod shock tube initial data (SURVEY §8 d): 1.0 for x < 0.5, else
    0.125, constant in y and z."""
    d = _dev(device)
    x = (torch.arange(grid_n, dtype=torch.float64, device=d) + 0.5) / grid_n
    col = torch.where(x < 0.5, 1.0, 0.125).to(torch.float64)
    return col[:, None, None].expand(grid_n, grid_n, grid_n).contiguous()


def max_speed(velocity=VELOCITY) -> float:
    return max(abs(v) for v in velocity)


def dt_over_dx(velocity=VELOCITY) -> float:
    return CFL / max_speed(velocity)


def ghost_cells(n: int) -> int:
    return (n + 2 * GHOST) ** 3 - n ** 3


def pool_from_field(field: torch.Tensor, n: int) -> torch.Tensor:
    """(g,g,g) field -> (S, E, E, E) pool, owned cells set, ghosts NaN."""
    g = field.shape[0]
    if g % n:
        raise ValidationError(f"sub-grid edge {n} does not divide grid {g}")
    m = g // n
    e = n + 2 * GHOST
    pool = torch.full((m ** 3, e, e, e), float("nan"), dtype=torch.float64,
                      device=field.device)
    blocks = field.reshape(m, n, m, n, m, n).permute(0, 2, 4, 1, 3, 5)
    pool[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n] = \
        blocks.reshape(m ** 3, n, n, n)
    return pool


def field_from_pool(pool: torch.Tensor, n: int, grid_n: int) -> torch.Tensor:
    """Inverse of pool_from_field (owned cells only)."""
    m = grid_n // n
    own = pool[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n]
    return own.reshape(m, m, m, n, n, n).permute(0, 3, 1, 4, 2, 5) \
        .reshape(grid_n, grid_n, grid_n).contiguous()


class _BlockView:
    """Mapping block tuple -> (E,E,E) view of one pool (dict-like)."""

    def __init__(self, state, which):
        self._state = state
        self._which = which

    def _pool(self):
        return getattr(self._state, self._which)

    def __getitem__(self, block):
        return self._pool()[self._state.block_id(block)]

    def __setitem__(self, block, value):
        self._pool()[self._state.block_id(block)] = value

    def __len__(self):
        return len(self._state.blocks)

    def __iter__(self):
        return iter(self._state.blocks)

    def keys(self):
        return list(self._state.blocks)


class HydroState:
    """scenario.py:52-80 on the device: two pools, pointer swap."""

    def __init__(self, subgrid_n: int, grid_n: int = GRID_N, device=None):
        if grid_n % subgrid_n != 0:
            raise ValidationError(
                f"sub-grid edge {subgrid_n} does not divide grid {grid_n}")
        if subgrid_n not in ops.SUPPORTED_N:
            raise ValidationError(
                f"sub-grid edge must be one of {ops.SUPPORTED_N}")
        self.n = subgrid_n
        self.grid_n = grid_n
        self.per_axis = grid_n // subgrid_n
        self.ext = subgrid_n + 2 * GHOST
        m = self.per_axis
        self.blocks = [(bx, by, bz) for bx in range(m) for by in range(m)
                       for bz in range(m)]
        self.device = _dev(device)
        e = self.ext
        self.u_pool = torch.full((m ** 3, e, e, e), float("nan"),
                                 dtype=torch.float64, device=self.device)
        self.u_next_pool = torch.full_like(self.u_pool, float("nan"))
        self.u = _BlockView(self, "u_pool")
        self.u_next = _BlockView(self, "u_next_pool")
        self.time = 0.0
        self.steps_taken = 0

    def block_id(self, block) -> int:
        m = self.per_axis
        return (block[0] * m + block[1]) * m + block[2]

    def swap(self) -> None:
        self.u_pool, self.u_next_pool = self.u_next_pool, self.u_pool

    def owned(self, block) -> torch.Tensor:
        n = self.n
        return self.u[block][GHOST:GHOST + n, GHOST:GHOST + n,
                             GHOST:GHOST + n]


def make_state(subgrid_n: int, grid_n: int = GRID_N, field=None,
               device=None) -> HydroState:
    """scenario.py:83-96.  `field` may be a numpy array or a tensor."""
    state = HydroState(subgrid_n, grid_n, device)
    if field is None:
        field = initial_field(grid_n, state.device)
    elif isinstance(field, np.ndarray):
        field = torch.from_numpy(np.ascontiguousarray(field, np.float64))
    field = field.to(state.device, torch.float64)
    if tuple(field.shape) != (grid_n,) * 3:
        raise ValidationError(f"field must be {(grid_n,) * 3}")
    state.u_pool.copy_(pool_from_field(field, subgrid_n))
    return state


def assemble(state: HydroState) -> np.ndarray:
    """scenario.py:99-106: owned regions gathered into one host array."""
    return field_from_pool(state.u_pool, state.n, state.grid_n).cpu().numpy()


def exchange_ghosts(state: HydroState, block=None) -> None:
    """scenario.py:124-142 on the device: one block, or (block=None) every
    block in one launch of the ghost-fill kernel."""
    ids = None
    if block is not None:
        ids = torch.tensor([state.block_id(block)], dtype=torch.int32,
                           device=state.device)
    ops.ghost_fill(state.u_pool, state.n, state.per_axis, ids=ids)


def dump_state(state: HydroState, path: str) -> None:
    """scenario.py:145-150 (same npz format, so checkpoints interoperate)."""
    np.savez(path, field=assemble(state), subgrid_n=state.n,
             grid_n=state.grid_n, time=state.time,
             steps_taken=state.steps_taken)


def load_state(path: str, device=None) -> HydroState:
    """scenario.py:153-157."""
    with np.load(path) as data:
        state = make_state(int(data["subgrid_n"]), int(data["grid_n"]),
                           field=data["field"], device=device)
        state.time = float(data["time"])
        state.steps_taken = int(data["steps_taken"])
    return state
