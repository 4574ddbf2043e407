"""CPU oracle for the strategy-3 hydro hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker or the timed CPU
baseline.  The product path (paper_2210_06438_b200) never imports it and
fails loudly when its CUDA library is missing.

A numpy restatement of the reference `taskfuse.hydro` numerics
(/root/reference/pkg/src/taskfuse/hydro), operation for operation, so the
results are bit-identical to the reference.  Every function cites the
reference lines it follows.  Two forms are provided:

* per-sub-grid bodies with the reference signatures (`reconstruct_body`,
  `flux_body`, ...) operating on a scratch dict — these are what the CPU
  baseline times, exactly like the reference task bodies;
* batched forms over a pool (S, E, E, E) — the same elementwise ops with a
  leading slice axis (numpy elementwise IEEE ops do not depend on the array
  shape), used to check whole GPU batches quickly.

Parity of this restatement is PINNED against golden vectors produced by
running the reference itself (tests/golden/make_golden.py, fixtures in
tests/golden/*.json.gz|npz) — see tests/test_oracle_golden.py.
"""

from __future__ import annotations

import math

import numpy as np

# scenario.py:20-27
GRID_N = 64
GHOST = 3
CENTER = (0.5, 0.5, 0.5)
WIDTH = 0.1
AMPLITUDE = 1.0
VELOCITY = (1.0, 1.0, 1.0)
CFL = 0.3
ITERATIONS_PER_STEP = 3
# kernels.py:22-24
KERNEL_ORDER = ("prep", "reconstruct", "flux", "reduce", "update")
THREADS_PER_BLOCK = 128


# ----------------------------------------------------------- scenario.py
def initial_field(grid_n: int = GRID_N) -> np.ndarray:
    """scenario.py:30-37 — 1 + Gaussian bump (the 'blast' field)."""
    x = (np.arange(grid_n) + 0.5) / grid_n
    dx2 = (x - CENTER[0]) ** 2
    dy2 = (x - CENTER[1]) ** 2
    dz2 = (x - CENTER[2]) ** 2
    r2 = (dx2[:, None, None] + dy2[None, :, None] + dz2[None, None, :])
    return 1.0 + AMPLITUDE * np.exp(-r2 / (2.0 * WIDTH ** 2))


def sod_field(grid_n: int) -> np.ndarray:
    """u = 1.0 where x_i < 0.5 else 0.125."""
    x = (np.arange(grid_n) + 0.5) / grid_n
    col = np.where(x < 0.5, 1.0, 0.125)
    return np.broadcast_to(col[:, None, None], (grid_n,) * 3).copy()


def stress_field(grid_n: int, seed: int = 20221012) -> np.ndarray:
    """SURVEY §8(d) parity stress: 1 + 0.1 * U[0,1) from default_rng(seed)."""
    return 1.0 + 0.1 * np.random.default_rng(seed).random((grid_n,) * 3)


def max_speed(velocity=VELOCITY) -> float:
    """scenario.py:40-41."""
    return max(abs(v) for v in velocity)


def dt_over_dx(velocity=VELOCITY) -> float:
    """scenario.py:44-45."""
    return CFL / max_speed(velocity)


def ghost_cells(n: int) -> int:
    """scenario.py:48-49."""
    return (n + 2 * GHOST) ** 3 - n ** 3


def lattice(grid_n: int, n: int) -> list[tuple[int, int, int]]:
    """scenario.py:58-68 — sub-grids in lexicographic (bx, by, bz) order."""
    m = grid_n // n
    return [(bx, by, bz) for bx in range(m) for by in range(m)
            for bz in range(m)]


def make_pool(field: np.ndarray, n: int) -> np.ndarray:
    """scenario.py:83-96 batched: (S, E, E, E) NaN ghosts, owned = field."""
    g = field.shape[0]
    m = g // n
    e = n + 2 * GHOST
    pool = np.full((m ** 3, e, e, e), np.nan)
    blocks = field.reshape(m, n, m, n, m, n).transpose(0, 2, 4, 1, 3, 5)
    pool[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n] = \
        blocks.reshape(m ** 3, n, n, n)
    return pool


def assemble_pool(pool: np.ndarray, n: int, grid_n: int) -> np.ndarray:
    """scenario.py:99-106 batched."""
    m = grid_n // n
    own = pool[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n]
    return own.reshape(m, m, m, n, n, n).transpose(0, 3, 1, 4, 2, 5) \
        .reshape(grid_n, grid_n, grid_n).copy()


def _ranges(offset: int, n: int):
    """scenario.py:109-116."""
    if offset == -1:
        return slice(0, GHOST), slice(n, n + GHOST)
    if offset == 1:
        return slice(n + GHOST, n + 2 * GHOST), slice(GHOST, 2 * GHOST)
    return slice(GHOST, n + GHOST), slice(GHOST, n + GHOST)


_OFFSETS = [(ox, oy, oz)
            for ox in (-1, 0, 1) for oy in (-1, 0, 1) for oz in (-1, 0, 1)
            if (ox, oy, oz) != (0, 0, 0)]


def exchange_ghosts_pool(pool: np.ndarray, n: int, per_axis: int,
                         ids=None) -> None:
    """scenario.py:124-142 over a pool: 26 periodic neighbour copies."""
    m = per_axis
    targets = range(m ** 3) if ids is None else ids
    for g in targets:
        b = (g // (m * m), (g // m) % m, g % m)
        for off in _OFFSETS:
            nb = tuple((b[i] + off[i]) % m for i in range(3))
            src_id = (nb[0] * m + nb[1]) * m + nb[2]
            dst, src = [], []
            for axis in range(3):
                d, s = _ranges(off[axis], n)
                dst.append(d)
                src.append(s)
            pool[g][tuple(dst)] = pool[src_id][tuple(src)]


# ------------------------------------------------------------ kernels.py
def make_scratch(n: int) -> dict:
    """kernels.py:27-36."""
    ext = n + 2 * GHOST
    cube = n + 2
    return {
        "w": np.empty((ext, ext, ext)),
        "up": np.empty((3, cube, cube, cube)),
        "um": np.empty((3, cube, cube, cube)),
        "F": np.empty((3, cube, cube, cube)),
        "reduce_out": np.empty(1),
    }


def domain_cells(kernel: str, n: int) -> int:
    """kernels.py:39-48."""
    ext = n + 2 * GHOST
    cube = n + 2
    return {"prep": ext ** 3, "reconstruct": cube ** 3, "flux": 3 * cube ** 3,
            "reduce": 1, "update": n ** 3}[kernel]


def blocks_for(kernel: str, n: int) -> int:
    """kernels.py:51-55."""
    if kernel == "flux":
        return 3 * math.ceil((n + 2) ** 3 / THREADS_PER_BLOCK)
    return math.ceil(domain_cells(kernel, n) / THREADS_PER_BLOCK)


def minmod(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """kernels.py:58-60."""
    return np.where(a * b <= 0.0, 0.0, np.where(np.abs(a) < np.abs(b), a, b))


def _cube(w: np.ndarray, n: int, shift=(0, 0, 0)) -> np.ndarray:
    """kernels.py:63-66, on the trailing three axes (leading axes batch)."""
    return w[..., 2 + shift[0]:n + 4 + shift[0],
             2 + shift[1]:n + 4 + shift[1],
             2 + shift[2]:n + 4 + shift[2]]


def prep_body(u_ext: np.ndarray, scratch: dict) -> None:
    """kernels.py:69-70."""
    scratch["w"][...] = u_ext


def reconstruct_body(scratch: dict, n: int) -> None:
    """kernels.py:73-81."""
    w = scratch["w"]
    base = _cube(w, n)
    for axis in range(3):
        shift = tuple(1 if k == axis else 0 for k in range(3))
        back = tuple(-s for s in shift)
        sigma = minmod(_cube(w, n, shift) - base, base - _cube(w, n, back))
        scratch["um"][axis] = base - 0.5 * sigma
        scratch["up"][axis] = base + 0.5 * sigma


def flux_body(scratch: dict, n: int, velocity=VELOCITY) -> None:
    """kernels.py:84-93."""
    for axis in range(3):
        a = velocity[axis]
        if a >= 0.0:
            scratch["F"][axis] = a * scratch["up"][axis]
        else:
            scratch["F"][axis] = a * np.roll(scratch["um"][axis], -1,
                                             axis=axis)


def reduce_body(scratch: dict, velocity=VELOCITY) -> None:
    """kernels.py:96-97."""
    scratch["reduce_out"][0] = max_speed(velocity)


def update_body(u_ext: np.ndarray, out_ext: np.ndarray, scratch: dict,
                n: int, dt_dx: float) -> None:
    """kernels.py:100-111."""
    F = scratch["F"]
    own = slice(1, n + 1)
    prev = slice(0, n)
    div = F[0][own, own, own] - F[0][prev, own, own]
    div = div + (F[1][own, own, own] - F[1][own, prev, own])
    div = div + (F[2][own, own, own] - F[2][own, own, prev])
    owned_src = u_ext[GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n]
    out_ext[GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n] = \
        owned_src - dt_dx * div


# ---------------------------------------------------- batched (S leading)
def reconstruct_batch(pool: np.ndarray, n: int, ids=None):
    """reconstruct_body over slices: pool (S,E,E,E) -> um, up (T,3,C,C,C)."""
    w = pool if ids is None else pool[np.asarray(ids)]
    c = n + 2
    um = np.empty((w.shape[0], 3, c, c, c))
    up = np.empty_like(um)
    base = _cube(w, n)
    for axis in range(3):
        shift = tuple(1 if k == axis else 0 for k in range(3))
        back = tuple(-s for s in shift)
        sigma = minmod(_cube(w, n, shift) - base, base - _cube(w, n, back))
        um[:, axis] = base - 0.5 * sigma
        up[:, axis] = base + 0.5 * sigma
    return um, up


def flux_batch(um: np.ndarray, up: np.ndarray, velocity=VELOCITY):
    """flux_body over slices (roll along the per-slice axis)."""
    F = np.empty_like(um)
    for axis in range(3):
        a = velocity[axis]
        if a >= 0.0:
            F[:, axis] = a * up[:, axis]
        else:
            F[:, axis] = a * np.roll(um[:, axis], -1, axis=axis + 1)
    return F


def flux_kt_batch(um: np.ndarray, up: np.ndarray, velocity=VELOCITY):
    """Kurganov-Tadmor central-upwind flux for f = a u:
    1/2 (f(u_L) + f(u_R)) - 1/2 a_max (u_R - u_L), u_L = up[c],
    u_R = um[c + e] (same roll as flux_body).  Equal to flux_batch in exact
    arithmetic; compared at 1e-12 relative (north_star tolerance)."""
    F = np.empty_like(um)
    for axis in range(3):
        a = velocity[axis]
        ul = up[:, axis]
        ur = np.roll(um[:, axis], -1, axis=axis + 1)
        F[:, axis] = 0.5 * (a * ul + a * ur) - (0.5 * abs(a)) * (ur - ul)
    return F


def update_batch(pool: np.ndarray, F: np.ndarray, n: int, dt_dx: float,
                 ids=None) -> np.ndarray:
    """update_body over slices: returns the owned block (T, n, n, n)."""
    u = pool if ids is None else pool[np.asarray(ids)]
    own = slice(1, n + 1)
    prev = slice(0, n)
    div = F[:, 0][:, own, own, own] - F[:, 0][:, prev, own, own]
    div = div + (F[:, 1][:, own, own, own] - F[:, 1][:, own, prev, own])
    div = div + (F[:, 2][:, own, own, own] - F[:, 2][:, own, own, prev])
    owned = u[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n]
    return owned - dt_dx * div


def recon_flux_batch(pool: np.ndarray, n: int, velocity=VELOCITY, ids=None):
    """The hot path: reconstruct then flux for every listed slice."""
    um, up = reconstruct_batch(pool, n, ids)
    return um, up, flux_batch(um, up, velocity)


# ---------------------------------------------------------- reference.py
def _limited_slope(u: np.ndarray, axis: int) -> np.ndarray:
    """reference.py:17-21."""
    fwd = np.roll(u, -1, axis=axis) - u
    bwd = u - np.roll(u, 1, axis=axis)
    return np.where(fwd * bwd <= 0.0, 0.0,
                    np.where(np.abs(fwd) < np.abs(bwd), fwd, bwd))


def advect_once(u: np.ndarray, velocity=VELOCITY, dt_dx=None) -> np.ndarray:
    """reference.py:24-39 — whole-grid periodic iteration."""
    if dt_dx is None:
        dt_dx = CFL / max_speed(velocity)
    div = None
    for axis in range(3):
        sigma = _limited_slope(u, axis)
        a = velocity[axis]
        if a >= 0.0:
            face = a * (u + 0.5 * sigma)
        else:
            minus = u - 0.5 * sigma
            face = a * np.roll(minus, -1, axis=axis)
        term = face - np.roll(face, 1, axis=axis)
        div = term if div is None else div + term
    return u - dt_dx * div


def reference_step(u: np.ndarray, velocity=VELOCITY, dt_dx=None,
                   iterations: int = ITERATIONS_PER_STEP) -> np.ndarray:
    """reference.py:42-48."""
    out = u
    for _ in range(iterations):
        out = advect_once(out, velocity, dt_dx)
    return out


def staged_iteration(pool: np.ndarray, n: int, per_axis: int,
                     velocity=VELOCITY) -> np.ndarray:
    """One staged iteration as HydroSim.task_iteration runs it
    (step.py:83-123): exchange ghosts, then prep/reconstruct/flux/update per
    sub-grid.  Returns the next pool (owned cells written, ghosts NaN)."""
    exchange_ghosts_pool(pool, n, per_axis)
    um, up, F = recon_flux_batch(pool, n, velocity)
    nxt = np.full_like(pool, np.nan)
    nxt[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n] = \
        update_batch(pool, F, n, dt_over_dx(velocity))
    return nxt


def slab_pack(pool: np.ndarray, n: int, mx: int, m: int):
    """exchange_ghosts (scenario.py:124-142) split across an x-slab
    partition: the slab's 3 lowest / highest owned x layers, (3, G, G)."""
    own = pool[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n]
    slab = own.reshape(mx, m, m, n, n, n).transpose(0, 3, 1, 4, 2, 5) \
        .reshape(mx * n, m * n, m * n)
    return slab[:GHOST].copy(), slab[-GHOST:].copy()


def slab_fill(pool: np.ndarray, n: int, mx: int, m: int, halo_lo, halo_hi):
    """Ghost fill of a slab pool from its own owned cells plus the x halo
    planes: the periodic window of the global field the slab overlays."""
    own = pool[:, GHOST:GHOST + n, GHOST:GHOST + n, GHOST:GHOST + n]
    slab = own.reshape(mx, m, m, n, n, n).transpose(0, 3, 1, 4, 2, 5) \
        .reshape(mx * n, m * n, m * n)
    ext = np.concatenate([halo_lo, slab, halo_hi], axis=0)  # x: -3..X+3
    G = m * n
    for g in range(mx * m * m):
        bx, by, bz = g // (m * m), (g // m) % m, g % m
        xi = np.arange(bx * n - GHOST, bx * n + n + GHOST) + GHOST
        yi = np.arange(by * n - GHOST, by * n + n + GHOST) % G
        zi = np.arange(bz * n - GHOST, bz * n + n + GHOST) % G
        pool[g] = ext[np.ix_(xi, yi, zi)]


def digest(a: np.ndarray) -> str:
    """sha256 of the C-contiguous little-endian float64 bytes."""
    import hashlib
    arr = np.ascontiguousarray(a, dtype="<f8")
    return hashlib.sha256(arr.tobytes()).hexdigest()
