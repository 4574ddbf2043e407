"""PPM reconstruction oracle — TEST INFRASTRUCTURE ONLY, PARITY UNPINNED.

north_star asks for a batched PPM reconstruction (Octo-Tiger's scheme,
PAPER.md:134), but the reference artifact substitutes minmod (SPEC.md:12,
506), so there is no reference implementation to pin against.
This is a self-written numpy statement of the piecewise-parabolic method of
Colella & Woodward (1984) for a scalar field — 4th-order interface values
clipped to their neighbours, then the CW84 monotonicity constraints — used as
the checker for the CUDA kernel (tf_recon_flux_ppm_f64).  Its arithmetic
order is the contract the kernel follows; the tests also check the method's
defining properties (linear data reproduced exactly, constants preserved,
monotone data stays bounded), which do not depend on this file.

Per axis, for cube cell c (extended index c + 2; the stencil reaches
c + 2 +- 2, so the reference's ghost width 3 is exactly what PPM needs):

    a_{i+1/2} = 7/12 (u_i + u_{i+1}) - 1/12 (u_{i-1} + u_{i+2})
    a_{i+1/2} = min(max(a, min(u_i, u_{i+1})), max(u_i, u_{i+1}))
    uL = a_{i-1/2}, uR = a_{i+1/2}
    if (uR - u)(u - uL) <= 0:               uL = uR = u
    elif (uR - uL)(u - (uL + uR)/2) > (uR - uL)^2 / 6:    uL = 3u - 2uR
    elif (uR - uL)(u - (uL + uR)/2) < -(uR - uL)^2 / 6:   uR = 3u - 2uL
    um = uL (minus face), up = uR (plus face)

Fluxes reuse oracle.hydro_oracle.flux_batch / flux_kt_batch unchanged.
"""

from __future__ import annotations

import numpy as np

C7 = 7.0 / 12.0
C1 = 1.0 / 12.0
SIXTH = 1.0 / 6.0


def _shift(w, n, axis, d):
    """The (n+2)^3 cube window of w shifted by d cells along axis (trailing
    three axes are x, y, z)."""
    sl = []
    for k in range(3):
        off = 2 + (d if k == axis else 0)
        sl.append(slice(off, off + n + 2))
    return w[(Ellipsis, *sl)]


def interface(w, n, axis, d):
    """a_{i+d+1/2} for every cube cell i (d in {-1, 0})."""
    u0 = _shift(w, n, axis, d)
    u1 = _shift(w, n, axis, d + 1)
    um1 = _shift(w, n, axis, d - 1)
    u2 = _shift(w, n, axis, d + 2)
    a = C7 * (u0 + u1) - C1 * (um1 + u2)
    lo = np.minimum(u0, u1)
    hi = np.maximum(u0, u1)
    return np.minimum(np.maximum(a, lo), hi)


def ppm_states(w, n, axis):
    u = _shift(w, n, axis, 0)
    uL = interface(w, n, axis, -1)
    uR = interface(w, n, axis, 0)
    dq = uR - uL
    mid = u - 0.5 * (uL + uR)
    flat = (uR - u) * (u - uL) <= 0.0
    over_l = dq * mid > dq * dq * SIXTH
    over_r = dq * mid < -(dq * dq * SIXTH)
    new_l = np.where(flat, u, np.where(over_l, 3.0 * u - 2.0 * uR, uL))
    new_r = np.where(flat, u, np.where(~over_l & over_r,
                                       3.0 * u - 2.0 * uL, uR))
    return new_l, new_r


def reconstruct_ppm_batch(pool, n, ids=None):
    """PPM face states over slices: pool (S,E,E,E) -> um, up (T,3,C,C,C)."""
    w = pool if ids is None else pool[np.asarray(ids)]
    c = n + 2
    um = np.empty((w.shape[0], 3, c, c, c))
    up = np.empty_like(um)
    for axis in range(3):
        um[:, axis], up[:, axis] = ppm_states(w, n, axis)
    return um, up
