"""Tensor-level wrappers over the C ABI (include/taskfuse_b200.h).

torch is plumbing here: device memory and the current CUDA stream.  Every
op validates dtype/device/shape, then calls the native entry point with raw
pointers on torch's current stream.  Nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import TaskfuseCudaError, ValidationError

GHOST = 3
SUPPORTED_N = (8, 16)


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _need_cuda_f64(t: torch.Tensor, name: str) -> None:
    if not isinstance(t, torch.Tensor):
        raise ValidationError(f"{name} must be a torch tensor")
    if not t.is_cuda:
        raise TaskfuseCudaError(f"{name} must live on a CUDA device "
                                "(there is no CPU path)")
    if t.dtype != torch.float64:
        raise ValidationError(f"{name} must be float64, got {t.dtype}")
    if not t.is_contiguous():
        raise ValidationError(f"{name} must be contiguous")


def _ids_ptr(ids) -> tuple[int | None, int | None]:
    """ids tensor -> (pointer, count); None -> (None, None).  A device
    tensor, or a PINNED host tensor, which the kernel reads zero-copy over
    PCIe (one 4-byte load per CTA) — a team's ids then need no copy."""
    if ids is None:
        return None, None
    if not (isinstance(ids, torch.Tensor) and ids.dtype == torch.int32
            and ids.dim() == 1 and ids.is_contiguous()
            and (ids.is_cuda or ids.is_pinned())):
        raise ValidationError("ids must be a contiguous 1-D int32 CUDA or "
                              "pinned host tensor")
    return ids.data_ptr(), ids.numel()


def _check_n(n: int) -> None:
    if n not in SUPPORTED_N:
        raise ValidationError(f"sub-grid edge must be one of {SUPPORTED_N}, "
                              f"got {n}")


def _check_pool(pool: torch.Tensor, n: int, name="pool") -> int:
    _need_cuda_f64(pool, name)
    e = n + 2 * GHOST
    if pool.dim() != 4 or tuple(pool.shape[1:]) != (e, e, e):
        raise ValidationError(f"{name} must be (S, {e}, {e}, {e}), "
                              f"got {tuple(pool.shape)}")
    return pool.shape[0]


def _check_faces(t: torch.Tensor, n: int, slots: int, name: str) -> None:
    _need_cuda_f64(t, name)
    c = n + 2
    if t.dim() != 5 or tuple(t.shape[1:]) != (3, c, c, c) \
            or t.shape[0] < slots:
        raise ValidationError(f"{name} must be (>= {slots}, 3, {c}, {c}, {c})"
                              f", got {tuple(t.shape)}")


def _slots(out_mode: int, T: int, pool_slices: int) -> int:
    return pool_slices if out_mode else T


def recon_flux(pool, n, velocity, um, up, F, ids=None, T=None, out_mode=1,
               amax=None, flux_form=0, stream=None,
               reconstruction: str = "minmod") -> None:
    """Fused reconstruct+flux over T slices (tf_recon_flux_f64).

    reconstruction: "minmod" — the reference's scheme (bit-exact, pinned);
    "ppm" — piecewise-parabolic (tf_recon_flux_ppm_f64; parity unpinned,
    checked against oracle/ppm_oracle.py)."""
    if reconstruction not in ("minmod", "ppm"):
        raise ValidationError(f"unknown reconstruction {reconstruction!r}")
    lib = _lib.load()
    _check_n(n)
    S = _check_pool(pool, n)
    ptr, cnt = _ids_ptr(ids)
    T = cnt if cnt is not None else (S if T is None else T)
    slots = _slots(out_mode, T, S)
    for t, nm in ((um, "um"), (up, "up"), (F, "F")):
        _check_faces(t, n, slots, nm)
    if amax is not None:
        _need_cuda_f64(amax, "amax")
        if amax.numel() < slots:
            raise ValidationError("amax too small")
    ax, ay, az = (float(v) for v in velocity)
    fn = lib.tf_recon_flux_ppm_f64 if reconstruction == "ppm" else \
        lib.tf_recon_flux_f64
    rc = fn(pool.data_ptr(), S, ptr, T, n, ax, ay, az, um.data_ptr(),
            up.data_ptr(), F.data_ptr(), int(out_mode),
            None if amax is None else amax.data_ptr(), int(flux_form),
            _stream(stream))
    _lib.check(rc, "tf_recon_flux_f64" if reconstruction == "minmod"
               else "tf_recon_flux_ppm_f64")


def recon_flux_team(pool, n, velocity, host_ids, um, up, F, out_mode=1,
                    amax=None, flux_form=0, stream=None) -> None:
    """One aggregated team launch; ids travel in the kernel parameters."""
    lib = _lib.load()
    _check_n(n)
    S = _check_pool(pool, n)
    ids = np.ascontiguousarray(np.asarray(host_ids, dtype=np.int32))
    T = ids.size
    if not 1 <= T <= _lib.MAX_TEAM:
        raise ValidationError(f"team size must be 1..{_lib.MAX_TEAM}")
    slots = _slots(out_mode, T, S)
    for t, nm in ((um, "um"), (up, "up"), (F, "F")):
        _check_faces(t, n, slots, nm)
    ax, ay, az = (float(v) for v in velocity)
    rc = lib.tf_recon_flux_team_f64(
        pool.data_ptr(), S, ids.ctypes.data_as(C.POINTER(C.c_int32)), T, n,
        ax, ay, az, um.data_ptr(), up.data_ptr(), F.data_ptr(), int(out_mode),
        None if amax is None else amax.data_ptr(), int(flux_form),
        _stream(stream))
    _lib.check(rc, "tf_recon_flux_team_f64")


def reconstruct(pool, n, um, up, ids=None, T=None, out_mode=1,
                stream=None) -> None:
    """reconstruct_body batched (tf_reconstruct_f64)."""
    lib = _lib.load()
    _check_n(n)
    S = _check_pool(pool, n)
    ptr, cnt = _ids_ptr(ids)
    T = cnt if cnt is not None else (S if T is None else T)
    slots = _slots(out_mode, T, S)
    _check_faces(um, n, slots, "um")
    _check_faces(up, n, slots, "up")
    rc = lib.tf_reconstruct_f64(pool.data_ptr(), S, ptr, T, n, um.data_ptr(),
                                up.data_ptr(), int(out_mode), _stream(stream))
    _lib.check(rc, "tf_reconstruct_f64")


def flux(n, velocity, um, up, F, ids=None, T=None, out_mode=1,
         stream=None) -> None:
    """flux_body batched (tf_flux_f64)."""
    lib = _lib.load()
    _check_n(n)
    ptr, cnt = _ids_ptr(ids)
    T = cnt if cnt is not None else (um.shape[0] if T is None else T)
    slots = um.shape[0] if out_mode else T
    for t, nm in ((um, "um"), (up, "up"), (F, "F")):
        _check_faces(t, n, slots, nm)
    ax, ay, az = (float(v) for v in velocity)
    rc = lib.tf_flux_f64(ptr, T, n, ax, ay, az, um.data_ptr(), up.data_ptr(),
                         F.data_ptr(), int(out_mode), _stream(stream))
    _lib.check(rc, "tf_flux_f64")


def update(pool, n, F, dt_dx, next_pool, ids=None, T=None, out_mode=1,
           stream=None) -> None:
    """update_body batched, no FMA (tf_update_f64)."""
    lib = _lib.load()
    _check_n(n)
    S = _check_pool(pool, n)
    _check_pool(next_pool, n, "next_pool")
    ptr, cnt = _ids_ptr(ids)
    T = cnt if cnt is not None else (S if T is None else T)
    _check_faces(F, n, _slots(out_mode, T, S), "F")
    rc = lib.tf_update_f64(pool.data_ptr(), ptr, T, n, F.data_ptr(),
                           int(out_mode), float(dt_dx), next_pool.data_ptr(),
                           _stream(stream))
    _lib.check(rc, "tf_update_f64")


def ghost_fill(pool, n, per_axis, ids=None, stream=None) -> None:
    """exchange_ghosts for listed (default: all) sub-grids."""
    lib = _lib.load()
    _check_n(n)
    S = _check_pool(pool, n)
    if S != per_axis ** 3:
        raise ValidationError(f"pool holds {S} sub-grids, lattice needs "
                              f"{per_axis ** 3}")
    ptr, cnt = _ids_ptr(ids)
    rc = lib.tf_ghost_fill_f64(pool.data_ptr(), ptr, S if cnt is None else cnt,
                               n, per_axis, _stream(stream))
    _lib.check(rc, "tf_ghost_fill_f64")


def field_to_pool(field, n, pool, stream=None) -> None:
    """make_state's owned-cell scatter (scenario.py:83-96) on the device."""
    lib = _lib.load()
    _check_n(n)
    _need_cuda_f64(field, "field")
    g = field.shape[0]
    if field.dim() != 3 or g % n or pool.shape[0] != (g // n) ** 3:
        raise ValidationError("field/pool shapes do not match")
    _check_pool(pool, n)
    _lib.check(lib.tf_field_to_pool_f64(field.data_ptr(), g, n,
                                        pool.data_ptr(), _stream(stream)),
               "tf_field_to_pool_f64")


def field_to_pool_layers(field, n, pool, layer0, layers, stream=None) -> None:
    """field_to_pool for the sub-grid layers [layer0, layer0+layers) along x
    (one chunk of a pipelined upload)."""
    lib = _lib.load()
    _check_n(n)
    _need_cuda_f64(field, "field")
    g = field.shape[0]
    if field.dim() != 3 or g % n or pool.shape[0] != (g // n) ** 3:
        raise ValidationError("field/pool shapes do not match")
    _check_pool(pool, n)
    _lib.check(lib.tf_field_to_pool_layers_f64(
        field.data_ptr(), g, n, int(layer0), int(layers), pool.data_ptr(),
        _stream(stream)), "tf_field_to_pool_layers_f64")


def pool_to_field(pool, n, field, stream=None) -> None:
    """assemble (scenario.py:99-106) on the device."""
    lib = _lib.load()
    _check_n(n)
    _need_cuda_f64(field, "field")
    g = field.shape[0]
    if field.dim() != 3 or g % n or pool.shape[0] != (g // n) ** 3:
        raise ValidationError("field/pool shapes do not match")
    _check_pool(pool, n)
    _lib.check(lib.tf_pool_to_field_f64(pool.data_ptr(), g, n,
                                        field.data_ptr(), _stream(stream)),
               "tf_pool_to_field_f64")


def prep(pool, n, w, ids=None, T=None, out_mode=1, stream=None) -> None:
    """prep_body batched: w[slot] = pool[id]."""
    lib = _lib.load()
    _check_n(n)
    S = _check_pool(pool, n)
    ptr, cnt = _ids_ptr(ids)
    T = cnt if cnt is not None else (S if T is None else T)
    _check_pool(w, n, "w")
    if w.shape[0] < _slots(out_mode, T, S):
        raise ValidationError("w too small")
    rc = lib.tf_prep_f64(pool.data_ptr(), ptr, T, n, w.data_ptr(),
                         int(out_mode), _stream(stream))
    _lib.check(rc, "tf_prep_f64")


def reduce(velocity, out, ids=None, T=None, out_mode=1, stream=None) -> None:
    """reduce_body batched: out[slot] = max |v|."""
    lib = _lib.load()
    _need_cuda_f64(out, "reduce_out")
    ptr, cnt = _ids_ptr(ids)
    T = cnt if cnt is not None else (out.numel() if T is None else T)
    ax, ay, az = (float(v) for v in velocity)
    rc = lib.tf_reduce_f64(ptr, T, ax, ay, az, out.data_ptr(), int(out_mode),
                           _stream(stream))
    _lib.check(rc, "tf_reduce_f64")
