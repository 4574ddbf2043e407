"""ctypes binding of the C ABI in include/taskfuse_b200.h.

This is the whole Python<->native seam: plain pointers, sizes and a CUDA
stream handle cross it; every entry point returns an int status that is
turned into `TaskfuseCudaError` here.  There is no fallback: if the library
is missing the import of any compute op raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import TaskfuseCudaError

LIB_PATH = Path(__file__).resolve().parent / "libtaskfuse_b200.so"

_i32, _i64, _f64 = C.c_int32, C.c_int64, C.c_double
_p = C.c_void_p
_pi32 = C.POINTER(C.c_int32)
_pi64 = C.POINTER(C.c_int64)

TF_E_INVALID = 1001
TF_E_NO_TMA = 1002
TF_E_ORDERING = 1003
TF_E_TIMEOUT = 1005
MAX_TEAM = 128
TF_LAUNCH_OVERLAP_PREV = 1
TF_PLAN_TEAM_BUFFERS = 2
TF_PLAN_REFGEO = 16
TF_STEP_HALO_YZ = 4
TF_STEP_HALO_X = 8
TF_MARCH_ROWS4 = 16
TF_MARCH_PDL_EDGE = 32
TF_MARCH_ALONG_Y = 64
TF_BARRIER_PDL = 1
TF_QUEUE_CHAIN = 2
TF_QUEUE_SORTED = 4


class EnterResult(C.Structure):
    _fields_ = [("parent", _i32), ("executor", _i32), ("team", _i64),
                ("slice_id", _i32), ("closed", _i32), ("queried", _i32)]


BUSY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32)

# name -> (restype, argtypes); mirrors include/taskfuse_b200.h
SIGNATURES = {
    "tf_recon_flux_f64": (C.c_int, [_p, _i64, _p, _i32, _i32, _f64, _f64, _f64,
                                    _p, _p, _p, _i32, _p, _i32, _p]),
    "tf_recon_flux_team_f64": (C.c_int, [_p, _i64, _pi32, _i32, _i32, _f64,
                                         _f64, _f64, _p, _p, _p, _i32, _p,
                                         _i32, _p]),
    "tf_recon_flux_team_ex_f64": (C.c_int, [_p, _i64, _pi32, _i32, _i32, _f64,
                                            _f64, _f64, _p, _p, _p, _i32, _p,
                                            _i32, _i32, _p]),
    "tf_recon_flux_refgeo_f64": (C.c_int, [_p, _i64, _pi32, _i32, _i32, _f64,
                                           _f64, _f64, _p, _p, _p, _i32, _p,
                                           _i32, _i32, _p]),
    "tf_recon_flux_ppm_f64": (C.c_int, [_p, _i64, _p, _i32, _i32, _f64, _f64,
                                        _f64, _p, _p, _p, _i32, _p, _i32,
                                        _p]),
    "tf_reconstruct_f64": (C.c_int, [_p, _i64, _p, _i32, _i32, _p, _p, _i32,
                                     _p]),
    "tf_flux_f64": (C.c_int, [_p, _i32, _i32, _f64, _f64, _f64, _p, _p, _p,
                              _i32, _p]),
    "tf_update_f64": (C.c_int, [_p, _p, _i32, _i32, _p, _i32, _f64, _p, _p]),
    "tf_ghost_fill_f64": (C.c_int, [_p, _p, _i32, _i32, _i32, _p]),
    "tf_prep_f64": (C.c_int, [_p, _p, _i32, _i32, _p, _i32, _p]),
    "tf_field_to_pool_f64": (C.c_int, [_p, _i32, _i32, _p, _p]),
    "tf_pool_to_field_f64": (C.c_int, [_p, _i32, _i32, _p, _p]),
    "tf_field_to_pool_layers_f64": (C.c_int, [_p, _i32, _i32, _i32, _i32, _p,
                                              _p]),
    "tf_reduce_f64": (C.c_int, [_p, _i32, _f64, _f64, _f64, _p, _i32, _p]),
    "tf_region_create": (C.c_int, [C.c_char_p, _i32, _i32, _i32,
                                   C.POINTER(_p)]),
    "tf_region_destroy": (None, [_p]),
    "tf_region_parent_executor": (_i32, [_p, _i32]),
    "tf_region_enter": (C.c_int, [_p, _i64, BUSY_FN, _p,
                                  C.POINTER(EnterResult)]),
    "tf_region_stream_idle": (C.c_int, [_p, _i32, _pi64, _i32]),
    "tf_region_watch_count": (_i32, [_p, _i32]),
    "tf_region_release_team": (C.c_int, [_p, _i64]),
    "tf_region_team_size": (C.c_int, [_p, _i64]),
    "tf_region_team_members": (C.c_int, [_p, _i64, _pi64, _i32]),
    "tf_region_team_parent": (C.c_int, [_p, _i64]),
    "tf_region_stats": (C.c_int, [_p, _pi64, _pi64, _pi64]),
    "tf_team_issue": (C.c_int, [_p, _i64, _i32, C.c_char_p, _pi32, _pi32]),
    "tf_team_leave": (C.c_int, [_p, _i64, _i32, _pi32]),
    "tf_team_op_begin": (C.c_int, [_p, _i64]),
    "tf_team_op_end": (C.c_int, [_p, _i64, _pi32]),
    "tf_team_set_lease": (C.c_int, [_p, _i64, _i32, _i64]),
    "tf_team_lease": (_i64, [_p, _i64, _i32]),
    "tf_team_leases": (C.c_int, [_p, _i64, _pi64, _i32]),
    "tf_team_step_info": (C.c_int, [_p, _i64, _i32, _pi32, C.c_char_p,
                                    _i32]),
    "tf_region_violations": (_i64, [_p]),
    "tf_region_error": (C.c_char_p, [_p]),
    "tf_hydro_create": (C.c_int, [_i32, _i32, _i32, _i32, _p, _f64, _f64,
                                  _f64, _f64, _p, _p, _p, _p, _p,
                                  C.POINTER(_p)]),
    "tf_hydro_destroy": (None, [_p]),
    "tf_hydro_presize": (C.c_int, [_p]),
    "tf_hydro_iteration": (C.c_int, [_p, _p, _p, _p]),
    "tf_hydro_region": (C.c_int, [_p, _i32, C.POINTER(_p)]),
    "tf_hydro_counters": (C.c_int, [_p, _pi64]),
    "tf_hydro_host_times": (C.c_int, [_p, _pi64]),
    "tf_executor_create": (C.c_int, [_p, _i32, C.POINTER(_p)]),
    "tf_executor_destroy": (None, [_p]),
    "tf_executor_stream": (_p, [_p, _i32]),
    "tf_executor_run_recon_flux": (C.c_int, [_p, _p, _i64, _pi32, _i64, _i32,
                                             _f64, _f64, _f64, _p, _p, _p, _p,
                                             _i32, _pi64]),
    "tf_executor_join": (C.c_int, [_p, _p]),
    "tf_executor_fork": (C.c_int, [_p, _p]),
    "tf_executor_set_flags": (C.c_int, [_p, _i32]),
    "tf_executor_sync": (C.c_int, [_p]),
    "tf_plan_capture_recon_flux": (C.c_int, [_pi32, _pi64, _pi32, _i64, _i32,
                                             _p, _i64, _i32, _f64, _f64, _f64,
                                             _p, _p, _p, _p, _i32, _i32,
                                             C.POINTER(_p)]),
    "tf_plan_capture_field_step": (C.c_int, [_pi32, _pi64, _pi32, _i64, _i32,
                                             _p, _i32, _i32, _i32, _i32, _f64,
                                             _f64, _f64, _f64, _p, _i32,
                                             C.POINTER(_p)]),
    "tf_plan_launch": (C.c_int, [_p, _p]),
    "tf_plan_kernels": (_i64, [_p]),
    "tf_plan_destroy": (None, [_p]),
    "tf_halo_pack_f64": (C.c_int, [_p, _i32, _i32, _i32, _p, _p, _p]),
    "tf_ghost_fill_slab_f64": (C.c_int, [_p, _i32, _i32, _i32, _p, _p, _i32,
                                         _i32, _p]),
    "tf_field_step_f64": (C.c_int, [_p, _i32, _i32, _i32, _i32, _p, _pi32,
                                    _i32, _f64, _f64, _f64, _f64, _p, _i32,
                                    _p]),
    "tf_field_halo_f64": (C.c_int, [_p, _i32, _i32, _i32, _i32, _p]),
    "tf_field_step_peer_f64": (C.c_int, [_p, _i32, _i32, _i32, _i32, _p, _i32,
                                         _f64, _f64, _f64, _f64, _p, _p, _p,
                                         _p]),
    "tf_field_march_f64": (C.c_int, [_p, _i32, _i32, _i32, _f64, _f64, _f64,
                                     _f64, _p, _p, _p, _i32, _i32, _p, _p]),
    "tf_peer_barrier": (C.c_int, [_p, _p, _p, _i64, _i64, _p, _p]),
    "tf_peer_barrier_ex": (C.c_int, [_p, _p, _p, _i64, _i64, _p, _i32, _p]),
    "tf_field_halo_layers_f64": (C.c_int, [_p, _i32, _i32, _i32, _i32, _i32,
                                           _p]),
    "tf_field_halo_xwrap_f64": (C.c_int, [_p, _i32, _i32, _i32, _i32, _p]),
    "tf_field_pad_f64": (C.c_int, [_p, _i32, _i32, _i32, _p, _p]),
    "tf_field_pad_halo_f64": (C.c_int, [_p, _i32, _i32, _i32, _p, _i32, _i32,
                                        _p]),
    "tf_field_unpad_f64": (C.c_int, [_p, _i32, _i32, _i32, _p, _p]),
    "tf_field_unpad_host_f64": (C.c_int, [_p, _i32, _i32, _i32, _p, _i32,
                                          _p]),
    "tf_memcpy_async": (C.c_int, [_p, _p, _i64, _p]),
    "tf_dlexec_create": (C.c_int, [_p, _i32, C.POINTER(_p)]),
    "tf_dlexec_destroy": (None, [_p]),
    "tf_dlexec_run_recon_flux": (C.c_int, [_p, _p, _i64, _pi32, _i64, _f64,
                                           _f64, _f64, _p, _p, _p, _p, _i32,
                                           _p, _pi64]),
    "tf_dlexec_wait": (C.c_int, [_p]),
    "tf_qexec_create": (C.c_int, [_p, _i32, C.POINTER(_p)]),
    "tf_qexec_destroy": (None, [_p]),
    # ids as a raw address (the step loop passes a numpy array's pointer)
    "tf_qexec_run_recon_flux": (C.c_int, [_p, _p, _i64, _p, _i64, _f64,
                                          _f64, _f64, _p, _p, _p, _p, _i32,
                                          _p, _p]),
    "tf_qexec_set_flags": (C.c_int, [_p, _i32]),
    "tf_qexec_completed": (_i64, [_p]),
    "tf_qexec_host_times": (C.c_int, [_p, _pi64]),
    "tf_qexec_wait": (C.c_int, [_p]),
    "tf_queue_consumer_launch": (C.c_int, [_p, _i64, _i32, _p, _p, _p, _i64,
                                           _p, C.c_uint64, _i32, _f64, _f64,
                                           _f64, _p, _p, _p, _p, _i32, _i64,
                                           _i32, _p]),
    "tf_version": (C.c_char_p, []),
    "tf_check_device": (C.c_int, [_i32]),
}

_lib = None


def load(build_if_missing: bool | None = None) -> C.CDLL:
    """Load (building first when allowed) the in-tree C-ABI library."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing is None:
        build_if_missing = os.environ.get("TASKFUSE_NO_BUILD", "0") != "1"
    if build_if_missing:
        from ._build import build
        build()
    if not LIB_PATH.exists():
        raise TaskfuseCudaError(
            f"native library {LIB_PATH} is missing; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` — there is "
            "no CPU fallback")
    lib = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        if rc == TF_E_INVALID:
            msg = "invalid argument"
        elif rc == TF_E_NO_TMA:
            msg = "cuTensorMapEncodeTiled unavailable"
        elif rc == TF_E_TIMEOUT:
            msg = "device queue timed out with work unprocessed"
        else:
            msg = f"CUDA error {rc}"
        raise TaskfuseCudaError(f"{what} failed: {msg} (rc={rc})")
