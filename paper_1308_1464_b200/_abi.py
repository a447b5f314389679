"""ctypes binding of the C ABI declared in include/wavestep.h.

This is the only place the package touches native code.  The shared
library is built in-tree (``__graft_entry__.build()`` or
``python -m paper_1308_1464_b200.build``) into ``paper_1308_1464_b200/_lib``.
There is no fallback: if the library is missing every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = LIB_DIR / "libwavestep.so"

WS_OK, WS_ERR_KERNEL, WS_ERR_CONFIG, WS_ERR_CUDA, WS_ERR_STATIONARY = 0, 1, 2, 3, 4
WS_ERR_INTERNAL = 5

SOLVER_IDS = {
    "acoustics-const": 0,
    "acoustics-var": 1,
    "euler": 2,
    "euler-hlle": 3,
    "shallow-water-roe": 4,
    "advection": 5,
}
LIMITER_IDS = {"none": 0, "minmod": 1, "superbee": 2, "mc": 3}
BC_IDS = {"periodic": 0, "extrapolate": 1}
PRECISION_IDS = {"f64": 0, "f32": 1, "f32fast": 2}
ROWS_MEMORY, ROWS_BC = 0, 1


class WsDesc(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32),
        ("dx", C.c_double), ("dy", C.c_double),
        ("num_ghost", C.c_int32), ("solver", C.c_int32),
        ("params", C.c_double * 4),
        ("order", C.c_int32), ("limiter", C.c_int32),
        ("bc_x", C.c_int32), ("bc_y", C.c_int32),
        ("precision", C.c_int32), ("device", C.c_int32),
        ("ny_global", C.c_int32), ("j_offset", C.c_int32),
        ("rows_lo", C.c_int32), ("rows_hi", C.c_int32),
        ("ext_q0", C.c_void_p), ("ext_q1", C.c_void_p),
        ("ext_aux", C.c_void_p), ("ext_slots", C.c_void_p),
    ]


class WsCtl(C.Structure):
    _fields_ = [("cfl", C.c_double), ("dt_max", C.c_double), ("fixed_dt", C.c_double),
                ("remaining", C.c_double), ("t_final", C.c_double)]


class WsReport(C.Structure):
    _fields_ = [("dt", C.c_double), ("cfl", C.c_double),
                ("max_speed_x", C.c_double), ("max_speed_y", C.c_double)]


class WsErrorInfo(C.Structure):
    _fields_ = [("code", C.c_int32), ("direction", C.c_int32), ("i", C.c_int32),
                ("j", C.c_int32), ("stage", C.c_int32), ("component", C.c_int32),
                ("step", C.c_int64)]


_P = C.c_void_p
# (name, restype, argtypes) — one row per declaration in include/wavestep.h
SIGNATURES = [
    ("ws_abi_version", C.c_int, []),
    ("ws_buffer_bytes", C.c_int, [C.POINTER(WsDesc), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("ws_create", C.c_int, [C.POINTER(WsDesc), C.POINTER(_P)]),
    ("ws_destroy", None, [_P]),
    ("ws_last_error", C.c_char_p, [_P]),
    ("ws_upload", C.c_int, [_P, _P, _P, _P]),
    ("ws_download", C.c_int, [_P, _P, _P]),
    ("ws_upload_f32", C.c_int, [_P, _P, _P, _P]),
    ("ws_download_f32", C.c_int, [_P, _P, _P]),
    ("ws_step", C.c_int, [_P, C.POINTER(WsCtl), _P]),
    ("ws_run", C.c_int, [_P, C.c_int32, C.POINTER(WsCtl), _P]),
    ("ws_download_async", C.c_int, [_P, _P, _P]),
    ("ws_download_aux_ghosts", C.c_int, [_P, _P, _P]),
    ("ws_pin_host", C.c_int, [_P, C.c_uint64]),
    ("ws_unpin_host", C.c_int, [_P]),
    ("ws_checked_counts", C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint32)]),
    ("ws_phase_speeds", C.c_int, [_P, _P]),
    ("ws_phase_speeds_part", C.c_int, [_P, C.c_int32, _P]),
    ("ws_phase_update", C.c_int, [_P, C.POINTER(WsCtl), _P]),
    ("ws_phase_update_part", C.c_int, [_P, C.POINTER(WsCtl), C.c_int32, _P]),
    ("ws_capture_begin", C.c_int, [_P]),
    ("ws_capture_end", C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("ws_replayed", C.c_int, [_P, C.c_int64, C.c_int64]),
    ("ws_slot_ptr", _P, [_P]),
    ("ws_halo_ptrs", C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P),
                               C.POINTER(_P), C.POINTER(C.c_uint64)]),
    ("ws_state_ptr", C.c_int, [_P, C.POINTER(_P), C.POINTER(C.c_int64),
                               C.POINTER(C.c_int64)]),
    ("ws_poll", C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(WsReport), C.c_int32,
                          C.POINTER(C.c_int32), C.POINTER(C.c_double),
                          C.POINTER(WsErrorInfo)]),
    ("ws_sync", C.c_int, [_P]),
    ("ws_launch_count", C.c_int64, [_P]),
    ("ws_trace", C.c_int, [_P, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]),
    ("ws_set_peers", C.c_int, [_P, C.c_int32, C.POINTER(C.c_void_p)]),
    ("ws_devstate_ptr", C.c_void_p, [_P]),
    ("ws_set_halo_peers", C.c_int, [_P, C.POINTER(C.c_void_p), C.c_void_p, C.c_int32,
                                    C.POINTER(C.c_void_p), C.c_void_p]),
    ("ws_riemann", C.c_int, [C.c_int32, C.POINTER(C.c_double), C.c_int32, C.c_int64,
                             _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_int32]),
    ("ws_fill_ghost", C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.c_int32]),
]

_LIB = None


class NativeUnavailable(RuntimeError):
    pass


def lib():
    """Load libwavestep.so (once).  Raises NativeUnavailable if not built."""
    global _LIB
    if _LIB is None:
        path = os.environ.get("WAVESTEP_LIB", str(LIB_PATH))
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (there is no CPU fallback)")
        handle = C.CDLL(path)
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.ws_abi_version() != 1:
            raise NativeUnavailable("libwavestep ABI version mismatch")
        _LIB = handle
    return _LIB


def nan_or(x):
    return math.nan if x is None else float(x)


def make_ctl(cfl=0.9, dt_max=None, fixed_dt=None, remaining=None, t_final=None) -> WsCtl:
    return WsCtl(float(cfl), nan_or(dt_max), nan_or(fixed_dt), nan_or(remaining),
                 nan_or(t_final))


class NativeError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(message)
        self.code = code


def check(rc: int, handle=None):
    if rc != WS_OK:
        msg = lib().ws_last_error(handle)
        raise NativeError(rc, msg.decode() if msg else f"wavestep error {rc}")
