"""ctypes binding of libescg_b200.so (include/escg_dev.h).  No CPU fallback: if the library or a
CUDA device is missing, calls fail loudly with EngineError."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import raise_for

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ESCG_LIB") or os.path.join(PKG, "libescg_b200.so")

ESCG_KERNEL_AUTO, ESCG_KERNEL_TILE, ESCG_KERNEL_BLOCK = 0, 1, 2
ESCG_STOP_TRACKED, ESCG_STOP_STASIS = 1, 2
ESCG_RUNNING = -1


class Params(C.Structure):
    """POD mirror of escg::SimParams (params.hpp:18-49) — escg_params in escg_dev.h."""

    _fields_ = [
        ("length", C.c_int32),
        ("height", C.c_int32),
        ("mcs_limit", C.c_int64),
        ("neighbourhood", C.c_int32),
        ("print_frequency", C.c_int32),
        ("mobility", C.c_double),
        ("species", C.c_int32),
        ("flux", C.c_int32),
        ("empty_prob", C.c_double),
        ("save", C.c_int32),
        ("dominance_import", C.c_int32),
        ("resume", C.c_int32),
        ("num_randoms", C.c_int64),
        ("max_step", C.c_int32),
        ("has_seed", C.c_int32),
        ("seed", C.c_uint64),
    ]


EXPORTS = [
    "escg_dev_last_error", "escg_params_default", "escg_validate", "escg_action_rates", "escg_thresholds",
    "escg_align_num_randoms", "escg_dev_create", "escg_dev_destroy", "escg_dev_init_lattice", "escg_dev_set_lattice",
    "escg_dev_get_lattice", "escg_dev_counts", "escg_dev_advance", "escg_dev_run", "escg_dev_read_trace",
    "escg_dev_replica_result", "escg_dev_replay", "escg_dev_last_timing", "escg_dev_describe",
    "escg_dev_draw_format", "escg_dev_block_mode", "escg_simulate", "escg_dev_create_band", "escg_dev_band_info",
    "escg_group_advance", "escg_dev_band_rows", "escg_dev_band_step", "escg_dev_set_stream",
    "escg_dev_create_ring_part", "escg_dev_ring_part_export", "escg_dev_ring_part_connect", "escg_ring_group_advance",
    "escg_ipc_open", "escg_ipc_close",
]

_lib = None

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_P = C.POINTER(Params)
_H = C.c_void_p


def lib():
    """Load (building if stale) the in-tree CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from .build import build

        build()
    L = C.CDLL(LIB_PATH)
    L.escg_dev_last_error.restype = C.c_char_p
    L.escg_dev_last_error.argtypes = []
    L.escg_params_default.argtypes = [_P]
    L.escg_validate.argtypes = [_P, _f64p, C.c_int32, C.c_int32]
    L.escg_action_rates.argtypes = [C.c_double, C.c_int64, _f64p]
    L.escg_thresholds.argtypes = [C.c_double, C.c_int64, _f64p, C.c_int32, _u32p, _u32p]
    L.escg_align_num_randoms.restype = C.c_int64
    L.escg_align_num_randoms.argtypes = [C.c_int64, C.c_int64]
    L.escg_dev_create.argtypes = [_P, _f64p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                  C.POINTER(_H)]
    L.escg_dev_destroy.argtypes = [_H]
    L.escg_dev_init_lattice.argtypes = [_H]
    L.escg_dev_set_lattice.argtypes = [_H, C.c_int32, _i32p, C.c_int64]
    L.escg_dev_get_lattice.argtypes = [_H, C.c_int32, C.c_void_p, C.POINTER(C.c_int64)]
    L.escg_dev_counts.argtypes = [_H, C.c_int32, _u64p]
    L.escg_dev_advance.argtypes = [_H, C.c_int64]
    L.escg_dev_run.argtypes = [_H, C.c_int64, C.c_int64, C.c_uint32, C.c_int32, C.c_int32, C.c_void_p]
    L.escg_dev_read_trace.argtypes = [_H, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
    L.escg_dev_replica_result.argtypes = [_H, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int32), _u64p]
    L.escg_dev_replay.argtypes = [_H, _u32p, _u32p, _u32p, C.c_int64]
    L.escg_dev_last_timing.argtypes = [_H, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    L.escg_dev_describe.argtypes = [_H, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32)]
    L.escg_dev_draw_format.argtypes = [_H, C.POINTER(C.c_int32)]
    L.escg_dev_block_mode.argtypes = [_H, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.escg_dev_create_band.argtypes = [_P, _f64p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(_H)]
    L.escg_dev_band_info.argtypes = [_H, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32)]
    L.escg_group_advance.argtypes = [C.POINTER(_H), C.c_int32, C.c_int64]
    _pp = C.POINTER(C.c_void_p)
    L.escg_dev_band_rows.argtypes = [_H, _pp, _pp, _pp, _pp, C.POINTER(C.c_int64)]
    L.escg_dev_band_step.argtypes = [_H, C.c_int32]
    L.escg_dev_set_stream.argtypes = [_H, C.c_void_p]
    if hasattr(L, "escg_dev_create_ring_part"):  # (diagnostic builds of older sources lack the multi-part ring)
        L.escg_dev_create_ring_part.argtypes = [_P, _f64p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                C.c_int32, C.POINTER(_H)]
        L.escg_dev_ring_part_export.argtypes = [_H, _pp, _pp, _pp, C.POINTER(C.c_int32), C.c_void_p,
                                                C.POINTER(C.c_int64)]
        L.escg_dev_ring_part_connect.argtypes = [_H, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                                 C.c_void_p, C.c_void_p, C.c_int32]
        L.escg_ring_group_advance.argtypes = [C.POINTER(_H), C.c_int32, C.c_int64]
        L.escg_ipc_open.argtypes = [C.c_int32, C.c_void_p, _pp]
        L.escg_ipc_close.argtypes = [C.c_int32, C.c_void_p]
    L.escg_simulate.argtypes = [_P, _f64p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                C.c_uint32, C.c_int32, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p, C.c_void_p,
                                C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    for name in EXPORTS:
        if name != "escg_dev_last_error" and name != "escg_align_num_randoms" and hasattr(L, name):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        raise_for(rc, lib().escg_dev_last_error().decode())


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)
