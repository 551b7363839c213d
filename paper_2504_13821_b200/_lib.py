"""ctypes binding of the C-ABI in include/rectri_cu.h (librectri_cu.so).

There is no fallback: if the in-tree library is missing the import of any
compute entry point raises, so a GPU run can never silently take a CPU path.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "librectri_cu.so"

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32


class Spec(ctypes.Structure):
    """rectri_cu_spec  <- rectri::TriangularSpec (flags.hpp:29-35)."""

    _fields_ = [
        ("side", c_i32),
        ("uplo", c_i32),
        ("trans", c_i32),
        ("diag", c_i32),
        ("alpha", ctypes.c_double),
    ]


class View(ctypes.Structure):
    """rectri_cu_view  <- rectri::MatrixView<T> (matrix.hpp:75-160)."""

    _fields_ = [
        ("origin", ctypes.c_void_p),
        ("origin_rows", c_i64),
        ("origin_cols", c_i64),
        ("row_offset", c_i64),
        ("col_offset", c_i64),
        ("rows", c_i64),
        ("cols", c_i64),
    ]


class BackendC(ctypes.Structure):
    """rectri_cu_backend  <- rectri::Backend (backend.hpp:20-29) + device/stream."""

    _fields_ = [
        ("parallel_width", c_i32),
        ("device", c_i32),
        ("stream", ctypes.c_void_p),
        ("flags", ctypes.c_uint32),
        ("mc", c_i64),
        ("kc", c_i64),
        ("nc", c_i64),
    ]


EVENT_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, c_i32, c_i64, c_i64)

# name -> (restype, argtypes)
_P = ctypes.POINTER
SIGNATURES = {
    "rectri_cu_rec_trmm_f64": (ctypes.c_int, [_P(Spec), View, View, c_i64, _P(BackendC), EVENT_FN, ctypes.c_void_p]),
    "rectri_cu_rec_trmm_f32": (ctypes.c_int, [_P(Spec), View, View, c_i64, _P(BackendC), EVENT_FN, ctypes.c_void_p]),
    "rectri_cu_rec_trsm_f64": (ctypes.c_int, [_P(Spec), View, View, c_i64, _P(BackendC), EVENT_FN, ctypes.c_void_p, _P(c_i64)]),
    "rectri_cu_rec_trsm_f32": (ctypes.c_int, [_P(Spec), View, View, c_i64, _P(BackendC), EVENT_FN, ctypes.c_void_p, _P(c_i64)]),
    "rectri_cu_trmm_base_f64": (ctypes.c_int, [_P(Spec), View, View, c_i64, _P(BackendC)]),
    "rectri_cu_trmm_base_f32": (ctypes.c_int, [_P(Spec), View, View, c_i64, _P(BackendC)]),
    "rectri_cu_trsm_base_f64": (ctypes.c_int, [_P(Spec), View, View, c_i64, _P(BackendC), _P(c_i64)]),
    "rectri_cu_trsm_base_f32": (ctypes.c_int, [_P(Spec), View, View, c_i64, _P(BackendC), _P(c_i64)]),
    "rectri_cu_gemm_f64": (ctypes.c_int, [ctypes.c_double, c_i32, View, c_i32, View, ctypes.c_double, View, _P(BackendC)]),
    "rectri_cu_gemm_f32": (ctypes.c_int, [ctypes.c_float, c_i32, View, c_i32, View, ctypes.c_float, View, _P(BackendC)]),
    "rectri_cu_scale_f64": (ctypes.c_int, [ctypes.c_double, View, _P(BackendC)]),
    "rectri_cu_scale_f32": (ctypes.c_int, [ctypes.c_float, View, _P(BackendC)]),
    "rectri_cu_schema_for": (ctypes.c_int, [c_i32, _P(Spec), _P(ctypes.c_double)]),
    "rectri_cu_sync": (ctypes.c_int, [ctypes.c_void_p, _P(c_i64)]),
    "rectri_cu_last_error": (ctypes.c_char_p, []),
    "rectri_cu_launch_count": (c_i64, []),
    "rectri_cu_clear_graph_cache": (None, []),
    "rectri_cu_release_staging": (None, []),
    "rectri_cu_device_bytes_held": (c_i64, []),
    "rectri_cu_abi_version": (ctypes.c_int, []),
    "rectri_cu_fill_uniform": (ctypes.c_int, [c_i32, View, c_i64, c_i64, ctypes.c_uint64, _P(BackendC)]),
    "rectri_cu_make_dominant": (ctypes.c_int, [c_i32, View, c_i32, _P(BackendC)]),
    "rectri_cu_probe_peak": (ctypes.c_double, [c_i32]),
    "rectri_cu_debug_ring_check": (c_i64, [c_i32]),
    "rectri_cu_profile_enable": (None, [c_i32]),
    "rectri_cu_profile_read": (ctypes.c_int, [_P(ctypes.c_double), _P(c_i64), _P(ctypes.c_double)]),
    "rectri_cu_bench_inputs_f64": (None, [ctypes.c_void_p, ctypes.c_void_p, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32,
                                          ctypes.c_uint64]),
    "rectri_cu_bench_inputs_f32": (None, [ctypes.c_void_p, ctypes.c_void_p, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32,
                                          ctypes.c_uint64]),
    "rectri_cu_gate_columns": (c_i32, [ctypes.c_uint64, c_i64, _P(c_i64)]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Loads the in-tree library (building it first if ``RECTRI_CU_AUTOBUILD``
    is set).  Raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() and os.environ.get("RECTRI_CU_AUTOBUILD"):
        from . import build as _build

        _build.build()
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: run `python -m paper_2504_13821_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().rectri_cu_last_error()
    return msg.decode() if msg else ""
