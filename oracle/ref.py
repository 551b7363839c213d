"""TEST INFRASTRUCTURE ONLY -- ctypes access to the reference library itself
(oracle/_ref/librectri_ref.so, compiled by oracle/Makefile from the
untouched sources under /root/reference/proj; see oracle/ref_shim.cpp).

Used to generate golden fixtures (tests/golden/make_golden.py), to pin the
C restatement, and as the CPU baseline (bench.py cpu_baseline and
``--impl reference``).  Never imported by the product.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Tuple

import numpy as np

from . import REF_SO, _flags

_c_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_ip = ctypes.POINTER(ctypes.c_int64)

_lib = None


def available() -> bool:
    return REF_SO.exists()


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        L = ctypes.CDLL(str(REF_SO))
        for pre, ptr in (("f64", _dp), ("f32", _fp)):
            for op in ("trsm", "trmm"):
                getattr(L, f"rref_rec_{op}_{pre}").argtypes = [ctypes.c_int] * 4 + [
                    ctypes.c_double, ptr, _c_i64, ptr, _c_i64, _c_i64, _c_i64, ctypes.c_int, _ip, _c_i64, _ip, _ip]
                getattr(L, f"rref_{op}_base_{pre}").argtypes = [ctypes.c_int] * 4 + [
                    ctypes.c_double, ptr, _c_i64, ptr, _c_i64, _c_i64, _c_i64, ctypes.c_int, _ip]
                getattr(L, f"rref_oracle_{op}_{pre}").argtypes = [ctypes.c_int] * 4 + [
                    ctypes.c_double, ptr, _c_i64, ptr, _c_i64, _c_i64, _dp, _ip]
            getattr(L, f"rref_make_random_{pre}").argtypes = [ptr, _c_i64, _c_i64, ctypes.c_uint64,
                                                              ctypes.c_double, ctypes.c_double]
            getattr(L, f"rref_make_dominant_{pre}").argtypes = [ptr, _c_i64, ctypes.c_int, ctypes.c_uint64]
            getattr(L, f"rref_damp_off_diagonal_{pre}").argtypes = [ptr, _c_i64, ctypes.c_double]
        L.rref_gemm_f64.argtypes = [ctypes.c_double, ctypes.c_int, _dp, _c_i64, _c_i64, ctypes.c_int, _dp,
                                    _c_i64, _c_i64, ctypes.c_double, _dp, _c_i64, _c_i64, ctypes.c_int]
        L.rref_schema_for.argtypes = [ctypes.c_int] * 4 + [_dp]
        L.rref_last_error.restype = ctypes.c_char_p
        L.rref_masked_norm_inf_f64.argtypes = [_dp, _c_i64, ctypes.c_int, ctypes.c_int]
        L.rref_masked_norm_inf_f64.restype = ctypes.c_double
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags.f_contiguous
    return a.ctypes.data_as(_dp if a.dtype == np.float64 else _fp)


def _sfx(a) -> str:
    return "f64" if a.dtype == np.float64 else "f32"


def last_error() -> str:
    return lib().rref_last_error().decode()


def rec(op: str, spec, a: np.ndarray, b: np.ndarray, threshold: int, width: int = 0,
        trace: bool = False) -> Tuple[int, np.ndarray, List[Tuple[int, int, int]], int]:
    """Runs rectri::rec_{op}<T> on copies; returns (status, B_out, events,
    singular_row).  width 0 = Backend::seq(), k > 0 = Backend::par(k), -1 =
    Backend::par() (hardware concurrency)."""
    side, uplo, trans, diag, alpha = _flags(spec)
    a = np.asfortranarray(a)
    out = np.array(b, dtype=a.dtype, order="F", copy=True)
    cap = 1 << 16 if trace else 0
    buf = np.zeros(3 * max(cap, 1), dtype=np.int64)
    cnt = ctypes.c_int64(0)
    row = ctypes.c_int64(-1)
    st = getattr(lib(), f"rref_rec_{op}_{_sfx(a)}")(
        side, uplo, trans, diag, alpha, _ptr(a), a.shape[0], _ptr(out), out.shape[0], out.shape[1], threshold,
        width, buf.ctypes.data_as(_ip) if trace else None, cap, ctypes.byref(cnt) if trace else None,
        ctypes.byref(row))
    events = [tuple(int(x) for x in buf[3 * i: 3 * i + 3]) for i in range(min(cnt.value, cap))]
    return st, out, events, row.value


def base(op: str, spec, a: np.ndarray, b: np.ndarray, tile_limit: int = 256, width: int = 0):
    side, uplo, trans, diag, alpha = _flags(spec)
    a = np.asfortranarray(a)
    out = np.array(b, dtype=a.dtype, order="F", copy=True)
    row = ctypes.c_int64(-1)
    st = getattr(lib(), f"rref_{op}_base_{_sfx(a)}")(side, uplo, trans, diag, alpha, _ptr(a), a.shape[0],
                                                      _ptr(out), out.shape[0], out.shape[1], tile_limit, width,
                                                      ctypes.byref(row))
    return st, out, row.value


def oracle(op: str, spec, a: np.ndarray, b: np.ndarray):
    side, uplo, trans, diag, alpha = _flags(spec)
    a = np.asfortranarray(a)
    b = np.asfortranarray(b, dtype=a.dtype)
    out = np.zeros(b.shape, order="F")
    row = ctypes.c_int64(-1)
    st = getattr(lib(), f"rref_oracle_{op}_{_sfx(a)}")(side, uplo, trans, diag, alpha, _ptr(a), a.shape[0],
                                                        _ptr(b), b.shape[0], b.shape[1],
                                                        out.ctypes.data_as(_dp), ctypes.byref(row))
    return st, out, row.value


def gemm(alpha: float, ta: int, a: np.ndarray, tb: int, b: np.ndarray, beta: float, c: np.ndarray, width=0):
    out = np.array(c, dtype=np.float64, order="F", copy=True)
    a = np.asfortranarray(a, dtype=np.float64)
    b = np.asfortranarray(b, dtype=np.float64)
    st = lib().rref_gemm_f64(alpha, ta, _ptr(a), a.shape[0], a.shape[1], tb, _ptr(b), b.shape[0], b.shape[1],
                             beta, _ptr(out), out.shape[0], out.shape[1], width)
    return st, out


def schema_for(op: str, spec) -> np.ndarray:
    out = np.zeros(8)
    lib().rref_schema_for(1 if op == "trsm" else 0, int(spec.side), int(spec.uplo), int(spec.trans),
                          out.ctypes.data_as(_dp))
    return out


def make_random(rows, cols, seed, lo=-1.0, hi=1.0, dtype=np.float64):
    a = np.zeros((rows, cols), dtype=dtype, order="F")
    getattr(lib(), f"rref_make_random_{_sfx(a)}")(_ptr(a), rows, cols, seed, lo, hi)
    return a


def make_dominant(n, uplo, seed, dtype=np.float64):
    a = np.zeros((n, n), dtype=dtype, order="F")
    getattr(lib(), f"rref_make_dominant_{_sfx(a)}")(_ptr(a), n, int(uplo), seed)
    return a


def damp_off_diagonal(a: np.ndarray, factor: float) -> None:
    getattr(lib(), f"rref_damp_off_diagonal_{_sfx(a)}")(_ptr(a), a.shape[0], factor)


def masked_norm_inf(a: np.ndarray, uplo: int, diag: int) -> float:
    a = np.asfortranarray(a, dtype=np.float64)
    return float(lib().rref_masked_norm_inf_f64(_ptr(a), a.shape[0], int(uplo), int(diag)))
