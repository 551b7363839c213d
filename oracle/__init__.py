"""TEST INFRASTRUCTURE ONLY -- the parity referee.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the CPU baseline.
The product (paper_2504_13821_b200/) never imports it.

Two libraries live behind this module:

* ``_build/librectri_oracle.so`` -- oracle/rectri_oracle.c, a plain-C
  restatement of the reference's oracle (src/oracle.cpp:39-137) and input
  generators (tests/test_support.hpp:38-85, src/bench.cpp:32-61); and
* ``_ref/librectri_ref.so`` -- the reference library itself, compiled from
  its untouched sources under /root/reference by oracle/Makefile (absent on a
  box without the reference; it travels to the GPU box as a built file).

Parity of the restatement is pinned against the reference by
tests/test_oracle_golden.py (fixtures from tests/golden/make_golden.py).

Matrices are numpy arrays of shape (rows, cols) in Fortran (column-major)
order.  ``spec`` arguments are any object with side/uplo/trans/diag/alpha
attributes (ints 0/1, trans 0/1/2), as in include/rectri_cu.h.
"""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "librectri_oracle.so"
REF_SO = HERE / "_ref" / "librectri_ref.so"
REFERENCE_SRC = Path("/root/reference/proj")

RO_OK, RO_SHAPE, RO_SINGULAR = 0, 2, 4

_c_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_ip = ctypes.POINTER(ctypes.c_int64)


class OracleSingular(Exception):
    def __init__(self, index: int):
        super().__init__(f"singular triangular matrix: zero diagonal at row {index}")
        self.index = index


def build(ref: bool = True) -> None:
    """Compiles the C restatement, and the reference library when its sources
    are present (never needed on the GPU box: the built files travel)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"], check=True)
    if ref and REFERENCE_SRC.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


_lib = None
_ref = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        L = ctypes.CDLL(str(ORACLE_SO))
        for pre, ptr in (("f64", _dp), ("f32", _fp)):
            getattr(L, f"ro_make_random_{pre}").argtypes = [ptr, _c_i64, _c_i64, ctypes.c_uint64,
                                                            ctypes.c_double, ctypes.c_double]
            getattr(L, f"ro_make_dominant_{pre}").argtypes = [ptr, _c_i64, ctypes.c_int, ctypes.c_uint64]
            getattr(L, f"ro_damp_off_diagonal_{pre}").argtypes = [ptr, _c_i64, ctypes.c_double]
            getattr(L, f"ro_oracle_trmm_{pre}").argtypes = [ctypes.c_int] * 4 + [
                ctypes.c_double, ptr, _c_i64, _c_i64, ptr, _c_i64, _c_i64, _c_i64, _dp]
            getattr(L, f"ro_oracle_trsm_{pre}").argtypes = [ctypes.c_int] * 4 + [
                ctypes.c_double, ptr, _c_i64, _c_i64, ptr, _c_i64, _c_i64, _c_i64, _dp, _ip]
        L.ro_bench_inputs_f64.argtypes = [_dp, _dp, _c_i64, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_uint64]
        L.ro_oracle_cols_f64.argtypes = [ctypes.c_int] * 4 + [ctypes.c_double, _dp, _c_i64, _c_i64, _dp,
                                                               _c_i64, _ip, _c_i64, _dp, _ip]
        L.ro_masked_norm_inf_f64.argtypes = [_dp, _c_i64, _c_i64, ctypes.c_int, ctypes.c_int]
        L.ro_masked_norm_inf_f64.restype = ctypes.c_double
        L.ro_trsm_residual_inf_f64.argtypes = [ctypes.c_int] * 4 + [ctypes.c_double, _dp, _c_i64, _c_i64, _dp,
                                                                     _c_i64, _dp, _c_i64, _c_i64, _c_i64]
        L.ro_trsm_residual_inf_f64.restype = ctypes.c_double
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags.f_contiguous, "column-major array expected"
    return a.ctypes.data_as(_dp if a.dtype == np.float64 else _fp)


def _sfx(dtype) -> str:
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def _flags(spec):
    return int(spec.side), int(spec.uplo), int(spec.trans), int(spec.diag), float(spec.alpha)


# ---------------------------------------------------------------- generators
def make_random(rows: int, cols: int, seed: int, lo: float = -1.0, hi: float = 1.0, dtype=np.float64):
    """tests/test_support.hpp:38-47 (mt19937_64, uniform_real_distribution)."""
    a = np.zeros((rows, cols), dtype=dtype, order="F")
    getattr(lib(), f"ro_make_random_{_sfx(dtype)}")(_ptr(a), rows, cols, seed, lo, hi)
    return a


def make_dominant(n: int, uplo: int, seed: int, dtype=np.float64):
    """tests/test_support.hpp:52-62."""
    a = np.zeros((n, n), dtype=dtype, order="F")
    getattr(lib(), f"ro_make_dominant_{_sfx(dtype)}")(_ptr(a), n, int(uplo), seed)
    return a


def damp_off_diagonal(a: np.ndarray, factor: float) -> None:
    """tests/test_support.hpp:66-70 (in place)."""
    getattr(lib(), f"ro_damp_off_diagonal_{_sfx(a.dtype)}")(_ptr(a), a.shape[0], factor)


def bench_inputs(n: int, brows: int, bcols: int, is_trsm: bool, uplo: int, diag: int, seed: int):
    """src/bench.cpp:32-61 (fp64)."""
    a = np.zeros((n, n), order="F")
    b = np.zeros((brows, bcols), order="F")
    lib().ro_bench_inputs_f64(_ptr(a), _ptr(b), n, brows, bcols, int(is_trsm), int(uplo), int(diag), seed)
    return a, b


def poison_opposite_triangle(a: np.ndarray, uplo: int) -> None:
    """tests/test_support.hpp:73-80"""
    n = a.shape[0]
    r, c = np.indices((n, n))
    stored = r >= c if int(uplo) == 0 else r <= c
    a[~stored] = np.nan


def set_diagonal(a: np.ndarray, value: float) -> None:
    """tests/test_support.hpp:83-85"""
    np.fill_diagonal(a, value)


def make_operand(spec, is_trsm: bool, n: int, seed: int, dtype=np.float64):
    """The conditioned triangular operand of test_recursion.cpp:35-44 and
    acceptance_main.cpp:41-49."""
    if is_trsm:
        a = make_dominant(n, spec.uplo, seed, dtype)
        if int(spec.diag) == 1:
            damp_off_diagonal(a, 1.0 / n)
        return a
    return make_random(n, n, seed, dtype=dtype)


def make_rhs(spec, n: int, m: int, seed: int, dtype=np.float64):
    """tests/test_support.hpp:226-230"""
    return make_random(n, m, seed, dtype=dtype) if int(spec.side) == 0 else make_random(m, n, seed, dtype=dtype)


# ------------------------------------------------------------------ oracles
def oracle_trmm(spec, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """src/oracle.cpp:57-82 -- returns float64."""
    side, uplo, trans, diag, alpha = _flags(spec)
    a = np.asfortranarray(a)
    b = np.asfortranarray(b, dtype=a.dtype)
    out = np.zeros(b.shape, order="F")
    rc = getattr(lib(), f"ro_oracle_trmm_{_sfx(a.dtype)}")(side, uplo, trans, diag, alpha, _ptr(a), a.shape[0],
                                                            a.shape[0], _ptr(b), b.shape[0], b.shape[0],
                                                            b.shape[1], _ptr(out))
    if rc != RO_OK:
        raise ValueError("oracle_trmm: shape mismatch")
    return out


def oracle_trsm(spec, a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """src/oracle.cpp:85-137 -- returns float64; raises OracleSingular."""
    side, uplo, trans, diag, alpha = _flags(spec)
    a = np.asfortranarray(a)
    b = np.asfortranarray(b, dtype=a.dtype)
    out = np.zeros(b.shape, order="F")
    row = ctypes.c_int64(-1)
    rc = getattr(lib(), f"ro_oracle_trsm_{_sfx(a.dtype)}")(side, uplo, trans, diag, alpha, _ptr(a), a.shape[0],
                                                            a.shape[0], _ptr(b), b.shape[0], b.shape[0],
                                                            b.shape[1], _ptr(out), ctypes.byref(row))
    if rc == RO_SINGULAR:
        raise OracleSingular(row.value)
    if rc != RO_OK:
        raise ValueError("oracle_trsm: shape mismatch")
    return out


def oracle_cols(is_trsm: bool, spec, a: np.ndarray, b_cols: np.ndarray) -> np.ndarray:
    """Exact per-column oracle for Left problems on a column sample
    (b_cols = n x k gathered columns of B)."""
    side, uplo, trans, diag, alpha = _flags(spec)
    assert side == 0
    a = np.asfortranarray(a, dtype=np.float64)
    b = np.asfortranarray(b_cols, dtype=np.float64)
    n, k = b.shape
    cols = np.arange(k, dtype=np.int64)
    out = np.zeros((n, k), order="F")
    row = ctypes.c_int64(-1)
    rc = lib().ro_oracle_cols_f64(int(is_trsm), uplo, trans, diag, alpha, _ptr(a), a.shape[0], n, _ptr(b), n,
                                  cols.ctypes.data_as(_ip), k, _ptr(out), ctypes.byref(row))
    if rc == RO_SINGULAR:
        raise OracleSingular(row.value)
    return out


# ---------------------------------------------------------------- metrics
def masked_norm_inf(a: np.ndarray, uplo: int, diag: int) -> float:
    """tests/test_support.hpp:129-140"""
    a64 = np.asfortranarray(a, dtype=np.float64)
    return float(lib().ro_masked_norm_inf_f64(_ptr(a64), a64.shape[0], a64.shape[0], int(uplo), int(diag)))


def trsm_residual_inf(spec, a: np.ndarray, x: np.ndarray, b: np.ndarray) -> float:
    """tests/test_support.hpp:182-202 (op(A) X - alpha B, through the mask)."""
    side, uplo, trans, diag, alpha = _flags(spec)
    a64 = np.asfortranarray(a, dtype=np.float64)
    x64 = np.asfortranarray(x, dtype=np.float64)
    b64 = np.asfortranarray(b, dtype=np.float64)
    eff = 0 if trans == 0 else 1
    return float(lib().ro_trsm_residual_inf_f64(side, uplo, eff, diag, alpha, _ptr(a64), a64.shape[0],
                                                a64.shape[0], _ptr(x64), x64.shape[0], _ptr(b64), b64.shape[0],
                                                x64.shape[0], x64.shape[1]))


def max_abs(m) -> float:
    m = np.asarray(m, dtype=np.float64)
    return float(np.max(np.abs(m))) if m.size else 0.0


def max_abs_diff(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b))) if a.size else 0.0


def bitwise_equal(a, b) -> bool:
    """tests/test_support.hpp:110-123 (NaN == NaN)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    return bool(np.all(same))


class _Spec:
    __slots__ = ("side", "uplo", "trans", "diag", "alpha")

    def __init__(self, side=0, uplo=0, trans=0, diag=0, alpha=1.0):
        self.side, self.uplo, self.trans, self.diag, self.alpha = side, uplo, trans, diag, alpha

    def __repr__(self):
        s = ("left", "right")[self.side], ("lower", "upper")[self.uplo], ("n", "t", "c")[self.trans], \
            ("nonunit", "unit")[self.diag]
        return "-".join(s) + f"(alpha={self.alpha})"


def spec(side=0, uplo=0, trans=0, diag=0, alpha=1.0) -> _Spec:
    return _Spec(side, uplo, trans, diag, alpha)


def all_variants(alpha: float = 1.0, include_conj: bool = False):
    """tests/test_support.hpp:210-222 (same order)."""
    out = []
    for side in (0, 1):
        for uplo in (0, 1):
            for trans in ((0, 1, 2) if include_conj else (0, 1)):
                for diag in (0, 1):
                    out.append(_Spec(side, uplo, trans, diag, alpha))
    return out
