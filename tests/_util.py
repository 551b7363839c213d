"""Shared test helpers: numpy (column-major) <-> device MatrixBuffer, and the
reference's tolerance formulas."""
from __future__ import annotations

import numpy as np
import torch

import oracle
from paper_2504_13821_b200 import (
    Backend,
    Diag,
    MatrixBuffer,
    Side,
    Threshold,
    Trans,
    TriangularSpec,
    Uplo,
    rec_trmm,
    rec_trsm,
    trmm_base,
    trsm_base,
)

EPS = {np.float64: np.finfo(np.float64).eps, np.float32: np.finfo(np.float32).eps}


def tspec(s) -> TriangularSpec:
    return TriangularSpec(Side(int(s.side)), Uplo(int(s.uplo)), Trans(int(s.trans)), Diag(int(s.diag)),
                          float(s.alpha))


def to_dev(a: np.ndarray, device="cuda") -> MatrixBuffer:
    return MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a)), device=device)


def to_np(m: MatrixBuffer) -> np.ndarray:
    return np.asfortranarray(m.numpy())


def run_op(op: str, s, a: np.ndarray, b: np.ndarray, threshold: int, backend=None, sink=None,
           device="cuda") -> np.ndarray:
    A = to_dev(a, device)
    B = to_dev(b, device)
    fn = rec_trmm if op == "trmm" else rec_trsm
    fn(tspec(s), A.cview(), B.view(), Threshold(threshold), backend or Backend.cuda(), sink)
    return to_np(B)


def run_base(op: str, s, a, b, tile_limit=256, device="cuda") -> np.ndarray:
    A = to_dev(a, device)
    B = to_dev(b, device)
    fn = trmm_base if op == "trmm" else trsm_base
    fn(tspec(s), A.cview(), B.view(), tile_limit)
    return to_np(B)


def tol_scale(s, a, b, got) -> float:
    """acceptance_main.cpp:82-92 scale factor."""
    return (oracle.masked_norm_inf(a, s.uplo, s.diag) * max(oracle.max_abs(b), oracle.max_abs(got), 1.0)
            * max(1.0, abs(s.alpha)))


def check_against_oracle(op: str, s, a, b, got, factor: float = 32.0) -> float:
    """Criterion-1 check: TRMM |got - oracle| and TRSM |op(A) X - alpha B|
    bounded by factor * n * eps * scale.  Returns the normalised error."""
    n = a.shape[0]
    eps = EPS[a.dtype.type]
    assert np.all(np.isfinite(got)), "non-finite output"
    if op == "trmm":
        err = oracle.max_abs_diff(got, oracle.oracle_trmm(s, a, b))
    else:
        err = oracle.trsm_residual_inf(s, a, got, b)
    bound = factor * max(n, 1) * eps * tol_scale(s, a, b, got)
    assert err <= bound, f"{op} {s}: err {err:.3e} > {bound:.3e}"
    return err / (max(n, 1) * eps * tol_scale(s, a, b, got))
