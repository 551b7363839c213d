"""C4: all 16 side/uplo/trans/diag variants of TRSM and TRMM at n = m = 4096
(fp64 and fp32), graph-replayed, CUDA events, best of 3 -- GFLOP/s = n^2 m / t
(bench.cpp:215-217), the reference's residual gate per variant
(bench.cpp:100-165: 8 sampled output columns, |op(A)X - alpha B| for TRSM,
|X - alpha op(A) B| for TRMM, bound 64 n eps * scale, computed here in torch
fp64 on the device) with an explicit finiteness check, and cuBLAS ?trsm /
?trmm on the same inputs.  Prints one JSON line per (op, dtype, variant);
exits 1 if any gate fails."""
import itertools
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import (Backend, Diag, MatrixBuffer, Side, Threshold, Trans,  # noqa: E402
                                   TriangularSpec, Uplo)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dtypes = [torch.float64, torch.float32] if len(sys.argv) < 3 else [
    torch.float64 if sys.argv[2] == "f64" else torch.float32]


def masked_op(A, uplo, trans, diag, n):
    """op(A) through the stored triangle (diag 1 for Unit), fp64."""
    a = A.data.t().double()
    m = torch.tril(a) if uplo == 0 else torch.triu(a)
    if diag == 1:
        m = m - torch.diag(torch.diagonal(m)) + torch.eye(n, dtype=torch.float64, device=m.device)
    return m.t() if trans else m


def gate(op, side, uplo, trans, diag, A, B0, B, n, dt, alpha=1.0):
    """bench.cpp:100-165 on 8 sampled output columns (the reference samples
    result columns for both sides)."""
    g = torch.Generator().manual_seed(1000 + 16 * side + 8 * uplo + 4 * trans + 2 * diag + (op == "trsm"))
    cols = torch.randint(0, n, (8,), generator=g).cuda()
    opa = masked_op(A, uplo, trans, diag, n)
    X = B.data.t().double()  # rows x cols
    B0d = B0.data.t().double()
    a_norm = opa.abs().sum(1).max().item()
    eps = torch.finfo(dt).eps
    if op == "trsm":
        lhs = (opa @ X[:, cols]) if side == 0 else (X @ opa[:, cols])
        r = lhs - alpha * B0d[:, cols]
        scale = a_norm * X.abs().max().item() + abs(alpha) * B0d.abs().max().item()
    else:
        ref = (opa @ B0d[:, cols]) if side == 0 else (B0d @ opa[:, cols])
        r = X[:, cols] - alpha * ref
        scale = (1.0 + abs(alpha)) * a_norm * B0d.abs().max().item()
    return float(r.abs().max().item()), 64.0 * n * eps * scale


def cublas_ms(op, side, uplo, trans, diag, A, B0, n, dt):
    import ctypes

    lib = ctypes.CDLL(str(Path(__file__).resolve().parents[1] / "tools" / "libcublas_cmp.so"))
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    d = 1 if dt == torch.float64 else 0
    work = B0.data.clone()
    if op == "trsm":
        f = lib.cmp_trsm
        f.argtypes = [i32, i32, i32, i32, i32, vp, i64, vp, i64, i64, i32]
        f.restype = ctypes.c_double
        return f(d, side, uplo, trans, diag, A.data.data_ptr(), n, work.data_ptr(), n, n, 3)
    out = torch.empty_like(work)
    f = lib.cmp_trmm
    f.argtypes = [i32, i32, i32, i32, i32, vp, i64, vp, vp, i64, i64, i32]
    f.restype = ctypes.c_double
    return f(d, side, uplo, trans, diag, A.data.data_ptr(), n, work.data_ptr(), out.data_ptr(), n, n, 3)


failures = 0
for dt in dtypes:
    A = MatrixBuffer(n, n, dt, "cuda")
    B0 = MatrixBuffer(n, n, dt, "cuda")
    B = MatrixBuffer(n, n, dt, "cuda")
    rc.fill_uniform(B0.view(), seed=2)
    for op in ("trsm", "trmm"):
        for side, uplo, trans, diag in itertools.product((0, 1), (0, 1), (0, 1), (0, 1)):
            rc.fill_uniform(A.view(), seed=1)
            if op == "trsm":
                rc.make_dominant(A.view(), Uplo(uplo))
                if diag == 1:  # test_support.hpp:52-70: damp the off-diagonal for Unit TRSM
                    t = A.data.t()
                    d = torch.diagonal(t).clone()
                    t.mul_(1.0 / n)
                    torch.diagonal(t).copy_(d)
            spec = TriangularSpec(Side(side), Uplo(uplo), Trans(trans), Diag(diag), 1.0)
            fn = rc.rec_trsm if op == "trsm" else rc.rec_trmm
            best = 1e30
            for it in range(4):
                B.data.copy_(B0.data)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn(spec, A.cview(), B.view(), Threshold(256), Backend.cuda())
                e1.record()
                torch.cuda.synchronize()
                if it:
                    best = min(best, e0.elapsed_time(e1))
            finite = bool(torch.isfinite(B.data).all().item())
            worst, tol = gate(op, side, uplo, trans, diag, A, B0, B, n, dt)
            ok = finite and worst <= tol
            failures += 0 if ok else 1
            cb = cublas_ms(op, side, uplo, trans, diag, A, B0, n, dt)
            print(json.dumps({"op": op, "dtype": str(dt).split(".")[-1], "side": "LR"[side], "uplo": "LU"[uplo],
                              "trans": "NT"[trans], "diag": "NU"[diag], "n": n, "ms": round(best, 4),
                              "gflops": round(n ** 3 / (best * 1e-3) / 1e9, 1), "finite": finite,
                              "gate": {"residual": worst, "tol": tol, "pass": ok},
                              "cublas_ms": round(cb, 4), "cublas_gflops": round(n ** 3 / (cb * 1e-3) / 1e9, 1),
                              "vs_cublas": round(cb / best, 3)}), flush=True)
sys.exit(1 if failures else 0)
