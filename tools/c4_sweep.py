"""C4: all 16 side/uplo/trans/diag variants of TRSM and TRMM at n = m = 4096
(fp64 and fp32), graph-replayed, CUDA events, best of 3 -- GFLOP/s = n^2 m / t
(bench.cpp:215-217) and the residual gate per variant.  Prints one JSON line
per (op, dtype, variant)."""
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
            print(json.dumps({"op": op, "dtype": str(dt).split(".")[-1], "side": "LR"[side], "uplo": "LU"[uplo],
                              "trans": "NT"[trans], "diag": "NU"[diag], "n": n, "ms": round(best, 4),
                              "gflops": round(n ** 3 / (best * 1e-3) / 1e9, 1), "finite": finite}), flush=True)
