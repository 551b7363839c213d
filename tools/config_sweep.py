"""Performance sweeps for BASELINE.json configs other than the headline.

    python tools/config_sweep.py c2   TRMM Left/Upper/NoTrans fp32+fp64, n = m = 256 .. 16384,
                                      leaf (threshold) 32 .. 256
    python tools/config_sweep.py c4   all 16 variants x {trmm, trsm} x {fp32, fp64} at n = m = 4096
    python tools/config_sweep.py t    threshold sweep for the C3 headline (trsm/trmm fp64 16384)

GFLOP/s = n^2 m / t (src/bench.cpp:215-217); device-resident inputs,
best-of-3 CUDA-event time per call (B restored between calls outside the
events).  Inputs follow the reference generators' conditioning: TRSM A is
diagonally dominant (+ off-diagonal damping 1/n for Unit).
Prints one JSON object per line (sweep CSV fields of bench.hpp:64-65).
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import (Backend, Diag, MatrixBuffer, Side, Threshold, Trans,  # noqa: E402
                                   TriangularSpec, Uplo)


def run(op, spec, n, m, t, dt, reps=3):
    A = MatrixBuffer(n, n, dt, "cuda")
    rc.fill_uniform(A.view(), seed=11)
    if op == "trsm":
        rc.make_dominant(A.view(), spec.uplo)
        if spec.diag == Diag.Unit:  # damp_off_diagonal(1/n), keep the diagonal
            d = A.data.diagonal().clone()
            A.data.mul_(1.0 / n)
            A.data.diagonal().copy_(d)
    rows, cols = (n, m) if spec.side == Side.Left else (m, n)
    B0 = MatrixBuffer(rows, cols, dt, "cuda")
    rc.fill_uniform(B0.view(), seed=12)
    B = MatrixBuffer(rows, cols, dt, "cuda")
    fn = rc.rec_trsm if op == "trsm" else rc.rec_trmm
    be = Backend.cuda()
    best = 1e30
    for i in range(reps + 1):
        B.data.copy_(B0.data)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(spec, A.cview(), B.view(), Threshold(t), be)
        e1.record()
        torch.cuda.synchronize()
        if i:
            best = min(best, e0.elapsed_time(e1))
    ok = bool(torch.isfinite(B.data).all().item())
    rc.clear_graph_cache()
    return {"op": op, "variant": rc.variant_string(spec), "n": n, "m": m, "threshold": t,
            "backend": "cuda", "elem": "f64" if dt == torch.float64 else "f32",
            "median_time_s": best * 1e-3, "gflops": float(n) * n * m / (best * 1e-3) / 1e9, "finite": ok}


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c4"
    if which == "c2":
        for dt in (torch.float64, torch.float32):
            for n in (256, 512, 1024, 2048, 4096, 8192, 16384):
                for t in (32, 64, 128, 256):
                    spec = TriangularSpec(Side.Left, Uplo.Upper, Trans.NoTrans, Diag.NonUnit)
                    print(json.dumps(run("trmm", spec, n, n, t, dt)), flush=True)
    elif which == "c4":
        for dt in (torch.float64, torch.float32):
            for op in ("trmm", "trsm"):
                for side in (Side.Left, Side.Right):
                    for uplo in (Uplo.Lower, Uplo.Upper):
                        for tr in (Trans.NoTrans, Trans.Trans):
                            for dg in (Diag.NonUnit, Diag.Unit):
                                spec = TriangularSpec(side, uplo, tr, dg)
                                print(json.dumps(run(op, spec, 4096, 4096, 256, dt)), flush=True)
    elif which == "t":
        for op in ("trsm", "trmm"):
            for t in (64, 128, 256, 512):
                uplo = Uplo.Lower if op == "trsm" else Uplo.Upper
                spec = TriangularSpec(Side.Left, uplo, Trans.NoTrans, Diag.NonUnit)
                print(json.dumps(run(op, spec, 16384, 16384, t, torch.float64, reps=2)), flush=True)


if __name__ == "__main__":
    main()
