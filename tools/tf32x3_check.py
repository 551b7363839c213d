"""3xTF32 tcgen05 GEMM (RECTRI_CU_FP32_TF32X3=1): error against an fp64
reference next to the FFMA kernel's, on every transpose form and ragged
shapes; then timing at the level shapes.  Tuning/validation tool.

    python tools/tf32x3_check.py [check] [time]
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import NO_GRAPH, Backend, MatrixBuffer, Trans  # noqa: E402

be = Backend.cuda(flags=NO_GRAPH)
args = sys.argv[1:] or ["check"]
f32 = torch.float32


def run(ta, tb, a, b, c0, alpha, beta, mode):
    os.environ["RECTRI_CU_FP32_TF32X3"] = mode
    A = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a)), device="cuda")
    B = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(b)), device="cuda")
    C = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(c0)), device="cuda")
    rc.gemm(alpha, Trans(ta), A.cview(), Trans(tb), B.cview(), beta, C.view(), be)
    torch.cuda.synchronize()
    return np.asfortranarray(C.numpy())


if "check" in args:
    rng = np.random.default_rng(0)
    worst = 0.0
    for M, N, K in ((128, 256, 32), (256, 512, 64), (300, 260, 100), (1024, 1000, 512), (128, 256, 8), (96, 40, 36)):
        for ta in (0, 1):
            for tb in (0, 1):
                a = np.asfortranarray(rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32))
                b = np.asfortranarray(rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32))
                c = np.asfortranarray(rng.uniform(-1, 1, (M, N)).astype(np.float32))
                opa = (a.T if ta else a).astype(np.float64)
                opb = (b.T if tb else b).astype(np.float64)
                ref = -1.0 * (opa @ opb) + c.astype(np.float64)
                got = run(ta, tb, a, b, c, -1.0, 1.0, "1")
                ffma = run(ta, tb, a, b, c, -1.0, 1.0, "0")
                e3 = np.max(np.abs(got - ref)) / (K * np.finfo(np.float32).eps)
                ef = np.max(np.abs(ffma - ref)) / (K * np.finfo(np.float32).eps)
                worst = max(worst, e3)
                print(f"M={M} N={N} K={K} ta={ta} tb={tb}: tf32x3 err {e3:.3f} K*eps, ffma {ef:.3f}", flush=True)
    print("worst tf32x3 error (units of K*eps_fp32):", worst)

if "time" in args:
    N = 16384
    for MK in (8192, 4096, 2048, 1024, 512, 256):
        for ta, tb, tag in ((0, 0, "NN"), (1, 0, "TN"), (0, 1, "NT")):
            M = K = MK
            A = MatrixBuffer(K if ta else M, M if ta else K, f32, "cuda")
            B = MatrixBuffer(N, K, f32, "cuda") if tb else MatrixBuffer(K, N, f32, "cuda")
            C = MatrixBuffer(M, N, f32, "cuda")
            for i, x in enumerate((A, B, C)):
                rc.fill_uniform(x.view(), seed=i)
            line = f"{tag} M=K={MK:5d} N={N}:"
            for mode in ("0", "1"):
                os.environ["RECTRI_CU_FP32_TF32X3"] = mode
                f = lambda: rc.gemm(-1.0, Trans(ta), A.cview(), Trans(tb), B.cview(), 1.0, C.view(), be)
                f()
                best = 1e30
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    f()
                    e1.record()
                    torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1))
                line += f"  {'tf32x3' if mode == '1' else 'ffma'}: {2.0 * M * N * K / (best * 1e-3) / 1e12:6.1f}"
            print(line + " TF/s", flush=True)
