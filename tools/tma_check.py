"""TMA DMMA GEMM: bitwise parity against the cp.async kernel on ragged
shapes and sub-views, then timing of each configuration at the recursion's
level shapes (CUDA events, best of 3).  Tuning tool, not a bench number.

    python tools/tma_check.py [check] [time] [cfgs=1,2,...] [N=16384]
"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import NO_GRAPH, Backend, MatrixBuffer, Trans  # noqa: E402

args = sys.argv[1:]
cfgs = [1, 2, 3, 4, 5, 6, 7]
N = 16384
for a in args:
    if a.startswith("cfgs="):
        cfgs = [int(x) for x in a[5:].split(",")]
    if a.startswith("N="):
        N = int(a[2:])
be = Backend.cuda(flags=NO_GRAPH)
f64 = torch.float64


if "check" in args:
    bad = 0
    shapes = [(130, 70, 50), (64, 64, 16), (256, 512, 300), (1000, 1000, 1000), (77, 129, 33), (8, 8, 1),
              (200, 24, 257), (512, 256, 256)]
    for (M, N_, K) in shapes:
        for ta in (0, 1):
            for tb in (0, 1):
                for off in (0, 2, 1):
                    Ar, Ac = (K, M) if ta else (M, K)
                    Br, Bc = (N_, K) if tb else (K, N_)
                    A = MatrixBuffer(Ar + 3, Ac + 3, f64, "cuda")
                    B = MatrixBuffer(Br + 3, Bc + 3, f64, "cuda")
                    C = MatrixBuffer(M + 2, N_ + 1, f64, "cuda")
                    rc.fill_uniform(A.view(), seed=1)
                    rc.fill_uniform(B.view(), seed=2)
                    rc.fill_uniform(C.view(), seed=3)
                    Av = A.view().subview(off, 1, Ar, Ac).as_const()
                    Bv = B.view().subview(off, 2, Br, Bc).as_const()
                    for beta in (1.0, 0.0):
                        outs = []
                        for cfg in [0] + cfgs:
                            os.environ["RECTRI_CU_GEMM64_TMA"] = str(cfg)
                            rc.fill_uniform(C.view(), seed=3)
                            Cv = C.view().subview(1, 0, M, N_)
                            rc.gemm(-1.0, Trans(ta), Av, Trans(tb), Bv, beta, Cv, be)
                            torch.cuda.synchronize()
                            outs.append(C.data.clone())
                        for cfg, o in zip(cfgs, outs[1:]):
                            if not torch.equal(o, outs[0]):
                                bad += 1
                                d = (o - outs[0]).abs().max().item()
                                print(f"MISMATCH cfg={cfg} M={M} N={N_} K={K} ta={ta} tb={tb} off={off} beta={beta} maxdiff={d}")
    print("check done, mismatches:", bad, flush=True)

if "time" in args:
    for MK in (8192, 4096, 2048, 1024, 512, 256):
        for ta, tb, tag in ((0, 0, "NN"), (1, 0, "TN"), (0, 1, "NT")):
            M = K = MK
            A = MatrixBuffer(K if ta else M, M if ta else K, f64, "cuda")
            B = MatrixBuffer(N, K, f64, "cuda") if tb else MatrixBuffer(K, N, f64, "cuda")
            C = MatrixBuffer(M, N, f64, "cuda")
            for i, x in enumerate((A, B, C)):
                rc.fill_uniform(x.view(), seed=i)
            line = f"{tag} M=K={MK:5d} N={N}:"
            for cfg in [0] + cfgs:
                os.environ["RECTRI_CU_GEMM64_TMA"] = str(cfg)
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
                tf = 2.0 * M * N * K / (best * 1e-3) / 1e12
                line += f"  c{cfg}:{tf:6.2f}"
            print(line + "  TF/s", flush=True)
