"""Times the fp64/fp32 GEMM update at the recursion's level shapes (CUDA
events, device-resident, best of 3).  RECTRI_CU_GEMM64 selects the fp64
tile variant.  Usage: python tools/gemm_bench.py [f64|f32] [N]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import NO_GRAPH, Backend, MatrixBuffer, Trans  # noqa: E402

dt = torch.float64 if (len(sys.argv) < 2 or sys.argv[1] == "f64") else torch.float32
N = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
be = Backend.cuda(flags=NO_GRAPH)
res = []
for MK in (8192, 4096, 2048, 1024, 512, 256, 128, 64):
    for ta, tb, tag in ((0, 0, "NN"), (1, 0, "TN"), (0, 1, "NT"), (1, 1, "TT")):
        M = K = MK
        A = MatrixBuffer(K if ta else M, M if ta else K, dt, "cuda")
        B = MatrixBuffer(N, K, dt, "cuda") if tb else MatrixBuffer(K, N, dt, "cuda")
        C = MatrixBuffer(M, N, dt, "cuda")
        for i, x in enumerate((A, B, C)):
            rc.fill_uniform(x.view(), seed=i)
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
        res.append((tag, M, N, K, best, tf))
        print(f"{tag} M=K={MK:5d} N={N}: {best:9.3f} ms  {tf:6.2f} TF/s", flush=True)
print("peak probe", rc.probe_peak("f64" if dt == torch.float64 else "f32"))
