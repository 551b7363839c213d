"""One-shot workloads for ncu (never a bench number):

    python tools/prof_run.py trsm N M T      one rec_trsm (direct launches; strsm: fp32)
    python tools/prof_run.py gemm M N K      one DMMA GEMM update C -= A*B (NN)
    python tools/prof_run.py leaf NB M       one trsm_base leaf (NB x M)
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import NO_GRAPH, Backend, MatrixBuffer, Threshold, Trans, TriangularSpec  # noqa: E402

kind = sys.argv[1]
args = [int(x) for x in sys.argv[2:]]
f64 = torch.float64
be = Backend.cuda(flags=NO_GRAPH)
if kind in ("trsm", "trmm", "strsm"):
    n, m, t = args
    if kind == "strsm":
        f64 = torch.float32
    A = MatrixBuffer(n, n, f64, "cuda")
    rc.fill_uniform(A.view(), seed=1)
    rc.make_dominant(A.view())
    B = MatrixBuffer(n, m, f64, "cuda")
    rc.fill_uniform(B.view(), seed=2)
    fn = rc.rec_trmm if kind == "trmm" else rc.rec_trsm
    fn(TriangularSpec(), A.cview(), B.view(), Threshold(t), be)
elif kind in ("gemm", "gemmtn", "sgemm", "sgemmtn", "tf32x3"):
    M, N, K = args
    if kind in ("sgemm", "sgemmtn", "tf32x3"):
        f64 = torch.float32
    if kind == "tf32x3":
        be = Backend.cuda(flags=NO_GRAPH | rc.TF32X3)
    ta = Trans.Trans if kind in ("gemmtn", "sgemmtn") else Trans.NoTrans
    A = MatrixBuffer(K, M, f64, "cuda") if ta == Trans.Trans else MatrixBuffer(M, K, f64, "cuda")
    B = MatrixBuffer(K, N, f64, "cuda")
    C = MatrixBuffer(M, N, f64, "cuda")
    for i, x in enumerate((A, B, C)):
        rc.fill_uniform(x.view(), seed=i)
    rc.gemm(-1.0, ta, A.cview(), Trans.NoTrans, B.cview(), 1.0, C.view(), be)
elif kind in ("leaf", "trmmleaf", "leaf32"):
    nb, m = args
    if kind == "leaf32":
        f64 = torch.float32
    A = MatrixBuffer(nb, nb, f64, "cuda")
    rc.fill_uniform(A.view(), seed=1)
    rc.make_dominant(A.view())
    B = MatrixBuffer(nb, m, f64, "cuda")
    rc.fill_uniform(B.view(), seed=2)
    fn = rc.trmm_base if kind == "trmmleaf" else rc.trsm_base
    fn(TriangularSpec(), A.cview(), B.view(), nb, be)
torch.cuda.synchronize()
print("done", kind, args)
