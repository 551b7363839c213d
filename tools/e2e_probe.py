"""C3 end to end (host-pinned A and B through rec_trsm) wall time, for tuning
the streamed host path; never a bench number.
    RECTRI_CU_E2E_TRACE=1 RECTRI_CU_E2E_PANELS=2 python tools/e2e_probe.py [n] [m] [reps]
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import Backend, MatrixBuffer, Threshold, TriangularSpec  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
f64 = torch.float64
A = MatrixBuffer(n, n, f64, "cuda")
rc.fill_uniform(A.view(), seed=1)
rc.make_dominant(A.view())
B = MatrixBuffer(n, m, f64, "cuda")
rc.fill_uniform(B.view(), seed=2)
torch.cuda.synchronize()
Ah = torch.empty((n, n), dtype=f64, pin_memory=True)
Ah.copy_(A.data)
Bh0 = torch.empty((m, n), dtype=f64, pin_memory=True)
Bh0.copy_(B.data)
Bh = torch.empty((m, n), dtype=f64, pin_memory=True)
del A, B
torch.cuda.empty_cache()
# raw PCIe: 1 GiB pinned -> device and back
x = torch.empty(1 << 27, dtype=f64, device="cuda")
h = Bh0.view(-1)[: 1 << 27]
for kind in ("h2d", "d2h"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        (x.copy_(h, non_blocking=True) if kind == "h2d" else h.copy_(x, non_blocking=True))
    torch.cuda.synchronize()
    print(f"{kind} {3 * 8 * (1 << 27) / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
del x
Av = rc.MatrixView(Ah, n, n).as_const()
Bv = rc.MatrixView(Bh, n, m)
be = Backend.cuda()
for i in range(reps):
    Bh.copy_(Bh0)
    t0 = time.perf_counter()
    rc.rec_trsm(TriangularSpec(), Av, Bv, Threshold(256), be)
    w = time.perf_counter() - t0
    print(f"rep {i}: {w * 1e3:.1f} ms  {n * n * m / w / 1e12:.2f} TF/s", flush=True)
