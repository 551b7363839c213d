"""Host<->device staging probe for the e2e path: pinned H2D / D2H / duplex
bandwidth, then the host-view rec_trsm wall time per panel width
(RECTRI_CU_HOST_PANEL).  Tuning tool, not a bench number.

    python tools/e2e_probe.py [n] [m] [panel widths...]
"""
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import Backend, Threshold, TriangularSpec  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
widths = [int(x) for x in sys.argv[3:]] or [4096]
f64 = torch.float64
nbytes = 2 << 30
h = torch.empty(nbytes // 8, dtype=f64, pin_memory=True)
h2 = torch.empty(nbytes // 8, dtype=f64, pin_memory=True)
d = torch.empty(nbytes // 8, dtype=f64, device="cuda")
d2 = torch.empty(nbytes // 8, dtype=f64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    print(f"{name}: {nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s", flush=True)
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"duplex: {2 * nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s total", flush=True)
del h, h2, d, d2

A = rc.MatrixBuffer(n, n, f64, "cuda")
rc.fill_uniform(A.view(), seed=1)
rc.make_dominant(A.view())
B = rc.MatrixBuffer(n, m, f64, "cuda")
rc.fill_uniform(B.view(), seed=2)
Ah = torch.empty((n, n), dtype=f64, pin_memory=True)
Ah.copy_(A.data)
Bh0 = torch.empty((m, n), dtype=f64, pin_memory=True)
Bh0.copy_(B.data)
Bh = torch.empty((m, n), dtype=f64, pin_memory=True)
Av = rc.MatrixView(Ah, n, n).as_const()
Bv = rc.MatrixView(Bh, n, m)
be = Backend.cuda()
for w in widths:
    if w:
        os.environ["RECTRI_CU_HOST_PANEL"] = str(w)  # panelled path
    else:
        os.environ.pop("RECTRI_CU_HOST_PANEL", None)  # first-use streamed path
    best = 1e30
    for i in range(3):
        Bh.copy_(Bh0)
        t = time.perf_counter()
        rc.rec_trsm(TriangularSpec(), Av, Bv, Threshold(256), be)
        best = min(best, time.perf_counter() - t)
    print(f"e2e panel={w}: {best * 1e3:.1f} ms  {n * n * m / best / 1e12:.2f} TF/s", flush=True)
