"""Times one recursive call (graph replay, device-resident, CUDA events,
B restored outside the events; best of `reps`).  Tuning tool, not the bench.

    python tools/trsm_time.py [trsm|trmm] [n] [m] [f64|f32] [threshold] [reps]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import Backend, MatrixBuffer, Threshold, TriangularSpec  # noqa: E402

a = sys.argv[1:]
op = a[0] if a else "trsm"
n = int(a[1]) if len(a) > 1 else 16384
m = int(a[2]) if len(a) > 2 else n
dt = torch.float32 if len(a) > 3 and a[3] == "f32" else torch.float64
t = int(a[4]) if len(a) > 4 else 256
reps = int(a[5]) if len(a) > 5 else 3
A = MatrixBuffer(n, n, dt, "cuda")
rc.fill_uniform(A.view(), seed=1)
rc.make_dominant(A.view())
B0 = MatrixBuffer(n, m, dt, "cuda")
rc.fill_uniform(B0.view(), seed=2)
B = MatrixBuffer(n, m, dt, "cuda")
fn = rc.rec_trsm if op == "trsm" else rc.rec_trmm
spec = TriangularSpec()
be = Backend.cuda()
best = 1e30
for i in range(reps + 1):
    B.data.copy_(B0.data)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(spec, A.cview(), B.view(), Threshold(t), be)
    e1.record()
    torch.cuda.synchronize()
    if i:
        best = min(best, e0.elapsed_time(e1))
print(f"{op} n={n} m={m} {dt} t={t}: {best:8.2f} ms  {n * n * m / (best * 1e-3) / 1e12:6.2f} TF/s", flush=True)
