"""Times one trsm_base / trmm_base leaf (nb x m, fp64/fp32) with CUDA events.
Usage: python tools/leaf_bench.py [nb] [m] [f64|f32]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import NO_GRAPH, Backend, Diag, MatrixBuffer, TriangularSpec  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
m = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
dt = torch.float32 if len(sys.argv) > 3 and sys.argv[3] == "f32" else torch.float64
A = MatrixBuffer(nb, nb, dt, "cuda")
rc.fill_uniform(A.view(), seed=1)
rc.make_dominant(A.view())
B = MatrixBuffer(nb, m, dt, "cuda")
rc.fill_uniform(B.view(), seed=2)
be = Backend.cuda(flags=NO_GRAPH)
spec = TriangularSpec(diag=Diag.Unit)  # Unit: no pivot pre-scan / host sync inside the timed call
for name, fn in (("trsm", rc.trsm_base), ("trmm", rc.trmm_base)):
    fn(spec, A.cview(), B.view(), nb, be)
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(spec, A.cview(), B.view(), nb, be)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name} nb={nb} m={m} {dt}: {best * 1e3:8.1f} us  {nb * nb * m / (best * 1e-3) / 1e12:6.2f} TF/s", flush=True)
