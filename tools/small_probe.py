"""Where the time goes at small n (C2 sweep, n = m = 256..8192): per call,
   sync   events around a synchronous call (what tools/rectri_bench.py times)
   async  events around one RECTRI_CU_ASYNC call (host enqueue + GPU)
   pipe   events around 20 back-to-back ASYNC calls / 20 (GPU-bound if the
          host keeps ahead)
   host   host wall time of one ASYNC enqueue (perf_counter)
   cublas cuBLAS ?trmm/?trsm through tools/libcublas_cmp.so (events inside C)
Never a bench number; run on the GPU box.

    python tools/small_probe.py [trmm|trsm] [f64|f32] [sizes]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import ASYNC, Backend, MatrixBuffer, Threshold, TriangularSpec  # noqa: E402
from paper_2504_13821_b200 import harness  # noqa: E402
from paper_2504_13821_b200.api import Diag, Side, Trans, Uplo  # noqa: E402

op = sys.argv[1] if len(sys.argv) > 1 else "trmm"
elem = sys.argv[2] if len(sys.argv) > 2 else "f64"
sizes = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "256,512,1024,2048,4096,8192").split(",")]
dt = torch.float64 if elem == "f64" else torch.float32
uplo = Uplo.Upper if op == "trmm" else Uplo.Lower
spec = TriangularSpec(Side.Left, uplo, Trans.NoTrans, Diag.NonUnit, 1.0)
fn = rc.rec_trmm if op == "trmm" else rc.rec_trsm


def ev_time(f, reps=1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for n in sizes:
    A = MatrixBuffer(n, n, dt, "cuda")
    rc.fill_uniform(A.view(), seed=1)
    rc.make_dominant(A.view())
    B = MatrixBuffer(n, n, dt, "cuda")
    rc.fill_uniform(B.view(), seed=2)
    be_s, be_a = Backend.cuda(), Backend.cuda(flags=ASYNC)
    run_s = lambda: fn(spec, A.cview(), B.view(), Threshold(256), be_s)  # noqa: E731
    run_a = lambda: fn(spec, A.cview(), B.view(), Threshold(256), be_a)  # noqa: E731
    for _ in range(3):
        run_s()
    rec = {"op": op, "elem": elem, "n": n}
    rec["sync_us"] = float(np.median([ev_time(run_s) for _ in range(7)]))
    rec["async_us"] = float(np.median([ev_time(run_a) for _ in range(7)]))
    rc.sync()
    rec["pipe_us"] = float(np.median([ev_time(run_a, 20) for _ in range(5)]))
    rc.sync()
    hs = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run_a()
        hs.append((time.perf_counter() - t0) * 1e6)
    rc.sync()
    rec["host_us"] = float(np.median(hs))
    try:
        cb = harness._cublas_call(rc.OpKind.Trmm if op == "trmm" else rc.OpKind.Trsm, spec, n, n, A.data, B.data)
        rec["cublas_us"] = float(np.median([cb() * 1e3 for _ in range(7)]))
    except Exception as e:  # noqa: BLE001
        rec["cublas_us"] = repr(e)
    print(json.dumps(rec), flush=True)
