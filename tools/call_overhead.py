"""Host cost of one rec_trsm call (n = m = 256, ASYNC, graph cached): the
Python argument marshalling alone vs the whole call.  Not a bench number.

    python tools/call_overhead.py
"""
import ctypes
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2504_13821_b200 as rc  # noqa: E402
from paper_2504_13821_b200 import ASYNC, Backend, MatrixBuffer, Threshold, TriangularSpec, _lib  # noqa: E402
from paper_2504_13821_b200 import api  # noqa: E402

n = 256
A = MatrixBuffer(n, n, torch.float64, "cuda")
rc.fill_uniform(A.view(), seed=1)
rc.make_dominant(A.view())
B = MatrixBuffer(n, n, torch.float64, "cuda")
spec, be = TriangularSpec(), Backend.cuda(flags=ASYNC)
Av, Bv = A.cview(), B.view()


def bench(f, reps=2000):
    for _ in range(50):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    t = (time.perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    return t


def marshal():
    api._spec_c(spec), Av._c(), Bv._c(), be._c(api._device_of(Av, Bv)), api._sink_c(None)


lib = _lib.load()
args = (ctypes.byref(api._spec_c(spec)), Av._c(), Bv._c(), 256, ctypes.byref(be._c(api._device_of(Av, Bv))),
        api._sink_c(None)[0], None, ctypes.byref(ctypes.c_int64(-1)))
raw = lambda: lib.rectri_cu_rec_trsm_f64(*args)  # noqa: E731
full = lambda: rc.rec_trsm(spec, Av, Bv, Threshold(256), be)  # noqa: E731
print({"marshal_us": bench(marshal), "raw_c_call_us": bench(raw), "full_call_us": bench(full),
       "cur_stream_us": bench(lambda: torch.cuda.current_stream())})
rc.sync()
