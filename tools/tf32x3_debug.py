"""Bring-up probe for the 3xTF32 kernel: one GEMM per shape given on the
command line (M,N,K,ta,tb), TF32X3 backend flag, printed before/after."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
from paper_2504_13821_b200 import NO_GRAPH, TF32X3, Backend, Trans, gemm  # noqa: E402
from tests._util import to_dev  # noqa: E402

F = np.asfortranarray
rng = np.random.default_rng(21)
for spec in sys.argv[1:]:
    M, N, K, ta, tb = (int(x) for x in spec.split(","))
    a = F(rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32))
    b = F(rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32))
    C = to_dev(F(rng.uniform(-1, 1, (M, N)).astype(np.float32)))
    print("start", spec, flush=True)
    t = time.time()
    gemm(-1.0, Trans(ta), to_dev(a).cview(), Trans(tb), to_dev(b).cview(), 1.0, C.view(),
         Backend.cuda(flags=TF32X3 | NO_GRAPH))
    torch.cuda.synchronize()
    print("done", time.time() - t, flush=True)
