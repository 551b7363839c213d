"""Stress: the captured-recursion sequence of tests/test_gpu_leaf.py
(v1 direct, v2 graph, v3 graph) repeated, residual of every result."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import oracle  # noqa: E402
from paper_2504_13821_b200 import NO_GRAPH, Backend, Threshold, rec_trmm, rec_trsm  # noqa: E402
from tests._util import to_dev, to_np, tspec  # noqa: E402

F = np.asfortranarray
rng = np.random.default_rng(7)
n, m = 1024, 4100
op = sys.argv[2] if len(sys.argv) > 2 else "trsm"
s = oracle.spec(0, 0, 0, 0, 1.0)
fails = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    seed = int(rng.integers(1 << 30))
    a = F(oracle.make_operand(s, op == "trsm", n, seed))
    b = F(oracle.make_rhs(s, n, m, seed + 1))
    for version, be in ((1, Backend.cuda(flags=NO_GRAPH)), (2, Backend.cuda()), (3, Backend.cuda())):
        os.environ["RECTRI_CU_LEAF"] = str(version)
        A, B = to_dev(a), to_dev(b)
        (rec_trsm if op == "trsm" else rec_trmm)(tspec(s), A.cview(), B.view(), Threshold(256), be)
        x = to_np(B)
        res = (oracle.trsm_residual_inf(s, a, x, b) if op == "trsm"
               else oracle.max_abs_diff(x, oracle.oracle_trmm(s, a, b)) / max(1.0, oracle.max_abs(x)) * 1e-4)
        print(f"it {it} v{version}: residual {res:.3e}", flush=True)
        if res > 1e-8:
            fails += 1
            ref = np.linalg.solve(np.tril(a), b) if op == "trsm" else oracle.oracle_trmm(s, a, b)
            err = np.abs(x - ref) > 1e-8 * np.maximum(1, np.abs(ref))
            rows = np.where(err.any(axis=1))[0]
            cols = np.where(err.any(axis=0))[0]
            print("  bad rows", rows.min(), rows.max(), len(rows), "bad cols", cols.min(), cols.max(), len(cols),
                  "first bad row blocks (256)", sorted(set((rows // 256).tolist())),
                  "col blocks (32)", sorted(set((cols // 32).tolist()))[:20], flush=True)
            print(f"it {it} v{version}: residual {res:.3e} ptrA {A.data.data_ptr():x} ptrB {B.data.data_ptr():x}",
                  flush=True)
print("fails", fails)
