"""Repro helper: rec_trsm/rec_trmm fp64 with the v3 leaf under the graph /
direct paths and 1-2 streams, residual against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import oracle  # noqa: E402
from paper_2504_13821_b200 import NO_GRAPH, Backend  # noqa: E402
from tests._util import run_op, check_against_oracle  # noqa: E402

F = np.asfortranarray
n, m = int(sys.argv[1]), int(sys.argv[2])
s = oracle.spec(0, 0, 0, 0, 1.0)
a = F(oracle.make_operand(s, True, n, 11))
b = F(oracle.make_rhs(s, n, m, 12))
for name, be in (("graph", Backend.cuda()), ("direct", Backend.cuda(flags=NO_GRAPH))):
    got = run_op("trsm", s, a, b, 256, backend=be)
    try:
        e = check_against_oracle("trsm", s, a, b, got)
        print(name, "ok", e, flush=True)
    except AssertionError as ex:
        bad = np.where(np.abs(got - np.linalg.solve(np.tril(a), b)) > 1e-6)
        print(name, "FAIL", str(ex)[:80], "bad rows", sorted(set(bad[0]))[:10], "... cols", sorted(set(bad[1]))[:5],
              len(set(bad[1])), flush=True)
