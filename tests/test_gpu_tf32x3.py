"""fp32 3xTF32 variant on tcgen05 (RECTRI_CU_TF32X3 / TF32X3 backend flag,
csrc/sgemm_tf32x3.cu): an opt-in path reported separately from the default
exact-FFMA fp32 path, held to its own tolerance.  The GEMM update must stay
within 8*K*eps_fp32 of an fp64 reference on every transpose form (the split
x = hi + lo keeps ~fp32 accuracy; FFMA is ~1 K*eps), and the recursive
drivers must meet the reference's 32*n*eps criterion on every variant."""
import itertools

import numpy as np
import pytest
import torch

import oracle
from paper_2504_13821_b200 import NO_GRAPH, TF32X3, Backend, MatrixBuffer, Trans, gemm
from tests._util import check_against_oracle, run_op, to_dev, to_np

pytestmark = pytest.mark.gpu
F = np.asfortranarray
EPS32 = np.finfo(np.float32).eps


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_tf32x3_gemm_accuracy(cuda, ta, tb):
    rng = np.random.default_rng(21)
    for M, N, K, beta in ((128, 256, 32, 1.0), (300, 260, 100, 1.0), (1024, 1000, 512, 0.0), (96, 40, 36, 1.0),
                          (256, 512, 1024, 1.0)):
        a = F(rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32))
        b = F(rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32))
        c = F(rng.uniform(-1, 1, (M, N)).astype(np.float32))
        ref = -1.0 * ((a.T if ta else a).astype(np.float64) @ (b.T if tb else b).astype(np.float64))
        ref += beta * c.astype(np.float64)
        C = to_dev(c)
        gemm(-1.0, Trans(ta), to_dev(a).cview(), Trans(tb), to_dev(b).cview(), beta, C.view(),
             Backend.cuda(flags=TF32X3 | NO_GRAPH))
        err = np.max(np.abs(to_np(C) - ref))
        assert err <= 8 * K * EPS32, (M, N, K, ta, tb, err / (K * EPS32))


@pytest.mark.parametrize("op", ["trsm", "trmm"])
def test_tf32x3_recursion_all_variants(cuda, op):
    n, m, t = 512, 96, 64  # 3 GEMM levels (K = 256, 128, 64)
    for side, uplo, trans, diag in itertools.product((0, 1), (0, 1), (0, 1), (0, 1)):
        s = oracle.spec(side, uplo, trans, diag, 1.0)
        a = oracle.make_operand(s, op == "trsm", n, 5).astype(np.float32)
        b = oracle.make_rhs(s, n, m, 6).astype(np.float32)
        for be in (Backend.cuda(flags=TF32X3), Backend.cuda(flags=TF32X3 | NO_GRAPH)):
            got = run_op(op, s, F(a), F(b), t, backend=be)
            check_against_oracle(op, s, F(a), F(b), got)


def test_tf32x3_differs_from_ffma_and_is_opt_in(cuda):
    """The default fp32 path stays exact FFMA (the flag changes bits)."""
    s = oracle.spec(0, 0, 0, 0, 1.0)
    n, m = 1024, 256
    a = oracle.make_operand(s, True, n, 7).astype(np.float32)
    b = oracle.make_rhs(s, n, m, 8).astype(np.float32)
    dflt = run_op("trsm", s, F(a), F(b), 256)
    ffma = run_op("trsm", s, F(a), F(b), 256, backend=Backend.cuda(flags=NO_GRAPH))
    tf = run_op("trsm", s, F(a), F(b), 256, backend=Backend.cuda(flags=TF32X3))
    assert oracle.bitwise_equal(dflt, ffma)
    assert not oracle.bitwise_equal(dflt, tf)
    check_against_oracle("trsm", s, F(a), F(b), tf)
