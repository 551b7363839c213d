"""Ring checking of the default leaves (leaf3_kernel, csrc/leaf64_v3.cu;
leaf32_kernel, csrc/leaf32_v3.cu):
the producer warp refills mbarrier-guarded shared-memory slots with
cp.async.bulk while the compute warps read them, an ordering that
compute-sanitizer racecheck does not model (and the tool may be closed on
the GPU pool).  With RECTRI_CU_RING_CHECK=1 every A fragment a compute warp
reads from a slot is compared, bit for bit, with its packed block in global
memory: a refill that overtook the slot's readers would show up as a
mismatch.  =2 plants a slot mix-up, which the checker must report -- the
role of the reference's workgroup race detector and its planted race
(src/workgroup.cpp:138-177, 333-349; tests/test_workgroup.cpp:144-176)."""
import numpy as np
import pytest

import oracle
from paper_2504_13821_b200 import NO_GRAPH, Backend, Threshold, rec_trmm, rec_trsm
from tests._util import check_against_oracle, to_dev, to_np, tspec

pytestmark = pytest.mark.gpu


def _inputs(op, s, n, m, rng):
    seed = int(rng.integers(1 << 30))
    return (np.asfortranarray(oracle.make_operand(s, op == "trsm", n, seed)),
            np.asfortranarray(oracle.make_rhs(s, n, m, seed + 1)))


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("op", ["trsm", "trmm"])
@pytest.mark.parametrize("width", ["8", "16", "32"])
@pytest.mark.parametrize("side", [0, 1])
def test_leaf_ring_check(cuda, monkeypatch, op, width, side, dtype):
    import paper_2504_13821_b200 as rc
    import torch

    monkeypatch.setenv("RECTRI_CU_LEAF", "3")
    monkeypatch.setenv("RECTRI_CU_LEAF_NC", width)
    monkeypatch.setenv("RECTRI_CU_RING_CHECK", "1")
    rc.clear_graph_cache()  # the checker instantiation is chosen at capture
    rng = np.random.default_rng(700 + int(width) + 2 * side)
    n, m = 1024, 2304
    s = oracle.spec(side, 0, 0, 0, 1.0)
    a, b = _inputs(op, s, n, m, rng)
    a, b = np.asfortranarray(a.astype(dtype)), np.asfortranarray(b.astype(dtype))
    A, B = to_dev(a), to_dev(b)
    B0 = B.data.clone()
    fn = rec_trmm if op == "trmm" else rec_trsm
    rc.debug_ring_check(reset=True)
    first = None
    for rep in range(12):  # graph replays, then direct launches
        B.data.copy_(B0)
        be = Backend.cuda() if rep < 8 else Backend.cuda(flags=NO_GRAPH)
        fn(tspec(s), A.cview(), B.view(), Threshold(256), be)
        torch.cuda.synchronize()
        if first is None:
            first = B.data.clone()
        else:
            assert torch.equal(B.data, first), (op, width, rep)
    assert rc.debug_ring_check(reset=True) == 0
    check_against_oracle(op, s, a, b, to_np(B))

    # planted slot mix-up: the checker must see it
    monkeypatch.setenv("RECTRI_CU_RING_CHECK", "2")
    rc.clear_graph_cache()
    B.data.copy_(B0)
    fn(tspec(s), A.cview(), B.view(), Threshold(256), Backend.cuda(flags=NO_GRAPH))
    assert rc.debug_ring_check(reset=True) > 0
    rc.clear_graph_cache()


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_dgemm_ring_check(cuda, monkeypatch, ta, tb):
    """The TMA DGEMM (dgemm_tma_kernel / dgemm_tma_split_kernel, the
    recursion's off-diagonal updates): every A / B fragment a consumer warp
    reads from a TMA-filled stage equals its element of op(A) / op(B) (zero
    outside the matrix), on ragged shapes and the 64x64, 32x32 and wave-tail
    split configurations; the result is bitwise the unchecked kernel's, and a
    planted stage mix-up is reported."""
    import paper_2504_13821_b200 as rc
    import torch
    from paper_2504_13821_b200 import Trans

    rng = np.random.default_rng(40 + 2 * ta + tb)
    rc.debug_ring_check(reset=True)

    def run(a, b, c):
        A, B, C = to_dev(np.asfortranarray(a)), to_dev(np.asfortranarray(b)), to_dev(np.asfortranarray(c))
        rc.gemm(-1.0, Trans(ta), A.cview(), Trans(tb), B.cview(), 1.0, C.view(), Backend.cuda(flags=NO_GRAPH))
        torch.cuda.synchronize()
        return to_np(C)

    for M, N, K, split in ((130, 70, 50, "1"), (1000, 3000, 700, "1"), (512, 8192, 256, "1"), (4096, 4096, 1024, "2"),
                           (64, 64, 2048, "1")):
        monkeypatch.setenv("RECTRI_CU_GEMM64_SPLIT", split)
        a = rng.uniform(-1, 1, (K, M) if ta else (M, K))
        b = rng.uniform(-1, 1, (N, K) if tb else (K, N))
        c = rng.uniform(-1, 1, (M, N))
        monkeypatch.setenv("RECTRI_CU_RING_CHECK", "0")
        plain = run(a, b, c)
        monkeypatch.setenv("RECTRI_CU_RING_CHECK", "1")
        checked = run(a, b, c)
        assert rc.debug_ring_check(reset=True) == 0, (M, N, K, split)
        assert oracle.bitwise_equal(plain, checked), (M, N, K)
        ref = c - (a.T if ta else a) @ (b.T if tb else b)
        assert np.max(np.abs(checked - ref)) <= 64 * K * np.finfo(float).eps * (1 + np.max(np.abs(ref)))
        if (M, N, K) == (1000, 3000, 700):  # planted stage mix-up
            monkeypatch.setenv("RECTRI_CU_RING_CHECK", "2")
            run(a, b, c)
            assert rc.debug_ring_check(reset=True) > 0


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_sgemm_ring_check(cuda, monkeypatch, ta, tb):
    """The fp32 FFMA2 GEMM (sgemm_ffma2_kernel: cp.async stages with
    per-stage mbarriers and a deferred refill): each k-step's A / B fragments
    equal their op(A) / op(B) elements (zero outside the matrix) on the
    128x128 and 128x256 tiles and both k-tile depths; bitwise the unchecked
    kernel's result; a planted stage mix-up is reported."""
    import paper_2504_13821_b200 as rc
    import torch
    from paper_2504_13821_b200 import Trans

    rng = np.random.default_rng(60 + 2 * ta + tb)
    rc.debug_ring_check(reset=True)

    def run(a, b, c):
        A, B, C = to_dev(np.asfortranarray(a)), to_dev(np.asfortranarray(b)), to_dev(np.asfortranarray(c))
        rc.gemm(-1.0, Trans(ta), A.cview(), Trans(tb), B.cview(), 1.0, C.view(), Backend.cuda(flags=NO_GRAPH))
        torch.cuda.synchronize()
        return to_np(C)

    for M, N, K, bk in ((128, 72, 52, "16"), (1000, 3000, 700, "32"), (512, 8192, 256, "16"), (4096, 4096, 1024, "32"),
                        (4096, 4096, 1000, "16")):
        monkeypatch.setenv("RECTRI_CU_SGEMM_BK", bk)
        a = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
        b = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
        c = rng.uniform(-1, 1, (M, N)).astype(np.float32)
        monkeypatch.setenv("RECTRI_CU_RING_CHECK", "0")
        plain = run(a, b, c)
        monkeypatch.setenv("RECTRI_CU_RING_CHECK", "1")
        checked = run(a, b, c)
        assert rc.debug_ring_check(reset=True) == 0, (M, N, K, bk)
        assert oracle.bitwise_equal(plain, checked), (M, N, K)
        ref = c.astype(float) - (a.T if ta else a).astype(float) @ (b.T if tb else b).astype(float)
        assert np.max(np.abs(checked - ref)) <= 8 * K * np.finfo(np.float32).eps * (1 + np.max(np.abs(ref)))
        if (M, N, K) == (1000, 3000, 700):  # planted stage mix-up
            monkeypatch.setenv("RECTRI_CU_RING_CHECK", "2")
            run(a, b, c)
            assert rc.debug_ring_check(reset=True) > 0

