"""fp64 leaf kernels: v2 (leaf64.cu: packed triangle, solver warps) against
v1 (leaf.cu) -- identical per-element arithmetic, so bit for bit on every
variant, tile order, right-hand-side count and alpha; v3 (leaf64_v3.cu, the
default: diagonal blocks as DMMA products with explicit inverses) against
the oracle tolerance and v1 to rounding; plus the masking rules for each."""
import itertools

import numpy as np
import pytest

import oracle
from paper_2504_13821_b200 import NO_GRAPH, Backend, Threshold, rec_trmm, rec_trsm, trmm_base, trsm_base
from tests._util import check_against_oracle, to_dev, to_np, tspec

pytestmark = pytest.mark.gpu
F = np.asfortranarray
VARIANTS = list(itertools.product((0, 1), (0, 1), (0, 1), (0, 1)))  # side, uplo, trans, diag


def _inputs(op, s, n, m, rng):
    seed = int(rng.integers(1 << 30))
    return F(oracle.make_operand(s, op == "trsm", n, seed)), F(oracle.make_rhs(s, n, m, seed + 1))


def _base(op, s, a, b, version, monkeypatch, backend=None):
    monkeypatch.setenv("RECTRI_CU_LEAF", str(version))
    A, B = to_dev(a), to_dev(b)
    fn = trmm_base if op == "trmm" else trsm_base
    fn(tspec(s), A.cview(), B.view(), 256, backend or Backend.cuda(flags=NO_GRAPH))
    return to_np(B)


@pytest.mark.parametrize("op", ["trsm", "trmm"])
@pytest.mark.parametrize("side,uplo,trans,diag", VARIANTS)
def test_leaf_v2_bitwise_equals_v1(cuda, monkeypatch, op, side, uplo, trans, diag):
    rng = np.random.default_rng(100 + 8 * side + 4 * uplo + 2 * trans + diag)
    for n, m, alpha in ((1, 3, 1.0), (5, 33, 1.0), (32, 32, 2.5), (33, 70, 1.0), (100, 65, -0.75),
                        (256, 96, 1.0), (255, 31, 1.0)):
        s = oracle.spec(side, uplo, trans, diag, alpha)
        a, b = _inputs(op, s, n, m, rng)
        v1 = _base(op, s, a, b, 1, monkeypatch)
        v2 = _base(op, s, a, b, 2, monkeypatch)
        assert oracle.bitwise_equal(v1, v2), (op, side, uplo, trans, diag, n, m, alpha)
        if n <= 100:
            check_against_oracle(op, s, a, b, v2)
        v3 = _base(op, s, a, b, 3, monkeypatch)
        check_against_oracle(op, s, a, b, v3)
        scale = max(1.0, float(np.max(np.abs(v1))))
        assert float(np.max(np.abs(v3 - v1))) <= 64 * n * np.finfo(np.float64).eps * scale


@pytest.mark.parametrize("op", ["trsm", "trmm"])
def test_leaf_v2_in_captured_recursion(cuda, monkeypatch, op):
    """The recursion's CUDA graph (leaves on the capture and panel streams)
    with the v2 leaf equals direct launches with the v1 leaf, bitwise."""
    rng = np.random.default_rng(7)
    n, m = 1024, 4100
    s = oracle.spec(0, 0, 0, 0, 1.0)
    a, b = _inputs(op, s, n, m, rng)
    fn = rec_trmm if op == "trmm" else rec_trsm
    outs = []
    for version, be in ((1, Backend.cuda(flags=NO_GRAPH)), (2, Backend.cuda()), (3, Backend.cuda())):
        monkeypatch.setenv("RECTRI_CU_LEAF", str(version))
        A, B = to_dev(a), to_dev(b)
        fn(tspec(s), A.cview(), B.view(), Threshold(256), be)
        outs.append(to_np(B))
    assert oracle.bitwise_equal(outs[0], outs[1])
    check_against_oracle(op, s, a, b, outs[2]) if n <= 1024 else None


@pytest.mark.parametrize("version", [2, 3])
def test_leaf_masking_and_alpha_zero(cuda, monkeypatch, version):
    rng = np.random.default_rng(3)
    n, m = 100, 40
    for op in ("trsm", "trmm"):
        for uplo in (0, 1):
            s = oracle.spec(0, uplo, 0, 1, 1.0)  # Unit: the stored diagonal is never read
            a, b = _inputs(op, s, n, m, rng)
            junk = a.copy()
            iu = np.triu_indices(n, 1) if uplo == 0 else np.tril_indices(n, -1)
            junk[iu] = np.nan
            np.fill_diagonal(junk, np.nan)
            ref = _base(op, s, a, b, version, monkeypatch)
            got = _base(op, s, junk, b, version, monkeypatch)
            assert np.all(np.isfinite(got)) and oracle.bitwise_equal(ref, got)
    s = oracle.spec(0, 0, 0, 0, 0.0)
    b = F(np.full((n, m), np.nan))
    got = _base("trmm", s, F(rng.uniform(-1, 1, (n, n))), b, version, monkeypatch)
    assert np.all(got == 0.0)


@pytest.mark.parametrize("op", ["trsm", "trmm"])
@pytest.mark.parametrize("side,uplo,trans,diag", VARIANTS)
def test_leaf32_v3_matches_v1_and_oracle(cuda, monkeypatch, op, side, uplo, trans, diag):
    """fp32 leaf v3 (leaf32_v3.cu: packed blocks, FFMA2, inverse diagonal
    blocks in fp64 rounded once) against the oracle and v1 (leaf.cu)."""
    rng = np.random.default_rng(300 + 8 * side + 4 * uplo + 2 * trans + diag)
    eps = np.finfo(np.float32).eps
    for n, m, alpha in ((1, 3, 1.0), (33, 70, 1.0), (100, 65, -0.75), (256, 96, 1.0)):
        s = oracle.spec(side, uplo, trans, diag, alpha)
        a, b = _inputs(op, s, n, m, rng)
        a, b = F(a.astype(np.float32)), F(b.astype(np.float32))
        v1 = _base(op, s, a, b, 1, monkeypatch)
        v3 = _base(op, s, a, b, 3, monkeypatch)
        check_against_oracle(op, s, a, b, v3)
        scale = max(1.0, float(np.max(np.abs(v1))))
        assert float(np.max(np.abs(v3 - v1))) <= 64 * n * eps * scale, (n, m)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("op", ["trsm", "trmm"])
@pytest.mark.parametrize("side,uplo,trans,diag", VARIANTS)
def test_leaf_v3_panel_widths_bitwise(cuda, monkeypatch, dt, op, side, uplo, trans, diag):
    """leaf3 / leaf32 with 8-, 16- and 32-wide right-hand-side panels (the
    width follows the leaf's right-hand-side count): the same products in the
    same order per element, so identical bits, ragged panels included."""
    rng = np.random.default_rng(500 + 8 * side + 4 * uplo + 2 * trans + diag)
    for n, m, alpha in ((33, 70, 1.0), (100, 13, -0.75), (256, 96, 1.0), (200, 41, 2.0)):
        s = oracle.spec(side, uplo, trans, diag, alpha)
        a, b = _inputs(op, s, n, m, rng)
        a, b = F(a.astype(dt)), F(b.astype(dt))
        outs = []
        for nc, wm in (("32", "1"), ("16", "1"), ("8", "1"), ("32", "2")):
            monkeypatch.setenv("RECTRI_CU_LEAF_NC", nc)
            monkeypatch.setenv("RECTRI_CU_LEAF_WM", wm)
            outs.append(_base(op, s, a, b, 3, monkeypatch))
        check_against_oracle(op, s, a, b, outs[0])
        for k, o in enumerate(outs[1:], 1):
            assert oracle.bitwise_equal(outs[0], o), (n, m, k)


@pytest.mark.parametrize("dtype", [np.float64, np.float32], ids=["f64", "f32"])
@pytest.mark.parametrize("op", ["trsm", "trmm"])
@pytest.mark.parametrize("width", [8, 16, 32])
def test_default_leaf_replay_stress(cuda, monkeypatch, op, dtype, width):
    """Ring-ordering stress of the DEFAULT leaves (leaf3_kernel / leaf32_kernel:
    a producer warp refills mbarrier-guarded bulk-copy slots while 4-8 compute
    warps read them -- the ordering compute-sanitizer racecheck cannot model).
    A refill racing a slot's readers shows up as run-to-run differences (it
    caught a real one: tools/leaf3_stress.py): 24 graph replays of the same
    recursion must be bitwise identical, and within the oracle tolerance
    (the reference's own role for the workgroup simulator's race detector,
    src/workgroup.cpp:138-177, tests/test_workgroup.cpp:144-176)."""
    import paper_2504_13821_b200 as rc
    import torch

    monkeypatch.setenv("RECTRI_CU_LEAF", "3")
    monkeypatch.setenv("RECTRI_CU_LEAF_NC", str(width))
    rc.clear_graph_cache()  # the panel width is fixed at capture
    rng = np.random.default_rng(300 + width)
    n, m = 1024, 2304
    s = oracle.spec(0, 0, 0, 0, 1.0)
    a, b = _inputs(op, s, n, m, rng)
    a, b = F(a.astype(dtype)), F(b.astype(dtype))
    A, B = to_dev(a), to_dev(b)
    B0 = B.data.clone()
    fn = rec_trmm if op == "trmm" else rec_trsm
    first = None
    for rep in range(24):
        B.data.copy_(B0)
        fn(tspec(s), A.cview(), B.view(), Threshold(256), Backend.cuda())
        torch.cuda.synchronize()
        if first is None:
            first = B.data.clone()
            check_against_oracle(op, s, a, b, to_np(B))
        else:
            assert torch.equal(B.data, first), (op, width, rep)
    rc.clear_graph_cache()


@pytest.mark.parametrize("side,uplo,trans,diag", VARIANTS)
def test_leaf_v5_trmm_bitwise_equals_v3(cuda, monkeypatch, side, uplo, trans, diag):
    """v5 (leaf64_v5.cu: row-block-owning warps, the TRMM leaf of direct
    trmm_base calls) performs v3's per-element arithmetic: identical bits on
    every variant, ragged orders / right-hand-side counts, alpha and every
    panel width -- so choosing between them by right-hand-side count never
    changes a result (the RHS-sharding invariant)."""
    rng = np.random.default_rng(500 + 8 * side + 4 * uplo + 2 * trans + diag)
    for n, m, alpha in ((1, 3, 1.0), (33, 70, 1.0), (100, 65, -0.75), (256, 200, 1.0), (255, 97, 2.5),
                        (256, 5000, 1.0)):
        s = oracle.spec(side, uplo, trans, diag, alpha)
        a, b = _inputs("trmm", s, n, m, rng)
        monkeypatch.setenv("RECTRI_CU_LEAF5_MAX", "0")  # v3
        v3 = _base("trmm", s, a, b, 3, monkeypatch)
        monkeypatch.setenv("RECTRI_CU_LEAF5_MAX", str(1 << 30))
        for nc in ("8", "16", "32"):
            monkeypatch.setenv("RECTRI_CU_LEAF5_NC", nc)
            v5 = _base("trmm", s, a, b, 3, monkeypatch)
            assert oracle.bitwise_equal(v3, v5), (side, uplo, trans, diag, n, m, alpha, nc)
        monkeypatch.delenv("RECTRI_CU_LEAF5_NC")
        monkeypatch.delenv("RECTRI_CU_LEAF5_MAX")
        check_against_oracle("trmm", s, a, b, v5)


@pytest.mark.parametrize("side", [0, 1])
def test_leaf_v5_in_recursion_bitwise(cuda, monkeypatch, side):
    """RECTRI_CU_LEAF=4 packs the recursion's TRMM triangles in v5's
    ascending order and runs v5 leaves: identical bits to the default (v3),
    device- and host-resident."""
    import paper_2504_13821_b200 as rc
    import torch

    rng = np.random.default_rng(77 + side)
    n, m = 1024, 5000
    s = oracle.spec(side, 1, 0, 0, 1.0)
    a, b = _inputs("trmm", s, n, m, rng)
    outs = []
    for version in ("3", "4"):
        monkeypatch.setenv("RECTRI_CU_LEAF", version)
        rc.clear_graph_cache()
        A, B = to_dev(a), to_dev(b)
        rec_trmm(tspec(s), A.cview(), B.view(), Threshold(256), Backend.cuda())
        outs.append(to_np(B))
        Ah = rc.MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a)), device="cpu")
        Bh = rc.MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(b)), device="cpu")
        rec_trmm(tspec(s), Ah.cview(), Bh.view(), Threshold(256), Backend.cuda())
        outs.append(np.asfortranarray(Bh.numpy()))
    for o in outs[1:]:
        assert oracle.bitwise_equal(outs[0], o)
    check_against_oracle("trmm", s, a, b, outs[0])
    rc.clear_graph_cache()

