"""GPU GEMM update kernels (DMMA fp64 / FFMA fp32) through rectri_cu_gemm_*,
against a float64 numpy reference -- test_gemm.cpp's cases plus odd shapes,
strided subviews and every transpose form."""
import itertools

import numpy as np
import pytest
import torch

import oracle
from paper_2504_13821_b200 import MatrixBuffer, Trans, gemm, scale
from tests._util import to_dev, to_np

pytestmark = pytest.mark.gpu
F = np.asfortranarray


def test_gemm_frozen(cuda):
    # test_gemm.cpp:26-53
    a = to_dev(F([[1.0, 2], [3, 4]]))
    c = MatrixBuffer(2, 2, torch.float64, "cuda")
    gemm(1.0, Trans.NoTrans, a.cview(), Trans.NoTrans, to_dev(F(np.eye(2))).cview(), 0.0, c.view())
    assert to_np(c).tolist() == [[1, 2], [3, 4]]
    gemm(1.0, Trans.NoTrans, a.cview(), Trans.NoTrans, to_dev(F([[5.0, 6], [7, 8]])).cview(), 0.0, c.view())
    assert to_np(c).tolist() == [[19, 22], [43, 50]]
    ones = to_dev(F([[1.0], [1.0]]))
    c2 = to_dev(F([[10.0], [10.0]]))
    gemm(1.0, Trans.Trans, a.cview(), Trans.NoTrans, ones.cview(), 1.0, c2.view())
    assert to_np(c2).ravel().tolist() == [14.0, 16.0]
    c3 = to_dev(F([[10.0], [10.0]]))
    gemm(1.0, Trans.ConjTrans, a.cview(), Trans.NoTrans, ones.cview(), 1.0, c3.view())
    assert oracle.bitwise_equal(to_np(c2), to_np(c3))


def test_beta_alpha_conventions(cuda):
    # test_gemm.cpp:190-208: beta == 0 never reads C; alpha == 0 skips A*B.
    nan = np.nan
    c = to_dev(F(np.full((2, 2), nan)))
    gemm(1.0, Trans.NoTrans, to_dev(F(np.eye(2))).cview(), Trans.NoTrans, to_dev(F([[2.0, 3], [4, 5]])).cview(),
         0.0, c.view())
    assert np.all(np.isfinite(to_np(c))) and to_np(c)[1, 0] == 4.0
    p = to_dev(F(np.full((2, 2), nan)))
    c2 = to_dev(F([[1.0, 2], [3, 4]]))
    gemm(0.0, Trans.NoTrans, p.cview(), Trans.NoTrans, p.cview(), 2.0, c2.view())
    assert to_np(c2).tolist() == [[2, 4], [6, 8]]
    c3 = to_dev(F(np.full((3, 3), nan)))
    gemm(0.0, Trans.NoTrans, p.cview(), Trans.NoTrans, p.cview(), 0.0, c3.view().subview(0, 0, 2, 2))
    assert np.all(to_np(c3)[:2, :2] == 0.0)


def test_scale(cuda):
    b = to_dev(F([[3.0, 4.0]]))
    scale(1.0, b.view())
    assert to_np(b).tolist() == [[3.0, 4.0]]
    scale(0.0, b.view())
    assert to_np(b).tolist() == [[0.0, 0.0]]
    m = MatrixBuffer(4, 4, torch.float64, "cuda", 1.0)
    scale(3.0, m.view().subview(1, 1, 2, 2))
    r = to_np(m)
    assert r[0, 0] == 1 and r[1, 1] == 3 and r[2, 2] == 3 and r[3, 3] == 1


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_gemm_shapes(cuda, dtype, ta, tb):
    rng = np.random.default_rng(7)
    eps = np.finfo(dtype).eps
    for M, N, K in ((1, 1, 1), (5, 3, 7), (64, 64, 64), (127, 129, 33), (128, 128, 128), (200, 65, 300),
                    (65, 300, 17), (256, 512, 1024)):
        a = F(rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(dtype))
        b = F(rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(dtype))
        c = F(rng.uniform(-1, 1, (M, N)).astype(dtype))
        opa = a.T if ta else a
        opb = b.T if tb else b
        ref = -1.25 * (opa.astype(np.float64) @ opb.astype(np.float64)) + 1.0 * c.astype(np.float64)
        C = to_dev(c)
        gemm(-1.25, Trans(ta), to_dev(a).cview(), Trans(tb), to_dev(b).cview(), 1.0, C.view())
        err = np.max(np.abs(to_np(C) - ref))
        assert err <= 4 * K * eps * 2.0, (M, N, K, err)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gemm_strided_subviews(cuda, dtype):
    """Odd leading dimensions and odd offsets take the unaligned cp.async path;
    the result must be bitwise the same as on a packed copy."""
    rng = np.random.default_rng(3)
    big_a = F(rng.uniform(-1, 1, (301, 177)).astype(dtype))
    big_b = F(rng.uniform(-1, 1, (263, 140)).astype(dtype))
    big_c = F(rng.uniform(-1, 1, (211, 150)).astype(dtype))
    A, B, C = to_dev(big_a), to_dev(big_b), to_dev(big_c)
    av = A.cview().subview(3, 5, 150, 101)
    bv = B.cview().subview(1, 7, 101, 129)
    cv = C.view().subview(11, 2, 150, 129)
    gemm(-1.0, Trans.NoTrans, av, Trans.NoTrans, bv, 1.0, cv)
    packed_c = to_dev(F(big_c[11:161, 2:131]))
    gemm(-1.0, Trans.NoTrans, to_dev(F(big_a[3:153, 5:106])).cview(), Trans.NoTrans,
         to_dev(F(big_b[1:102, 7:136])).cview(), 1.0, packed_c.view())
    got = to_np(C)
    assert oracle.bitwise_equal(got[11:161, 2:131], to_np(packed_c))
    untouched = big_c.copy()
    untouched[11:161, 2:131] = got[11:161, 2:131]
    assert oracle.bitwise_equal(got, untouched)


def test_gemm_result_independent_of_n(cuda):
    """Per-element k order does not depend on the tile chosen for N: column j
    of C is bitwise the same whether N = 1, 64 or 1000."""
    rng = np.random.default_rng(5)
    M, K = 300, 513
    a = F(rng.uniform(-1, 1, (M, K)))
    b = F(rng.uniform(-1, 1, (K, 1000)))
    full = to_dev(F(np.zeros((M, 1000))))
    gemm(1.0, Trans.NoTrans, to_dev(a).cview(), Trans.NoTrans, to_dev(b).cview(), 0.0, full.view())
    for w in (1, 64):
        part = to_dev(F(np.zeros((M, w))))
        gemm(1.0, Trans.NoTrans, to_dev(a).cview(), Trans.NoTrans, to_dev(F(b[:, :w])).cview(), 0.0, part.view())
        assert oracle.bitwise_equal(to_np(full)[:, :w], to_np(part))


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_tma_kernel_bitwise_equals_cp_async(cuda, ta, tb, monkeypatch):
    """The TMA-fed DMMA kernel (every instantiated configuration) and the
    cp.async kernel accumulate each element in the same k order: identical
    bits on ragged shapes (TMA zero-fill of the M/N/K tails) and sub-views."""
    rng = np.random.default_rng(11)
    for M, N, K in ((130, 70, 50), (77, 129, 33), (200, 24, 1100), (64, 64, 16), (8, 8, 1)):
        a = F(rng.uniform(-1, 1, (K + 4, M + 2) if ta else (M + 4, K + 2)))
        b = F(rng.uniform(-1, 1, (N + 2, K + 4) if tb else (K + 2, N + 4)))
        c0 = F(rng.uniform(-1, 1, (M + 2, N)))
        A, B = to_dev(a), to_dev(b)
        av = A.cview().subview(2, 2, K, M) if ta else A.cview().subview(2, 2, M, K)
        bv = B.cview().subview(2, 2, N, K) if tb else B.cview().subview(2, 2, K, N)
        outs = []
        for cfg in ("0", "1", "2", "3", "4"):
            monkeypatch.setenv("RECTRI_CU_GEMM64_TMA", cfg)
            C = to_dev(c0)
            gemm(-1.0, Trans(ta), av, Trans(tb), bv, 1.0, C.view().subview(2, 0, M, N))
            outs.append(to_np(C))
        for cfg, o in enumerate(outs[1:], 1):
            assert oracle.bitwise_equal(o, outs[0]), (M, N, K, cfg)


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_sgemm_v2_bitwise_equals_v1(cuda, ta, tb, monkeypatch):
    """fp32 FFMA GEMM v2 (one [k][o] shared layout, transposing 4-byte copies,
    FFMA2 for every case; 16- and 32-deep k-tiles) against v1: the same k-ascending fma chain per
    element, so identical bits -- ragged tails, sub-views at 4-byte offsets
    (the 4-byte copy paths), alpha / beta including beta = 0."""
    rng = np.random.default_rng(12)
    for (M, N, K), (alpha, beta) in itertools.product(
            ((130, 70, 50), (77, 129, 33), (200, 24, 1100), (128, 128, 16), (8, 8, 1), (257, 300, 129)),
            ((-1.0, 1.0), (0.5, 0.0), (2.0, -0.25))):
        for off in (0, 1):
            a = F(rng.uniform(-1, 1, (K + 4, M + 2) if ta else (M + 4, K + 2)).astype(np.float32))
            b = F(rng.uniform(-1, 1, (N + 2, K + 4) if tb else (K + 2, N + 4)).astype(np.float32))
            c0 = F(rng.uniform(-1, 1, (M + 2, N)).astype(np.float32))
            A, B = to_dev(a), to_dev(b)
            av = A.cview().subview(off, 2, K, M) if ta else A.cview().subview(off, 2, M, K)
            bv = B.cview().subview(off, 2, N, K) if tb else B.cview().subview(off, 2, K, N)
            outs = []
            variants = (("1", "16", "0"), ("2", "16", "0"), ("2", "32", "0"), ("2", "16", "1"), ("2", "32", "1"))
            for ver, bk, wide in variants:
                monkeypatch.setenv("RECTRI_CU_SGEMM", ver)
                monkeypatch.setenv("RECTRI_CU_SGEMM_BK", bk)
                monkeypatch.setenv("RECTRI_CU_SGEMM_WIDE", wide)  # 128x256 tiles, 8x16 per thread
                C = to_dev(c0)
                gemm(alpha, Trans(ta), av, Trans(tb), bv, beta, C.view().subview(2, 0, M, N))
                outs.append(to_np(C))
            for o, v in zip(outs[1:], variants[1:]):
                assert oracle.bitwise_equal(outs[0], o), (M, N, K, off, alpha, beta, v)


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_sgemm_v2_vector_epilogue_bitwise(cuda, ta, tb, monkeypatch):
    """Full-height tiles with a 16-byte aligned C take the float4 epilogue
    (reads of four columns before their writes): bitwise v1, ragged N, beta
    0 and != 0; a ragged M (the scalar epilogue) alongside."""
    rng = np.random.default_rng(13)
    for (M, N, K), beta in itertools.product(((256, 200, 300), (128, 129, 64), (250, 130, 40)), (1.0, 0.0, -0.5)):
        a = F(rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32))
        b = F(rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32))
        ld = (M + 3) // 4 * 4 + 4
        c0 = F(rng.uniform(-1, 1, (ld, N)).astype(np.float32))
        A, B = to_dev(a), to_dev(b)
        outs = []
        for ver in ("1", "2"):
            monkeypatch.setenv("RECTRI_CU_SGEMM", ver)
            C = to_dev(c0)
            gemm(0.75, Trans(ta), A.cview(), Trans(tb), B.cview(), beta, C.view().subview(0, 0, M, N))
            outs.append(to_np(C))
        assert oracle.bitwise_equal(outs[0], outs[1]), (M, N, K, beta)



@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_wave_tail_split_bitwise(cuda, ta, tb, monkeypatch):
    """The wave-tail split kernel (64x64 tiles for the leading columns, 32x32
    tiles for the last wave's) keeps every element's k-tile order: bit for
    bit the uniform 64x64 kernel (RECTRI_CU_GEMM64_TMA=2), ragged M / N / K,
    beta 0 and not; RECTRI_CU_GEMM64_SPLIT=2 forces the split at N / 2."""
    rng = np.random.default_rng(41 + 2 * ta + tb)
    for (M, N, K), beta in itertools.product(((2048, 2048, 1024), (130, 300, 50), (2000, 2100, 300), (77, 129, 1100)),
                                             (1.0, 0.0)):
        a = F(rng.uniform(-1, 1, (K, M) if ta else (M, K)))
        b = F(rng.uniform(-1, 1, (N, K) if tb else (K, N)))
        c0 = F(rng.uniform(-1, 1, (M, N)))
        A, B = to_dev(a), to_dev(b)
        outs = []
        for env in ({"RECTRI_CU_GEMM64_TMA": "2"}, {"RECTRI_CU_GEMM64_SPLIT": "2"}):
            monkeypatch.delenv("RECTRI_CU_GEMM64_TMA", raising=False)
            monkeypatch.delenv("RECTRI_CU_GEMM64_SPLIT", raising=False)
            for k, v in env.items():
                monkeypatch.setenv(k, v)
            C = to_dev(c0)
            gemm(-1.0, Trans(ta), A.cview(), Trans(tb), B.cview(), beta, C.view())
            outs.append(to_np(C))
        assert oracle.bitwise_equal(outs[0], outs[1]), (M, N, K, beta)
        opa = a.T if ta else a
        opb = b.T if tb else b
        ref = -(opa @ opb) + beta * c0
        assert np.max(np.abs(outs[1] - ref)) <= 2 * K * np.finfo(float).eps * np.max(np.abs(opa) @ np.abs(opb) + 1)


def test_sgemm_mbarrier_staging_replay_stress(cuda, monkeypatch):
    """The default fp32 GEMM (v2) refills its shared stages under per-stage
    mbarriers instead of a CTA barrier -- an ordering compute-sanitizer's
    racecheck cannot model.  A refill racing a stage's readers would show as
    run-to-run differences: 12 runs of a many-CTA GEMM are bitwise identical
    and bitwise the barrier-synchronised v1 kernel."""
    rng = np.random.default_rng(71)
    M, N, K = 1536, 2048, 1040
    a = F(rng.uniform(-1, 1, (M, K)).astype(np.float32))
    b = F(rng.uniform(-1, 1, (K, N)).astype(np.float32))
    c0 = F(rng.uniform(-1, 1, (M, N)).astype(np.float32))
    A, B = to_dev(a), to_dev(b)
    monkeypatch.setenv("RECTRI_CU_SGEMM", "1")
    C = to_dev(c0)
    gemm(-1.0, Trans.NoTrans, A.cview(), Trans.NoTrans, B.cview(), 1.0, C.view())
    want = C.data.clone()
    monkeypatch.setenv("RECTRI_CU_SGEMM", "2")
    C0 = to_dev(c0).data.clone()
    for wide in ("0", "1"):  # 128x128 and 128x256 tiles
        monkeypatch.setenv("RECTRI_CU_SGEMM_WIDE", wide)
        for rep in range(12):
            C.data.copy_(C0)
            gemm(-1.0, Trans.NoTrans, A.cview(), Trans.NoTrans, B.cview(), 1.0, C.view())
            assert torch.equal(C.data, want), (wide, rep)

