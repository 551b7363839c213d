"""GPU parity: the sm_100a path (librectri_cu.so through the C-ABI) against the
oracle and the reference's golden vectors, at the reference's tolerances,
plus the behavioural contract of SURVEY.md 8(b').  Mirrors
test_recursion.cpp / test_base_kernels.cpp / acceptance_main.cpp."""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2504_13821_b200 import (
    NO_GRAPH,
    AliasError,
    Backend,
    ConfigError,
    Diag,
    MatrixBuffer,
    MatrixView,
    OpKind,
    RecEvent,
    ShapeError,
    Side,
    SingularityError,
    Threshold,
    TileLimitError,
    Trans,
    TriangularSpec,
    Uplo,
    rec_trmm,
    rec_trsm,
    schema_for,
    trmm_base,
    trsm_base,
)
from tests._util import check_against_oracle, run_base, run_op, to_dev, to_np, tspec

pytestmark = pytest.mark.gpu

F = np.asfortranarray


def _golden_cases(golden, prefix):
    for i in range(int(golden[f"{prefix}/count"])):
        k = f"{prefix}/{i:04d}"
        meta = golden[k + "/meta"]
        s = oracle.spec(int(meta[1]), int(meta[2]), int(meta[3]), int(meta[4]), float(golden[k + "/alpha"]))
        yield ("trmm" if meta[0] == 0 else "trsm"), s, int(meta[7]), F(golden[k + "/a"]), F(golden[k + "/b"]), \
            golden[k + "/events"]


# ----------------------------------------------------------------- frozen KATs
def test_trsm_base_frozen(cuda):
    # test_base_kernels.cpp:13-43 / SPEC.md:191-194
    s = oracle.spec(alpha=2.0)
    assert run_base("trsm", s, F(np.eye(2)), F([[1.0], [3.0]])).ravel().tolist() == [2.0, 6.0]
    s = oracle.spec()
    assert run_base("trsm", s, F([[2.0, 0], [1, 4]]), F([[2.0], [6.0]])).ravel().tolist() == [1.0, 1.25]
    A = to_dev(F([[0.0, 0], [1, 4]]))
    B = to_dev(F([[2.0], [6.0]]))
    with pytest.raises(SingularityError) as e:
        trsm_base(tspec(s), A.cview(), B.view())
    assert e.value.index() == 0
    assert to_np(B).ravel().tolist() == [2.0, 6.0]  # found before B is touched


def test_trmm_base_frozen(cuda):
    # test_base_kernels.cpp:45-68 / SPEC.md:199-202
    A = F([[2.0, 0], [3, 4]])
    ones = F([[1.0], [1.0]])
    assert run_base("trmm", oracle.spec(trans=1), A, ones).ravel().tolist() == [5.0, 4.0]
    assert run_base("trmm", oracle.spec(), A, ones).ravel().tolist() == [2.0, 7.0]
    G = F([[999.0, 0], [3, 999]])
    assert run_base("trmm", oracle.spec(diag=1), G, ones).ravel().tolist() == [1.0, 4.0]


def test_rec_frozen(cuda):
    # test_recursion.cpp:93-131 / SPEC.md:271-282
    b = oracle.make_random(4, 3, 11)
    out = run_op("trmm", oracle.spec(trans=1), F(np.eye(4)), b, 2)
    assert oracle.bitwise_equal(out, b)
    out = run_op("trmm", oracle.spec(trans=1), F([[2.0, 0], [3, 4]]), F([[1.0], [1.0]]), 1)
    assert out.ravel().tolist() == [5.0, 4.0]
    out = run_op("trmm", oracle.spec(side=1, uplo=1), F([[1.0, 1], [0, 1]]), F([[1.0, 1.0]]), 1)
    assert out.ravel().tolist() == [1.0, 2.0]
    b = oracle.make_random(8, 3, 21)
    assert oracle.bitwise_equal(run_op("trsm", oracle.spec(), F(np.eye(8)), b, 2), b)
    assert run_op("trsm", oracle.spec(), F([[2.0, 0], [1, 4]]), F([[2.0], [6.0]]), 1).ravel().tolist() == [1.0, 1.25]


def test_schema_table_matches_reference(golden):
    for row in golden["schema"]:
        op, side, uplo, trans = (int(x) for x in row[:4])
        sc = schema_for(OpKind(op), TriangularSpec(Side(side), Uplo(uplo), Trans(trans)))
        got = [sc.first_block == 1, int(sc.update.off_trans), sc.update.off_on_left, int(sc.update.read_half),
               int(sc.update.write_half), sc.update.sign, sc.update.carries_alpha, sc.second_block == 1]
        assert [float(x) for x in got] == [float(x) for x in row[4:]], row


# ------------------------------------------------------- golden vector parity
@pytest.mark.parametrize("prefix", ["case", "mid"])
def test_golden_cases_parity_and_events(cuda, golden, prefix):
    """Every golden case: GPU result within the criterion-1 bound of the
    oracle, and the EventSink sequence identical to the reference's trace."""
    worst = 0.0
    for op, s, thr, a, b, ref_events in _golden_cases(golden, prefix):
        events = []
        got = run_op(op, s, a, b, thr, sink=lambda e, n, m: events.append((int(e), n, m)))
        worst = max(worst, check_against_oracle(op, s, a, b, got))
        assert np.array_equal(np.array(events, dtype=np.int64).reshape(-1, 3), ref_events), (op, s)
    assert worst < 32


# ---------------------------------------------------- acceptance criterion 1
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("op", ["trmm", "trsm"])
def test_variant_coverage(cuda, op, dtype):
    """acceptance_main.cpp:67-113: all 16 variants, n in {64, 257}, m in
    {1, 3, 256}, threshold 8, alpha 1.5."""
    seed = 1000
    for s in oracle.all_variants(alpha=1.5):
        for n in (64, 257):
            for m in (1, 3, 256):
                seed += 1
                a = oracle.make_operand(s, op == "trsm", n, seed, dtype)
                b = oracle.make_rhs(s, n, m, seed * 3, dtype)
                got = run_op(op, s, a, b, 8)
                check_against_oracle(op, s, a, b, got)


@pytest.mark.parametrize("op", ["trmm", "trsm"])
def test_leaf_sizes_and_thresholds(cuda, op):
    """Leaf kernel across tile orders 1..256 (partial 32-row blocks) and the
    internal split above 256 (tile_limit raised)."""
    for n, thr in ((1, 1), (31, 64), (33, 64), (100, 128), (256, 256), (300, 512), (512, 512)):
        for s in (oracle.spec(0, 0, 0, 0, 1.5), oracle.spec(1, 1, 1, 1, -0.5), oracle.spec(0, 1, 1, 0, 2.0),
                  oracle.spec(1, 0, 0, 1, 1.0)):
            a = oracle.make_operand(s, op == "trsm", n, 77 + n)
            b = oracle.make_rhs(s, n, 45, 78 + n)
            check_against_oracle(op, s, a, b, run_op(op, s, a, b, thr))


# ---------------------------------------------------- criterion 2 / 3
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_threshold_invariance_and_single_base(cuda, dtype):
    eps = np.finfo(dtype).eps
    n, m = 17, 3
    for op in ("trmm", "trsm"):
        for s in oracle.all_variants(alpha=1.5):
            a = oracle.make_operand(s, op == "trsm", n, 2000 + n)
            a = a.astype(dtype, order="F")
            b = oracle.make_rhs(s, n, m, 2001, dtype)
            ref = run_op(op, s, a, b, n)
            tol = 32 * n * eps * oracle.masked_norm_inf(a, s.uplo, s.diag) * max(
                oracle.max_abs(b), oracle.max_abs(ref), 1.0) * 1.5
            for t in (1, 2, 16):
                assert oracle.max_abs_diff(run_op(op, s, a, b, t), ref) <= tol
            single = run_base(op, s, a, b, tile_limit=n)
            assert oracle.bitwise_equal(ref, single)
            assert oracle.bitwise_equal(run_op(op, s, a, b, n + 9), single)


def test_call_counts(cuda):
    """acceptance_main.cpp:172-203: 2^k - 1 GEMMs and 2^k leaves."""
    for op in ("trmm", "trsm"):
        for k in range(1, 6):
            n = 8 << k
            s = oracle.spec()
            a = oracle.make_operand(s, op == "trsm", n, 3000 + n)
            b = oracle.make_random(n, 3, 3001)
            ev = []
            run_op(op, s, a, b, 8, sink=lambda e, nn, mm: ev.append(e))
            assert ev.count(RecEvent.Gemm) == (1 << k) - 1
            leaf = RecEvent.BaseTrmm if op == "trmm" else RecEvent.BaseTrsm
            assert ev.count(leaf) == 1 << k and len(ev) == (1 << (k + 1)) - 1


# ------------------------------------------------------------ criterion 4
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_round_trip(cuda, dtype):
    eps = np.finfo(dtype).eps
    seed = 4000
    for n in (64, 257, 1024):
        for s in (oracle.spec(0, 0, 0, 0), oracle.spec(1, 1, 1, 0)):
            seed += 1
            a = oracle.make_dominant(n, s.uplo, seed, dtype)
            b = oracle.make_rhs(s, n, 4, seed * 3, dtype)
            x = run_op("trsm", s, a, b, 64)
            back = run_op("trmm", s, a, x, 64)
            tol = 64 * n * eps * oracle.masked_norm_inf(a, s.uplo, s.diag) * max(oracle.max_abs(b), 1.0)
            assert oracle.max_abs_diff(back, b) <= tol


# ------------------------------------------------------------ criterion 6
def test_masking_and_unit_diag_bitwise(cuda):
    for op in ("trmm", "trsm"):
        for s in oracle.all_variants():
            n, m = 17, 3
            clean = oracle.make_operand(s, True, n, 6000 + n)
            b = oracle.make_rhs(s, n, m, 6001)
            r_clean = run_op(op, s, clean, b, 4)
            poisoned = clean.copy(order="F")
            oracle.poison_opposite_triangle(poisoned, s.uplo)
            r_p = run_op(op, s, poisoned, b, 4)
            assert np.all(np.isfinite(r_p)) and oracle.bitwise_equal(r_clean, r_p), (op, s)
            if s.diag == 1:
                garbled = clean.copy(order="F")
                oracle.set_diagonal(garbled, 1234.5)
                assert oracle.bitwise_equal(r_clean, run_op(op, s, garbled, b, 4))
                oracle.set_diagonal(garbled, np.nan)
                assert oracle.bitwise_equal(r_clean, run_op(op, s, garbled, b, 4))


# ------------------------------------------------------------ criterion 7
def test_singular_global_index_matches_reference(cuda, golden):
    for side, uplo, trans, r, st, ref_row in golden["singular"]:
        s = oracle.spec(int(side), int(uplo), int(trans), 0)
        a = oracle.make_dominant(64, s.uplo, 7000 + int(r))
        a[r, r] = 0.0
        b = oracle.make_rhs(s, 64, 2, 7001)
        A, B = to_dev(a), to_dev(b)
        with pytest.raises(SingularityError) as e:
            rec_trsm(tspec(s), A.cview(), B.view(), Threshold(8))
        assert st == 4 and e.value.index() == ref_row == r


def test_unit_diag_ignores_zero_pivot(cuda):
    s = oracle.spec(diag=1)
    a = oracle.make_operand(s, True, 5, 61)
    a[3, 3] = 0.0
    run_base("trsm", s, a, oracle.make_random(5, 2, 62))


# ------------------------------------------------------------ alpha rules
def test_alpha_factoring(cuda):
    # TRSM: alpha applied once at entry -> bitwise equal to prescaled B
    # (test_recursion.cpp:283-301).
    n = 24
    s = oracle.spec(alpha=2.5)
    a = oracle.make_dominant(n, 0, 8900)
    b = oracle.make_random(n, 3, 8901)
    direct = run_op("trsm", s, a, b, 4)
    pre = F(b * 2.5)
    assert oracle.bitwise_equal(direct, run_op("trsm", oracle.spec(), a, pre, 4))
    # TRMM: folded alpha within 4 ulp of scaling afterwards (:262-281).
    for n in (8, 33):
        s = oracle.spec(trans=1, alpha=2.5)
        a = oracle.make_random(n, n, 8800 + n, 0.1, 1.0)
        b = oracle.make_random(n, 3, 8801, 0.1, 1.0)
        folded = run_op("trmm", s, a, b, 4)
        plain = run_op("trmm", oracle.spec(trans=1), a, b, 4) * 2.5
        assert np.all(np.abs(folded - plain) <= 4 * np.finfo(float).eps * np.abs(plain))


def test_trmm_alpha_zero_writes_zeros(cuda):
    s = oracle.spec(alpha=0.0)
    a = oracle.make_dominant(4, 0, 81)
    b = F(np.full((4, 2), np.nan))
    out = run_base("trmm", s, a, b)
    assert np.all(out == 0.0)
    out = run_op("trmm", s, oracle.make_random(40, 40, 3), F(np.full((40, 5), np.nan)), 8)
    assert np.all(out == 0.0)


# ------------------------------------------------------------ right == left^T
def test_right_equals_transposed_left(cuda):
    eps = np.finfo(float).eps
    for op in ("trmm", "trsm"):
        for uplo in (0, 1):
            for trans in (0, 1):
                n, m = 12, 5
                rs = oracle.spec(1, uplo, trans, 0)
                a = oracle.make_operand(rs, op == "trsm", n, 9500)
                b = oracle.make_random(m, n, 9501)
                right = run_op(op, rs, a, b, 3)
                ls = oracle.spec(0, uplo, 1 - trans, 0)
                left = run_op(op, ls, a, F(b.T), 3)
                tol = 32 * n * eps * oracle.masked_norm_inf(a, uplo, 0) * max(oracle.max_abs(b),
                                                                              oracle.max_abs(right), 1.0)
                assert oracle.max_abs_diff(right, left.T) <= tol


# ------------------------------------------------------------ validation
def test_driver_validation(cuda):
    s = tspec(oracle.spec())
    a = to_dev(oracle.make_dominant(4, 0, 9600))
    b = to_dev(oracle.make_random(4, 2, 9601))
    with pytest.raises(ConfigError):
        rec_trsm(s, a.cview(), b.view(), Threshold(0))
    with pytest.raises(ShapeError):
        rec_trmm(s, to_dev(oracle.make_random(4, 3, 1)).cview(), b.view(), Threshold(2))
    with pytest.raises(ShapeError):
        rec_trsm(s, a.cview(), to_dev(oracle.make_random(5, 2, 1)).view(), Threshold(2))
    shared = MatrixBuffer(8, 8, torch.float64, "cuda", 1.0)
    v = shared.view()
    with pytest.raises(AliasError):
        rec_trmm(s, v.subview(0, 0, 4, 4).as_const(), v.subview(3, 3, 4, 4), Threshold(2))
    # disjoint windows of one buffer are fine
    rec_trmm(s, v.subview(0, 0, 4, 4).as_const(), v.subview(4, 4, 4, 4), Threshold(2))
    rec_trsm(s, a.cview(), MatrixBuffer(4, 0, torch.float64, "cuda").view(), Threshold(2))
    rec_trmm(s, MatrixBuffer(0, 0, torch.float64, "cuda").cview(), MatrixBuffer(0, 2, torch.float64, "cuda").view())
    bad = TriangularSpec(alpha=math.inf)
    with pytest.raises(ConfigError):
        rec_trsm(bad, a.cview(), b.view())
    with pytest.raises(TileLimitError):
        trsm_base(s, to_dev(oracle.make_dominant(260, 0, 7)).cview(), to_dev(oracle.make_random(260, 2, 8)).view())


# ------------------------------------------------------------ determinism
def test_deterministic_and_shard_invariant(cuda):
    """run == rerun, graph == direct launch, and any column split of B gives
    bitwise the same columns (the P-GPU == 1-GPU invariant)."""
    for op in ("trsm", "trmm"):
        for dt in (np.float64, np.float32):
            s = oracle.spec(0, 0, 1, 0, 1.0)
            n, m = 700, 300
            a = oracle.make_operand(s, op == "trsm", n, 11, dt)
            b = oracle.make_random(n, m, 12, dtype=dt)
            full = run_op(op, s, a, b, 64)
            assert oracle.bitwise_equal(full, run_op(op, s, a, b, 64))
            assert oracle.bitwise_equal(full, run_op(op, s, a, b, 64, backend=Backend.cuda(flags=NO_GRAPH)))
            parts = [run_op(op, s, a, F(b[:, c0:c1]), 64) for c0, c1 in ((0, 37), (37, 200), (200, 300))]
            assert oracle.bitwise_equal(full, F(np.concatenate(parts, axis=1)))


def test_host_staged_equals_device(cuda):
    s = oracle.spec(0, 1, 0, 0, 0.75)
    a = oracle.make_operand(s, True, 300, 5)
    b = oracle.make_random(300, 70, 6)
    dev = run_op("trsm", s, a, b, 64)
    host = run_op("trsm", s, a, b, 64, device="cpu")
    assert oracle.bitwise_equal(dev, host)
    A = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a)), device="cpu")
    B = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(b)), device="cpu")
    B.data = B.data.pin_memory()
    rec_trsm(tspec(s), A.cview(), B.view(), Threshold(64))
    assert oracle.bitwise_equal(dev, to_np(B))


@pytest.mark.parametrize("op", ["trsm", "trmm"])
def test_host_streamed_all_variants(cuda, op, monkeypatch):
    """Host views take the first-use streamed path (A blocks and B chunks
    copied in, chunks copied back after their last writer): bitwise the
    device result for every variant, with several B chunks, alpha != 1, a
    device A with a host B, and the panelled fallback."""
    n, m = 2600, 96
    for side, uplo, trans, diag in [(0, 0, 0, 0), (0, 1, 1, 1), (1, 0, 1, 0), (1, 1, 0, 1), (0, 1, 0, 0), (1, 0, 0, 1)]:
        s = oracle.spec(side, uplo, trans, diag, 1.5)
        a = oracle.make_operand(s, op == "trsm", n, 11)
        b = oracle.make_rhs(s, n, m, 12)
        dev = run_op(op, s, a, b, 256)
        evs_dev, evs_host = [], []
        host = run_op(op, s, a, b, 256, device="cpu", sink=lambda e, nn, mm: evs_host.append((int(e), nn, mm)))
        run_op(op, s, a, b, 256, sink=lambda e, nn, mm: evs_dev.append((int(e), nn, mm)))
        assert oracle.bitwise_equal(dev, host), (side, uplo, trans, diag)
        assert evs_dev == evs_host
        # device A, host B
        A = to_dev(a)
        B = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(b)), device="cpu")
        fn = rec_trmm if op == "trmm" else rec_trsm
        fn(tspec(s), A.cview(), B.view(), Threshold(256))
        assert oracle.bitwise_equal(dev, to_np(B))
    monkeypatch.setenv("RECTRI_CU_HOST_PANEL", "40")  # panelled fallback
    s = oracle.spec(0, 0, 0, 0, 1.0)
    a = oracle.make_operand(s, op == "trsm", n, 13)
    b = oracle.make_rhs(s, n, m, 14)
    assert oracle.bitwise_equal(run_op(op, s, a, b, 256), run_op(op, s, a, b, 256, device="cpu"))


def test_host_streamed_singular(cuda):
    n = 2100
    s = oracle.spec(0, 0, 0, 0, 1.0)
    a = oracle.make_operand(s, True, n, 3)
    a[1500, 1500] = 0.0
    b = oracle.make_rhs(s, n, 8, 4)
    A = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a)), device="cpu")
    B = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(b)), device="cpu")
    with pytest.raises(SingularityError) as ei:
        rec_trsm(tspec(s), A.cview(), B.view(), Threshold(256))
    assert ei.value.index() == 1500


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_trmm_concurrent_halves_bitwise_serial(cuda, dt, monkeypatch):
    """Small TRMM nodes run the first half beside the GEMM into a scratch
    product and add it after the join (driver.cu ConcCtx): bitwise the
    serial recursion (RECTRI_CU_TRMM_CONC=0) on every variant, alpha != 1,
    graph and direct launches, several depths of concurrent nodes."""
    for n, m, t in ((1000, 130, 64), (520, 40, 32)):
        for s in oracle.all_variants(alpha=-1.25):
            a = oracle.make_operand(s, False, n, 31, dt)
            b = oracle.make_rhs(s, n, m, 32, dt)
            monkeypatch.setenv("RECTRI_CU_TRMM_CONC", "0")
            ser = run_op("trmm", s, a, b, t, backend=Backend.cuda(flags=NO_GRAPH))
            monkeypatch.setenv("RECTRI_CU_TRMM_CONC", "1")
            conc_graph = run_op("trmm", s, a, b, t)
            conc_direct = run_op("trmm", s, a, b, t, backend=Backend.cuda(flags=NO_GRAPH))
            assert oracle.bitwise_equal(ser, conc_graph), (n, s)
            assert oracle.bitwise_equal(ser, conc_direct), (n, s)


@pytest.mark.parametrize("op", ["trsm", "trmm"])
def test_host_streamed_time_panels(cuda, op, monkeypatch):
    """The streamed host path in consecutive right-hand-side panels (copy-back
    of panel t under the compute of panel t+1): bitwise the device result,
    Left and Right, ragged last panel, alpha != 1."""
    n, m = 1100, 150
    monkeypatch.setenv("RECTRI_CU_E2E_PANELS", "3")
    for side, uplo, trans, diag in [(0, 0, 0, 0), (1, 1, 1, 1), (0, 1, 0, 0), (1, 0, 0, 1)]:
        s = oracle.spec(side, uplo, trans, diag, 0.5)
        a = oracle.make_operand(s, op == "trsm", n, 21)
        b = oracle.make_rhs(s, n, m, 22)
        dev = run_op(op, s, a, b, 128)
        host = run_op(op, s, a, b, 128, device="cpu")
        assert oracle.bitwise_equal(dev, host), (side, uplo, trans, diag)


@pytest.mark.parametrize("side,uplo,trans", list(__import__("itertools").product((0, 1), (0, 1), (0, 1))))
def test_trsm_non_dominant_well_conditioned(cuda, monkeypatch, side, uplo, trans):
    """The default leaf applies explicit inverses of its 32x32 diagonal blocks
    (leaf64_v3.cu) instead of the reference's substitution; every other test
    uses diagonally dominant triangles.  Here A is the Cholesky factor of an
    SPD matrix with eigenvalues in [1, 100] -- condition number about 10, far
    from diagonally dominant (off-diagonal row sums exceed the diagonal).
    The result must pass the reference's residual criterion and agree with
    the reference-order leaf (RECTRI_CU_LEAF=2) to a cond-scaled forward bound."""
    import paper_2504_13821_b200 as rc

    n, m = 768, 300
    rng = np.random.default_rng(900 + 4 * side + 2 * uplo + trans)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    spd = (q * np.logspace(0, 2, n)) @ q.T
    low = np.linalg.cholesky(spd)
    a = F(low if uplo == 0 else low.T)
    offsum = np.abs(np.tril(low, -1)).sum(1)
    assert np.mean(offsum > np.abs(np.diag(low))) > 0.5  # not diagonally dominant
    s = oracle.spec(side, uplo, trans, 0, 1.0)
    b = F(rng.uniform(-1, 1, (n, m) if side == 0 else (m, n)))
    got = run_op("trsm", s, a, b, 256)
    check_against_oracle("trsm", s, a, b, got)
    monkeypatch.setenv("RECTRI_CU_LEAF", "2")
    rc.clear_graph_cache()
    ref_order = run_op("trsm", s, a, b, 256)
    monkeypatch.delenv("RECTRI_CU_LEAF")
    rc.clear_graph_cache()
    cond = np.linalg.cond(low)
    err = np.max(np.abs(got - ref_order)) / np.max(np.abs(ref_order))
    assert err <= 64 * n * np.finfo(float).eps * cond, (err, cond)
