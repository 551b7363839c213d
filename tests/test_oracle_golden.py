"""Pins the C restatement in oracle/ against the reference's own outputs
(tests/golden/golden_v1.npz, written by tests/golden/make_golden.py from
oracle/_ref = the reference compiled from /root/reference).  CPU only."""
import numpy as np
import pytest

import oracle


def _spec_of(meta, alpha):
    return oracle.spec(int(meta[1]), int(meta[2]), int(meta[3]), int(meta[4]), float(alpha))


@pytest.mark.parametrize("tag,dt", [("f64", np.float64), ("f32", np.float32)])
def test_generators_bitwise(golden, tag, dt):
    # tests/test_support.hpp:38-62 -- mt19937_64 + uniform_real_distribution.
    assert np.array_equal(golden[f"gen/random_4x3_s11_{tag}"], oracle.make_random(4, 3, 11, dtype=dt))
    assert np.array_equal(golden[f"gen/random_64x5_s12345_{tag}"], oracle.make_random(64, 5, 12345, dtype=dt))
    assert np.array_equal(golden[f"gen/random_9x9_s3_lo01_{tag}"], oracle.make_random(9, 9, 3, 0.1, 1.0, dtype=dt))
    assert np.array_equal(golden[f"gen/dominant_33_lower_s7_{tag}"], oracle.make_dominant(33, 0, 7, dt))
    assert np.array_equal(golden[f"gen/dominant_33_upper_s7_{tag}"], oracle.make_dominant(33, 1, 7, dt))


def test_bench_inputs_follow_one_stream():
    # src/bench.cpp:32-61: A then B from ONE mt19937_64 stream; TRSM NonUnit
    # diagonal := off-diagonal |row sum| + 1.
    n, m, seed = 6, 4, 99
    a, b = oracle.bench_inputs(n, n, m, True, 0, 0, seed)
    stream = oracle.make_random(n * n + n * m, 1, seed)[:, 0]
    a_raw = stream[: n * n].reshape(n, n, order="F")
    assert np.array_equal(b, stream[n * n:].reshape(n, m, order="F"))
    off = np.tril(a_raw, -1)
    expect = a_raw.copy()
    np.fill_diagonal(expect, np.abs(off).sum(axis=1) + 1.0)
    assert np.array_equal(a, expect)


def _cases(golden, prefix):
    for i in range(int(golden[f"{prefix}/count"])):
        k = f"{prefix}/{i:04d}"
        yield golden[k + "/meta"], float(golden[k + "/alpha"]), golden[k + "/a"], golden[k + "/b"], \
            golden[k + "/oracle"], golden[k + "/rec"]


@pytest.mark.parametrize("prefix", ["case", "mid"])
def test_oracle_restatement_matches_reference_oracle(golden, prefix):
    """src/oracle.cpp restated in C gives the reference oracle's results bit
    for bit (same double arithmetic in the same order)."""
    n_checked = 0
    for meta, alpha, a, b, orc, _ in _cases(golden, prefix):
        s = _spec_of(meta, alpha)
        a = np.asfortranarray(a)
        b = np.asfortranarray(b)
        got = oracle.oracle_trmm(s, a, b) if meta[0] == 0 else oracle.oracle_trsm(s, a, b)
        assert np.array_equal(got, orc), f"case meta={meta}"
        n_checked += 1
    assert n_checked > 0


def test_reference_recursion_within_oracle_tolerance(golden):
    """The reference's own rec_* outputs satisfy the criterion-1 bound against
    the restated oracle -- the bound the GPU path is held to."""
    for meta, alpha, a, b, orc, rec in _cases(golden, "case"):
        s = _spec_of(meta, alpha)
        eps = np.finfo(a.dtype).eps
        n = a.shape[0]
        scale = oracle.masked_norm_inf(a, s.uplo, s.diag) * max(oracle.max_abs(b), oracle.max_abs(rec), 1.0) \
            * max(1.0, abs(alpha))
        tol = 32 * max(n, 1) * eps * scale
        if meta[0] == 0:
            assert oracle.max_abs_diff(rec, orc) <= tol
        else:
            assert oracle.trsm_residual_inf(s, a, rec, b) <= tol


def test_oracle_singularity_index():
    # src/oracle.cpp:101-102: exact zero on the materialized diagonal.
    a = oracle.make_dominant(8, 0, 3)
    a[5, 5] = 0.0
    with pytest.raises(oracle.OracleSingular) as e:
        oracle.oracle_trsm(oracle.spec(), a, oracle.make_random(8, 2, 4))
    assert e.value.index == 5


def test_frozen_examples_oracle():
    # SPEC.md:191-202, test_base_kernels.cpp:13-68 through the oracle.
    A = np.asfortranarray([[2.0, 0.0], [1.0, 4.0]])
    B = np.asfortranarray([[2.0], [6.0]])
    assert oracle.oracle_trsm(oracle.spec(), A, B).ravel().tolist() == [1.0, 1.25]
    A2 = np.asfortranarray([[2.0, 0.0], [3.0, 4.0]])
    ones = np.asfortranarray([[1.0], [1.0]])
    assert oracle.oracle_trmm(oracle.spec(trans=1), A2, ones).ravel().tolist() == [5.0, 4.0]
    assert oracle.oracle_trmm(oracle.spec(), A2, ones).ravel().tolist() == [2.0, 7.0]
    garbage = np.asfortranarray([[999.0, 0.0], [3.0, 999.0]])
    assert oracle.oracle_trmm(oracle.spec(diag=1), garbage, ones).ravel().tolist() == [1.0, 4.0]


def test_events_golden_shape(golden):
    """Event traces recorded from the reference: 2^k-1 GEMMs / 2^k leaves for
    power-of-two n, leaf events carry (n, rhs) (recursion.cpp:94-97, 139)."""
    for meta, alpha, a, b, _, _ in _cases(golden, "mid"):
        k = None
    ev = golden["mid/0000/events"]
    # n = 64, t = 8, trmm: 8 leaves + 7 GEMMs.
    assert (ev[:, 0] == 0).sum() == 7 and (ev[:, 0] == 1).sum() == 8
