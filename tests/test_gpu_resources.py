"""GPU tests of the library's cross-call resources: cached graphs own their
scratch (so replays of different graphs never share or outlive it), the
host-operand staging serves one call at a time, deferred ASYNC singularity
checks survive cache clears and are bounded per stream, and the non-finite
behaviour of the default leaf is pinned (documented divergence from the
reference's substitution order)."""
import threading

import numpy as np
import pytest
import torch

import oracle
import paper_2504_13821_b200 as rc
from paper_2504_13821_b200 import (ASYNC, NO_GRAPH, TF32X3, Backend, SingularityError, Threshold, rec_trmm,
                                   rec_trsm)
from tests._util import check_against_oracle, run_op, to_dev, to_np, tspec

pytestmark = pytest.mark.gpu

F = np.asfortranarray


def test_tf32x3_graph_replay_after_larger_capture(cuda):
    """3xTF32 at n = 1024, then 4096, then 1024 again on the first buffers:
    the replayed first graph uses its own split scratch (the larger capture
    must not have freed it).  Bitwise equal to an uncached direct run."""
    rc.clear_graph_cache()
    s = oracle.spec(0, 0, 0, 0, 1.0)
    be = Backend.cuda(flags=TF32X3)
    bufs = {}
    for n in (1024, 4096):
        a = oracle.make_dominant(n, 0, 3).astype(np.float32)
        b = oracle.make_random(n, n, 4).astype(np.float32)
        A, B = to_dev(F(a)), to_dev(F(b))
        rec_trsm(tspec(s), A.cview(), B.view(), Threshold(256), be)
        bufs[n] = (a, b, A, B)
    a, b, A, B = bufs[1024]
    # other allocations take whatever memory a freed buffer released
    junk = [torch.full((1 << 22,), 7.0, device=cuda) for _ in range(8)]
    B.tensor().copy_(torch.from_numpy(F(b)).to(cuda))
    rec_trsm(tspec(s), A.cview(), B.view(), Threshold(256), be)  # replay of the first graph
    got = to_np(B)
    want = run_op("trsm", s, F(a), F(b), 256, Backend.cuda(flags=TF32X3 | NO_GRAPH))
    assert oracle.bitwise_equal(got, want)
    del junk


def test_disjoint_async_calls_on_two_streams_threshold_above_tile(cuda):
    """threshold > 256 leaves run the internal unpacked-leaf path with scratch:
    two disjoint cached problems replayed at once on two streams must not
    share it (the reference is reentrant for disjoint problems)."""
    rc.clear_graph_cache()
    s = oracle.spec(0, 0, 0, 0, 1.0)
    n, m = 1024, 3000
    probs = []
    for k in range(2):
        a = oracle.make_dominant(n, 0, 10 + k)
        b = oracle.make_random(n, m, 20 + k)
        probs.append((a, b, to_dev(a), to_dev(b)))
    want = [run_op("trsm", s, a, b, 512, Backend.cuda(flags=NO_GRAPH)) for a, b, _, _ in probs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    for rep in range(3):  # first call captures, later ones replay concurrently
        for (a, b, A, B) in probs:
            B.tensor().copy_(torch.from_numpy(F(b)).to(cuda))
        torch.cuda.synchronize()
        for (a, b, A, B), st in zip(probs, streams):
            rec_trsm(tspec(s), A.cview(), B.view(), Threshold(512), Backend.cuda(stream=st, flags=ASYNC))
        for st in streams:
            rc.sync(st)
        for (a, b, A, B), w in zip(probs, want):
            assert oracle.bitwise_equal(to_np(B), w), rep


def test_host_operands_from_two_threads(cuda):
    """Host-resident A and B from two threads at once: each call owns the
    device staging for its duration, so both results are exact."""
    s = oracle.spec(0, 0, 0, 0, 1.0)
    n, m = 768, 1500
    cases = [(oracle.make_dominant(n, 0, 30 + k), oracle.make_random(n, m + 300 * k, 40 + k)) for k in range(2)]
    want = [run_op("trsm", s, a, b, 256) for a, b in cases]
    outs = [None, None]
    errs = []

    def work(k):
        try:
            torch.cuda.set_device(0)
            for _ in range(3):
                a, b = cases[k]
                A = rc.MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a)), device="cpu")
                B = rc.MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(b)), device="cpu")
                rec_trsm(tspec(s), A.cview(), B.view(), Threshold(256), Backend.cuda(device=0))
                outs[k] = to_np(B)
                assert oracle.bitwise_equal(outs[k], want[k])
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert rc.device_bytes_held() > 0
    rc.release_staging()
    held = rc.device_bytes_held()
    rc.clear_graph_cache()
    assert rc.device_bytes_held() <= held


def _singular_problem(n=64, row=37):
    a = oracle.make_dominant(n, 0, 50)
    a[row, row] = 0.0
    return a, oracle.make_random(n, 8, 51)


def test_deferred_singularity_survives_cache_clear(cuda):
    s = oracle.spec(0, 0, 0, 0, 1.0)
    a, b = _singular_problem()
    A, B = to_dev(a), to_dev(b)
    st = torch.cuda.Stream()
    rec_trsm(tspec(s), A.cview(), B.view(), Threshold(8), Backend.cuda(stream=st, flags=ASYNC))
    rc.clear_graph_cache()
    with pytest.raises(SingularityError) as e:
        rc.sync(st)
    assert e.value.index() == 37
    rc.sync(st)  # reported once


def test_pending_checks_bounded_per_stream(cuda):
    """More ASYNC singular calls than the per-stream pending bound: the early
    settlement keeps the first singular row for the caller's sync."""
    s = oracle.spec(0, 0, 0, 0, 1.0)
    a, b = _singular_problem()
    A, B = to_dev(a), to_dev(b)
    st = torch.cuda.Stream()
    for _ in range(600):
        rec_trsm(tspec(s), A.cview(), B.view(), Threshold(8), Backend.cuda(stream=st, flags=ASYNC))
    with pytest.raises(SingularityError) as e:
        rc.sync(st)
    assert e.value.index() == 37
    rc.sync(st)


@pytest.mark.parametrize("version", [2, 3])
def test_nonfinite_rhs_row_propagation(cuda, monkeypatch, version):
    """An Inf in one right-hand-side row k.  Substitution (the reference,
    base_kernels.cpp:73-88; leaf v2) leaves rows before k finite and exact.
    The default v3 leaf applies each 32x32 diagonal block as a dense product
    (-inv(L'_II) b_I), so 0 * Inf reaches the rows of k's own 32-row block
    above k as NaN; rows of earlier blocks stay finite and equal the
    reference order to rounding.  Rows at or after k are non-finite in both."""
    monkeypatch.setenv("RECTRI_CU_LEAF", str(version))
    rc.clear_graph_cache()
    s = oracle.spec(0, 0, 0, 0, 1.0)
    n, m, k = 128, 16, 70  # k in the 64..95 row block
    a = oracle.make_dominant(n, 0, 60)
    b = oracle.make_random(n, m, 61)
    b[k, 3] = np.inf
    got = run_op("trsm", s, a, b, 128)
    ref = oracle.oracle_trsm(s, a, b)
    col = got[:, 3]
    assert np.all(np.isfinite(col[:64]))
    assert np.allclose(col[:64], ref[:64, 3], rtol=1e-13, atol=1e-13)
    assert not np.isfinite(col[k])
    if version == 2:
        assert np.all(np.isfinite(col[:k])) and np.allclose(col[:k], ref[:k, 3], rtol=1e-13, atol=1e-13)
    else:
        assert np.all(np.isnan(col[64:k]))
    others = np.delete(np.arange(m), 3)
    assert np.all(np.isfinite(got[:, others]))
    monkeypatch.delenv("RECTRI_CU_LEAF")
    rc.clear_graph_cache()


def test_pageable_host_operands_singular_and_exact(cuda):
    """Pageable (plain numpy / CPU-tensor) A and B go through the pinned
    bounce staging: bitwise the device-resident result, and a zero pivot
    still raises SingularityError with its global row (the staging drains
    before the error surfaces)."""
    s = oracle.spec(0, 0, 0, 0, 1.0)
    n, m = 1500, 2300
    a = oracle.make_dominant(n, 0, 70)
    b = oracle.make_random(n, m, 71)
    want = run_op("trsm", s, a, b, 256)
    A = rc.MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a)), device="cpu")
    B = rc.MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(b)), device="cpu")
    rec_trsm(tspec(s), A.cview(), B.view(), Threshold(256), Backend.cuda(device=0))
    assert oracle.bitwise_equal(to_np(B), want)
    a2 = a.copy()
    a2[777, 777] = 0.0
    A2 = rc.MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a2)), device="cpu")
    B2 = rc.MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(b)), device="cpu")
    with pytest.raises(SingularityError) as e:
        rec_trsm(tspec(s), A2.cview(), B2.view(), Threshold(256), Backend.cuda(device=0))
    assert e.value.index() == 777


_PDL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import oracle
import paper_2504_13821_b200 as rc
from paper_2504_13821_b200 import Backend, Threshold, rec_trmm, rec_trsm
from tests._util import to_dev, to_np, tspec
outs = []
for dt in (np.float64, np.float32):
    for op, uplo in (("trsm", 0), ("trmm", 1)):
        s = oracle.spec(0, uplo, 0, 0, 1.0)
        a = oracle.make_dominant(1024, uplo, 5).astype(dt)
        b = oracle.make_random(1024, 1500, 6).astype(dt)
        A, B = to_dev(np.asfortranarray(a)), to_dev(np.asfortranarray(b))
        (rec_trsm if op == "trsm" else rec_trmm)(tspec(s), A.cview(), B.view(), Threshold(256), Backend.cuda())
        outs.append(to_np(B))
np.savez({out!r}, *outs)
"""


def test_pdl_launch_is_bitwise_neutral(cuda, tmp_path):
    """Programmatic dependent launch (RECTRI_CU_PDL, read once per process)
    only moves launch latency: captured recursions give the same bits with
    and without it, both precisions, TRSM and TRMM."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    res = []
    for pdl in ("0", "1"):
        out = str(tmp_path / f"pdl{pdl}.npz")
        env = dict(os.environ, RECTRI_CU_PDL=pdl)
        r = subprocess.run([sys.executable, "-c", _PDL_SCRIPT.format(root=root, out=out)], env=env,
                           capture_output=True, text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stderr[-2000:]
        z = np.load(out)
        res.append([z[k] for k in sorted(z.files)])
    for x, y in zip(*res):
        assert oracle.bitwise_equal(x, y)
