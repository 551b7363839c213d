"""Bench harness parity: CSV schema, ratio join and
exit codes on CPU; sweeps and the residual gate on the GPU
(tests/test_bench.cpp, acceptance criterion 9)."""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2504_13821_b200 import OpKind, TriangularSpec, harness as h
from paper_2504_13821_b200.errors import JoinError

ROOT = Path(__file__).resolve().parents[1]
CLI = [sys.executable, str(ROOT / "tools" / "rectri_bench.py")]


def _rec(n, t=1e-3):
    return h.BenchRecord("trsm", "left-lower-n-nonunit", n, 3, 2, "cuda", "f32", t, t / 2, n * n * 3 / t / 1e9)


def test_csv_headers_and_round_trip(tmp_path):
    assert h.SWEEP_CSV_HEADER == "op,variant,n,m,threshold,backend,elem,median_time_s,min_time_s,gflops"
    assert h.RATIO_CSV_HEADER == "op,variant,n,m,baseline_s,candidate_s,ratio_percent"
    p = tmp_path / "s.csv"
    h.write_sweep_csv(str(p), [_rec(4), _rec(8)])
    text = p.read_text().splitlines()
    assert text[0] == h.SWEEP_CSV_HEADER and len(text) == 3
    back = h.read_sweep_csv(str(p))
    assert [r.n for r in back] == [4, 8] and back[0].backend == "cuda"


def test_ratio_self_is_100_and_join_errors(tmp_path):
    a = tmp_path / "a.csv"
    b = tmp_path / "b.csv"
    h.write_sweep_csv(str(a), [_rec(4), _rec(8)])
    h.write_sweep_csv(str(b), [_rec(4)])
    recs = h.ratio_report(str(a), str(a), str(tmp_path / "r.csv"))
    assert [r.ratio_percent for r in recs] == [100.0, 100.0]
    assert (tmp_path / "r.csv").read_text().splitlines()[0] == h.RATIO_CSV_HEADER
    with pytest.raises(JoinError):
        h.ratio_report(str(a), str(b))


def test_cli_exit_codes(tmp_path):
    r = subprocess.run(CLI + ["sweep", "--op", "bogus", "--sizes", "4"], capture_output=True, text=True)
    assert r.returncode == 2
    r = subprocess.run(CLI + ["frobnicate"], capture_output=True, text=True)
    assert r.returncode == 2
    a = tmp_path / "a.csv"
    h.write_sweep_csv(str(a), [_rec(4), _rec(8)])
    r = subprocess.run(CLI + ["ratio", "--baseline", str(a), "--candidate", str(a)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.splitlines()[0] == h.RATIO_CSV_HEADER


def test_reference_generator_stream():
    """make_inputs is the reference's bench stream (bench.cpp:32-61): A then
    B from one mt19937_64; checked against the oracle's restatement."""
    import oracle

    a, b = h.make_inputs(OpKind.Trsm, TriangularSpec(), 6, 4, 99, "f64")
    ra, rb = oracle.bench_inputs(6, 6, 4, True, 0, 0, 99)
    assert np.array_equal(a, ra) and np.array_equal(b, rb)


@pytest.mark.gpu
def test_gpu_sweep_and_fault_gate(cuda, tmp_path):
    out = tmp_path / "s.csv"
    base = CLI + ["sweep", "--op", "trsm", "--side", "left", "--uplo", "lower", "--trans", "n", "--diag", "nonunit",
                  "--sizes", "64,96", "--m", "fixed:3", "--threshold", "16", "--backend", "cuda", "--reps", "3",
                  "--warmup", "1", "--elem", "f64"]
    r = subprocess.run(base + ["--out", str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert out.read_text().splitlines()[0] == h.SWEEP_CSV_HEADER
    r = subprocess.run(base + ["--inject-fault"], capture_output=True, text=True)
    assert r.returncode == 1, r.stderr
    r = subprocess.run(CLI + ["crossover", "--op", "trmm", "--sizes", "128", "--m", "square", "--thresholds", "32,64",
                              "--elem", "f32", "--reps", "2", "--warmup", "1"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert len(r.stdout.splitlines()) == 3


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["trsm", "trmm"])
def test_gpu_cublas_backend_every_variant(cuda, tmp_path, op):
    """The cuBLAS comparison backend covers all 16 variants (the gate checks
    its results too), so the Fig.-3-style ratio report can join any variant."""
    import itertools

    for side, uplo, trans, diag in itertools.product(("left", "right"), ("lower", "upper"), ("n", "t"),
                                                     ("nonunit", "unit")):
        outs = {}
        for backend in ("cuda", "cublas"):
            out = tmp_path / f"{op}-{side}-{uplo}-{trans}-{diag}-{backend}.csv"
            r = subprocess.run(CLI + ["sweep", "--op", op, "--side", side, "--uplo", uplo, "--trans", trans,
                                      "--diag", diag, "--sizes", "96", "--m", "fixed:40", "--threshold", "32",
                                      "--backend", backend, "--reps", "2", "--warmup", "1", "--elem", "f64",
                                      "--out", str(out)], capture_output=True, text=True)
            assert r.returncode == 0, (side, uplo, trans, diag, backend, r.stderr)
            outs[backend] = out
        recs = h.ratio_report(str(outs["cublas"]), str(outs["cuda"]))
        assert len(recs) == 1 and recs[0].ratio_percent > 0
