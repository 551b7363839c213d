"""Runs the C++ drop-in example (reference-style user code linked to the
sm_100a library) on the GPU."""
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_cpp_dropin_example_runs(cuda):
    from paper_2504_13821_b200 import build as b

    exe = b.build_dropin_example()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin_example: ok" in r.stdout


def test_dropin_bench_pageable_vectors(cuda):
    """Reference-caller-shaped e2e: rec_trsm<double> on std::vector-backed
    MatrixBuffers (pageable) through the pinned bounce staging -- its
    residual gate must pass (exit 0) and the timing line must parse."""
    import json

    from paper_2504_13821_b200 import build as b

    exe = b.build_dropin_bench()
    r = subprocess.run([str(exe), "2048", "3000", "2", "1"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["finite"] and d["eta"] <= 32 and len(d["step_ms"]) == 2
