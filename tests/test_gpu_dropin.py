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
