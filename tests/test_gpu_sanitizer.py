"""Race / sync / memory checking of the real kernels with compute-sanitizer
(the role of the reference's workgroup simulator and its planted-race test,
workgroup.cpp:138-177, 333-349; test_workgroup.cpp:144-176)."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SAN = "/usr/local/cuda/bin/compute-sanitizer"


def _san(tool, args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    cmd = [SAN, "--tool", tool, "--kernel-name", "kns=rectri_cu", "--print-limit", "5",
           sys.executable, str(ROOT / "tools" / "prof_run.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    # GPU pools may close the tool (it exits 86 with a notice instead of
    # running): nothing was checked, so the test is skipped, not passed.
    if r.returncode == 86 and "closed" in (r.stdout + r.stderr):
        pytest.skip("compute-sanitizer is closed on this GPU pool: " + (r.stdout + r.stderr).strip()[:160])
    return r


@pytest.mark.parametrize("tool", ["racecheck", "synccheck", "memcheck"])
@pytest.mark.parametrize("args", [["leaf", "100", "70"], ["trmmleaf", "100", "70"], ["gemm", "130", "70", "50"], ["gemm", "200", "130", "1100"],
                                  ["trsm", "300", "40", "64"], ["sgemm", "130", "70", "50"], ["sgemm", "256", "200", "300"],
                                  ["leaf32", "100", "70"], ["strsm", "300", "40", "64"], ["trmm", "520", "40", "32"]])
def test_kernels_clean(cuda, tool, args):
    # racecheck does not model mbarrier-ordered refills (the default fp64
    # leaf's bulk-copy ring, leaf64_v3.cu, and the fp32 GEMM's per-stage
    # cp.async mbarriers, gemm_f32.cu, report as hazards); it checks the
    # barrier-synchronised v2 leaf and v1 fp32 GEMM, the other tools the
    # defaults, whose ordering test_gpu_leaf.py / test_gpu_gemm.py stress.
    env = None
    if tool == "racecheck" and "gemm" not in args[0]:
        env = {"RECTRI_CU_LEAF": "2", "RECTRI_CU_SGEMM": "1"}
    elif tool == "racecheck" and args[0] == "sgemm":
        env = {"RECTRI_CU_SGEMM": "1"}
    r = _san(tool, args, env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    if tool == "racecheck":
        # racecheck prints its own summary line instead of "ERROR SUMMARY"
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, out[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]


def test_planted_race_is_detected(cuda):
    # the planted missing barrier lives in the v1 leaf (leaf.cu)
    r = _san("racecheck", ["leaf", "100", "70"], {"RECTRI_CU_LEAF_DEBUG": "3", "RECTRI_CU_LEAF": "1"})
    out = r.stdout + r.stderr
    m = re.search(r"RACECHECK SUMMARY: (\d+) hazards displayed \((\d+) errors", out)
    assert m and int(m.group(1)) > 0 and int(m.group(2)) > 0, out[-3000:]


@pytest.mark.parametrize("tool", ["synccheck", "initcheck"])
@pytest.mark.parametrize("args", [["leaf", "256", "16384"], ["leaf", "256", "3000"], ["leaf", "256", "1000"],
                                  ["trmmleaf", "256", "16384"], ["leaf32", "256", "16384"],
                                  ["leaf32", "256", "1000"], ["trsm", "1024", "4096", "256"]])
def test_default_leaves_at_c3_leaf_shape(cuda, tool, args):
    """The DEFAULT leaves (leaf3_kernel, fp64; leaf32_kernel, fp32) at the C3
    leaf shape (256 x 16384: 32-wide panels) and at the 16- / 8-wide panel
    widths: barrier use (synccheck) and no read of uninitialised device
    memory (initcheck).  Their ring ordering -- which racecheck cannot model
    -- is covered by test_gpu_leaf.py's replay-determinism stress test."""
    r = _san(tool, args)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
