"""CPU test of bench.py's reference arm (the reference's own CPU path from
oracle/_ref) and its JSON-line contract, at a tiny size."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built here")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--n", "256", "--ref-cols", "16",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GFLOP/s"
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_gpus_flag_spawns_ranks_dry_gloo():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks itself (the
    driver's `--gpus N` form), rendezvous on 127.0.0.1, broadcasts A from rank
    0 and takes the max over ranks -- here on gloo, with no compute."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-gloo", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] and d["broadcast_ok"] and d["backend"] == "gloo"
    assert d["value"] is None  # nothing computed: no number is claimed
    assert d["config"]["m_total"] == 2 * d["config"]["m_per_gpu"]
    assert "rank 0 of 2" in r.stderr and "rank 1 of 2" in r.stderr
