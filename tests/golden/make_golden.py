"""Generates tests/golden/golden_v1.npz from the REFERENCE itself.

Run in the build container (needs /root/reference and oracle/_ref, built by
``make -C oracle ref``):

    python tests/golden/make_golden.py

Everything stored here is an output of the unmodified reference library
(oracle/_ref/librectri_ref.so): its generators (tests/test_support.hpp),
its oracle (src/oracle.cpp), its recursive drivers (src/recursion.cpp) with
the EventSink trace, its singularity reporting and its schema table.  The
fixtures pin the C restatement in oracle/ (CPU tests) and serve as golden
vectors for the GPU path (GPU tests).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from oracle import ref  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden_v1.npz"


def operand(spec, op, n, seed, dtype):
    # test_recursion.cpp:35-44, through the REFERENCE generators.
    if op == "trsm":
        a = ref.make_dominant(n, spec.uplo, seed, dtype)
        if spec.diag == 1:
            ref.damp_off_diagonal(a, 1.0 / n)
        return a
    return ref.make_random(n, n, seed, dtype=dtype)


def rhs(spec, n, m, seed, dtype):
    return ref.make_random(n, m, seed, dtype=dtype) if spec.side == 0 else ref.make_random(m, n, seed, dtype=dtype)


def main() -> None:
    if not ref.available():
        raise SystemExit("oracle/_ref/librectri_ref.so missing: make -C oracle ref")
    g: dict[str, np.ndarray] = {}

    # 1. Generator streams (tests/test_support.hpp:38-62).
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        g[f"gen/random_4x3_s11_{tag}"] = ref.make_random(4, 3, 11, dtype=dt)
        g[f"gen/random_64x5_s12345_{tag}"] = ref.make_random(64, 5, 12345, dtype=dt)
        g[f"gen/random_9x9_s3_lo01_{tag}"] = ref.make_random(9, 9, 3, 0.1, 1.0, dtype=dt)
        g[f"gen/dominant_33_lower_s7_{tag}"] = ref.make_dominant(33, 0, 7, dtype=dt)
        g[f"gen/dominant_33_upper_s7_{tag}"] = ref.make_dominant(33, 1, 7, dtype=dt)

    # 2. Oracle + recursion outputs across every variant (the sizes of
    #    test_recursion.cpp:149-183, threshold 2, alpha 1.5), both kinds.
    idx = 0
    seed = 5000
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        for op in ("trmm", "trsm"):
            for spec in oracle.all_variants(alpha=1.5):
                for n in (1, 2, 3, 5, 8, 17):
                    for m in (1, 3):
                        seed += 1
                        a = operand(spec, op, n, seed, dt)
                        b = rhs(spec, n, m, seed * 5, dt)
                        st, out, events, _ = ref.rec(op, spec, a, b, 2, trace=True)
                        assert st == 0, ref.last_error()
                        st2, orc, _ = ref.oracle(op, spec, a, b)
                        assert st2 == 0
                        k = f"case/{idx:04d}"
                        g[k + "/meta"] = np.array([0 if op == "trmm" else 1, spec.side, spec.uplo, spec.trans,
                                                   spec.diag, n, m, 2, 0 if tag == "f32" else 1], dtype=np.int64)
                        g[k + "/alpha"] = np.array(spec.alpha)
                        g[k + "/a"] = a
                        g[k + "/b"] = b
                        g[k + "/rec"] = out
                        g[k + "/oracle"] = orc
                        g[k + "/events"] = np.array(events, dtype=np.int64).reshape(-1, 3)
                        idx += 1
    g["case/count"] = np.array(idx)

    # 3. Medium fp64 cases through deeper recursion (threshold 8) incl. the
    #    odd split sizes of acceptance criterion 1 (acceptance_main.cpp:67-113).
    midx = 0
    for op in ("trmm", "trsm"):
        for spec in oracle.all_variants(alpha=1.5):
            for n, m in ((64, 3), (57, 5)):
                seed += 1
                a = operand(spec, op, n, seed, np.float64)
                b = rhs(spec, n, m, seed * 3, np.float64)
                st, out, events, _ = ref.rec(op, spec, a, b, 8, trace=True)
                assert st == 0
                _, orc, _ = ref.oracle(op, spec, a, b)
                k = f"mid/{midx:04d}"
                g[k + "/meta"] = np.array([0 if op == "trmm" else 1, spec.side, spec.uplo, spec.trans, spec.diag,
                                           n, m, 8, 1], dtype=np.int64)
                g[k + "/alpha"] = np.array(spec.alpha)
                g[k + "/a"] = a
                g[k + "/b"] = b
                g[k + "/rec"] = out
                g[k + "/oracle"] = orc
                g[k + "/events"] = np.array(events, dtype=np.int64).reshape(-1, 3)
                midx += 1
    g["mid/count"] = np.array(midx)

    # 4. Singularity reporting (acceptance_main.cpp:365-397): n = 64, t = 8.
    rows = []
    for s in (oracle.spec(0, 0, 0, 0), oracle.spec(0, 1, 1, 0), oracle.spec(1, 1, 0, 0)):
        for r in (5, 32, 49):
            a = ref.make_dominant(64, s.uplo, 7000 + r)
            a[r, r] = 0.0
            b = rhs(s, 64, 2, 7001, np.float64)
            st, _, _, row = ref.rec("trsm", s, a, b, 8)
            rows.append([s.side, s.uplo, s.trans, r, st, row])
    g["singular"] = np.array(rows, dtype=np.int64)

    # 5. Schema table (recursion.cpp:18-46) for all 32 (op, side, uplo, trans).
    sch = []
    for op in ("trmm", "trsm"):
        for side in (0, 1):
            for uplo in (0, 1):
                for trans in (0, 1, 2):
                    s = oracle.spec(side, uplo, trans, 0)
                    sch.append([0 if op == "trmm" else 1, side, uplo, trans, *ref.schema_for(op, s)])
    g["schema"] = np.array(sch)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {idx} small + {midx} mid cases)")


if __name__ == "__main__":
    main()
