#!/usr/bin/env python
"""Bench CLI with the reference's contract (tools/bench_main.cpp:124-184):

    rectri_bench.py sweep     --op trsm --sizes 1024,2048 [--side ..] [--m fixed:256|square] ...
    rectri_bench.py crossover --op trsm --sizes 4096 --thresholds 64,128,256 ...
    rectri_bench.py ratio     --baseline a.csv --candidate b.csv [--out r.csv]

Same options, CSV schema (bench.hpp:64-67) and exit codes: 0 ok, 1 residual
gate failure (ValidationError), 2 usage / any other error.  --backend is
cuda (this library) or cublas (reported comparison); seq/par are accepted
and mean cuda (the reference's CPU backends do not exist here).
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 2 like CLI11's ParseError path
        self.print_usage(sys.stderr)
        print(f"error: {message}", file=sys.stderr)
        sys.exit(2)


def _sweep_opts(p):
    p.add_argument("--op", required=True)
    p.add_argument("--side", default="left")
    p.add_argument("--uplo", default="lower")
    p.add_argument("--trans", default="n")
    p.add_argument("--diag", default="nonunit")
    p.add_argument("--alpha", type=float, default=1.0)
    p.add_argument("--sizes", required=True)
    p.add_argument("--m", dest="m_mode", default="fixed:256")
    p.add_argument("--threshold", type=int, default=256)
    p.add_argument("--backend", default="par")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--elem", default="f32")
    p.add_argument("--out", default="")
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--inject-fault", action="store_true")


def _sizes(text, what):
    from paper_2504_13821_b200.errors import ConfigError

    out = []
    for item in text.split(","):
        try:
            out.append(int(item))
        except ValueError:
            raise ConfigError(f"bad {what} entry '{item}'")
    return out


def _config(a):
    from paper_2504_13821_b200 import TriangularSpec, parse_diag, parse_op_kind, parse_side, parse_trans, parse_uplo
    from paper_2504_13821_b200.api import Threshold
    from paper_2504_13821_b200.errors import ConfigError
    from paper_2504_13821_b200.harness import BenchConfig

    c = BenchConfig()
    c.op = parse_op_kind(a.op)
    c.spec = TriangularSpec(parse_side(a.side), parse_uplo(a.uplo), parse_trans(a.trans), parse_diag(a.diag), a.alpha)
    c.sizes = _sizes(a.sizes, "--sizes")
    if a.m_mode == "square":
        c.m_mode = "square"
    elif a.m_mode.startswith("fixed:"):
        c.m_mode = "fixed"
        try:
            c.fixed_m = int(a.m_mode[6:])
        except ValueError:
            raise ConfigError(f"bad --m value '{a.m_mode}'")
    else:
        raise ConfigError(f"--m must be fixed:<width> or square, got '{a.m_mode}'")
    c.threshold = Threshold(a.threshold)
    if a.backend in ("seq", "par", "cuda"):
        c.backend = "cuda"
    elif a.backend == "cublas":
        c.backend = "cublas"
    else:
        raise ConfigError(f"--backend must be seq, par, cuda or cublas, got '{a.backend}'")
    c.repetitions, c.warmup, c.elem, c.out_path, c.seed = a.reps, a.warmup, a.elem, a.out, a.seed
    c.inject_fault = a.inject_fault
    return c


def main(argv=None):
    ap = _Parser(description="Runtime sweeps and runtime-ratio reports for recursive TRMM/TRSM (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    _sweep_opts(sub.add_parser("sweep"))
    cx = sub.add_parser("crossover")
    _sweep_opts(cx)
    cx.add_argument("--thresholds", required=True)
    ra = sub.add_parser("ratio")
    ra.add_argument("--baseline", required=True)
    ra.add_argument("--candidate", required=True)
    ra.add_argument("--out", default="")
    a = ap.parse_args(argv)
    try:
        from paper_2504_13821_b200 import harness as h
        from paper_2504_13821_b200.errors import ValidationError

        if a.cmd == "sweep":
            recs = h.run_sweep(_config(a))
            if not a.out:
                sys.stdout.write(h.sweep_csv_text(recs))
        elif a.cmd == "crossover":
            recs = h.crossover_scan(_config(a), _sizes(a.thresholds, "--thresholds"))
            if not a.out:
                sys.stdout.write(h.sweep_csv_text(recs))
        else:
            recs = h.ratio_report(a.baseline, a.candidate, a.out)
            if not a.out:
                sys.stdout.write(h.ratio_csv_text(recs))
    except Exception as e:  # noqa: BLE001 -- exit-code contract
        from paper_2504_13821_b200.errors import ValidationError

        if isinstance(e, ValidationError):
            print(f"validation failure: {e}", file=sys.stderr)
            return 1
        print(f"error: {e}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
