"""Benchmark harness with the reference's contract.

Mirrors include/rectri/bench.hpp:13-96 / src/bench.cpp:17-393 for the GPU
path: `run_sweep` (fresh inputs per size from the reference's own generator,
warmups, timed repetitions, median/min, a residual gate on every iteration),
`crossover_scan`, `ratio_report`, and the CSV I/O with the byte-exact
headers of bench.hpp:64-67.  Differences, all deliberate:

* backend is "cuda" (recorded as such in the `backend` column); "cublas"
  times cuBLAS ?trsm/?trmm on the same inputs through tools/libcublas_cmp.so
  so `ratio` can compare the two (Fig.-3-style reports);
* timing uses CUDA events around each call, inputs copied to the device
  outside the timed region like the reference copies B; the call is made
  with RECTRI_CU_ASYNC and completed (singularity reported) by `sync()`
  after the end event, so the events bracket enqueue + device time the same
  way they bracket the cuBLAS call of the "cublas" backend (a synchronous
  call would add the host's wake-up from the stream synchronize, ~14 us);
* the residual gate also rejects non-finite results (the reference's gate
  passes inf because std::max drops NaN).
"""
from __future__ import annotations

import csv
import ctypes
import io
import math
import statistics
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional

import numpy as np
import torch

from . import _lib
from .api import (ASYNC, Backend, Diag, MatrixBuffer, OpKind, Side, Threshold, Trans, TriangularSpec, Uplo, effective_op,
                  rec_trmm, rec_trsm, sync, to_string, validate, variant_string)
from .errors import ConfigError, IoError, JoinError, SingularityError, ValidationError

SWEEP_CSV_HEADER = "op,variant,n,m,threshold,backend,elem,median_time_s,min_time_s,gflops"
RATIO_CSV_HEADER = "op,variant,n,m,baseline_s,candidate_s,ratio_percent"


@dataclass
class BenchConfig:
    """bench.hpp:19-35"""
    op: OpKind = OpKind.Trsm
    spec: TriangularSpec = field(default_factory=TriangularSpec)
    sizes: List[int] = field(default_factory=list)
    m_mode: str = "fixed"  # "fixed" | "square"
    fixed_m: int = 256
    threshold: Threshold = field(default_factory=Threshold)
    backend: str = "cuda"  # "cuda" | "cublas"
    repetitions: int = 5
    warmup: int = 2
    out_path: str = ""
    elem: str = "f32"
    seed: int = 42
    inject_fault: bool = False


@dataclass
class BenchRecord:
    """bench.hpp:39-50"""
    op: str
    variant: str
    n: int
    m: int
    threshold: int
    backend: str
    elem: str
    median_time_s: float
    min_time_s: float
    gflops: float


@dataclass
class RatioRecord:
    """bench.hpp:54-62"""
    op: str
    variant: str
    n: int
    m: int
    baseline_s: float
    candidate_s: float
    ratio_percent: float


def _check_config(c: BenchConfig) -> None:
    """bench.cpp:225-235"""
    validate(c.spec)
    if c.repetitions < 1:
        raise ConfigError("repetitions must be >= 1")
    if c.warmup < 0:
        raise ConfigError("warmup must be >= 0")
    if not c.sizes:
        raise ConfigError("no sizes given")
    if any(n < 1 for n in c.sizes):
        raise ConfigError("sizes must be >= 1")
    if c.m_mode == "fixed" and c.fixed_m < 1:
        raise ConfigError("fixed m must be >= 1")
    if c.threshold.value < 1:
        raise ConfigError("threshold must be >= 1")
    if c.backend not in ("cuda", "cublas"):
        raise ConfigError(f"unknown backend '{c.backend}' (cuda|cublas)")
    if c.elem not in ("f32", "f64"):
        raise ConfigError(f"--elem must be f32 or f64, got '{c.elem}'")


def make_inputs(op: OpKind, spec: TriangularSpec, n: int, m: int, seed: int, elem: str):
    """src/bench.cpp:32-61 through the library's libstdc++ <random> (bit-identical)."""
    dt = np.float64 if elem == "f64" else np.float32
    brows, bcols = (n, m) if Side(spec.side) == Side.Left else (m, n)
    a = np.zeros((n, n), dtype=dt, order="F")
    b = np.zeros((brows, bcols), dtype=dt, order="F")
    fn = getattr(_lib.load(), f"rectri_cu_bench_inputs_{elem}")
    fn(a.ctypes.data, b.ctypes.data, n, brows, bcols, 1 if op == OpKind.Trsm else 0, int(spec.uplo), int(spec.diag),
       seed)
    return a, b


def _gate_columns(seed: int, cols: int) -> List[int]:
    out = (ctypes.c_int64 * 8)()
    k = _lib.load().rectri_cu_gate_columns(ctypes.c_uint64(seed & (2 ** 64 - 1)), cols, out)
    return [int(out[i]) for i in range(k)]


def validate_result(op: OpKind, spec: TriangularSpec, a: torch.Tensor, b_orig: torch.Tensor, result: torch.Tensor,
                    column_seed: int) -> None:
    """Residual gate of bench.cpp:100-165 on up to 8 sampled output columns,
    computed in float64 on the device, plus an explicit finiteness check.
    Tensors are (rows, cols) views of column-major storage."""
    n = a.shape[0]
    left = Side(spec.side) == Side.Left
    eff = effective_op(spec.trans)
    a64 = a.to(torch.float64)
    stored = torch.tril(a64, -1) if Uplo(spec.uplo) == Uplo.Lower else torch.triu(a64, 1)
    diag = torch.ones(n, dtype=torch.float64, device=a.device) if Diag(spec.diag) == Diag.Unit else a64.diagonal()
    M = stored + torch.diag(diag)
    if eff != Trans.NoTrans:
        M = M.t()
    cols = _gate_columns(column_seed, result.shape[1])
    res = result.to(torch.float64)
    bo = b_orig.to(torch.float64)
    alpha = spec.alpha
    eps = float(np.finfo(np.float32 if result.dtype == torch.float32 else np.float64).eps)
    a_norm = float((stored.abs().sum(1) + diag.abs()).max().item())
    if not bool(torch.isfinite(res).all().item()):
        raise ValidationError(f"residual gate failed: non-finite result for {to_string(OpKind(op))} "
                              f"{variant_string(spec)} n={n}")
    if op == OpKind.Trsm:
        scale = a_norm * float(res.abs().max().item()) + abs(alpha) * float(bo.abs().max().item())
        if left:
            lhs = M @ res[:, cols] - alpha * bo[:, cols]
        else:
            lhs = res @ M[:, cols] - alpha * bo[:, cols]
    else:
        scale = (1.0 + abs(alpha)) * a_norm * float(bo.abs().max().item())
        ref = M @ bo[:, cols] if left else bo @ M[:, cols]
        lhs = res[:, cols] - alpha * ref
    worst = float(lhs.abs().max().item()) if lhs.numel() else 0.0
    tol = 64.0 * max(n, 1) * eps * scale
    if not (worst <= tol) or not math.isfinite(worst):
        raise ValidationError(f"residual gate failed: |r| = {worst} > {tol} for {to_string(OpKind(op))} "
                              f"{variant_string(spec)} n={n}")


def _cublas_call(op, spec, n, m, A, B):
    """cuBLAS ?trsm / ?trmm (tools/libcublas_cmp.so) on the same device
    buffers, every side/uplo/trans/diag variant (ConjTrans == Trans on reals).
    trmm is out of place in cuBLAS: its result is copied back into B (outside
    the timed call).  Returns a callable giving the call's time in ms."""
    lib = ctypes.CDLL(str(Path(__file__).resolve().parents[1] / "tools" / "libcublas_cmp.so"))
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    dtype = 1 if A.dtype == torch.float64 else 0
    side, uplo = int(Side(spec.side)), int(Uplo(spec.uplo))
    trans = 0 if Trans(spec.trans) == Trans.NoTrans else 1
    diag = int(Diag(spec.diag))
    rows, cols = (n, m) if side == 0 else (m, n)
    if op == OpKind.Trsm:
        f = lib.cmp_trsm
        f.argtypes = [i32, i32, i32, i32, i32, vp, i64, vp, i64, i64, i32]
        f.restype = ctypes.c_double
        return lambda: f(dtype, side, uplo, trans, diag, A.data_ptr(), n, B.data_ptr(), rows, cols, 0)
    out = torch.empty_like(B)
    f = lib.cmp_trmm
    f.argtypes = [i32, i32, i32, i32, i32, vp, i64, vp, vp, i64, i64, i32]
    f.restype = ctypes.c_double

    def run():
        t = f(dtype, side, uplo, trans, diag, A.data_ptr(), n, B.data_ptr(), out.data_ptr(), rows, cols, 0)
        B.copy_(out)
        return t
    return run


def time_one(config: BenchConfig, n: int, m: int, seed: int) -> BenchRecord:
    """bench.cpp:174-223 on the GPU."""
    dt = torch.float64 if config.elem == "f64" else torch.float32
    for attempt in range(11):
        a, b = make_inputs(config.op, config.spec, n, m, seed + attempt, config.elem)
        A = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a)), device="cuda")
        B0 = torch.from_numpy(np.ascontiguousarray(b)).to("cuda")
        B = MatrixBuffer.from_tensor(B0, device="cuda")
        try:
            times = []
            for it in range(config.warmup + config.repetitions):
                B.data.copy_(B0.t().contiguous())
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                if config.backend == "cublas":
                    run = _cublas_call(config.op, config.spec, n, m, A.data, B.data)
                    ms = run()
                else:
                    fn = rec_trsm if config.op == OpKind.Trsm else rec_trmm
                    e0.record()
                    fn(config.spec, A.cview(), B.view(), config.threshold, Backend.cuda(flags=ASYNC))
                    e1.record()
                    sync()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                res = B.tensor()
                if config.inject_fault:  # bench.cpp:194-198
                    shift = float(res.abs().max().item()) + 1.0
                    res.add_(shift)
                validate_result(config.op, config.spec, A.tensor(), B0, res,
                                config.seed ^ (0x51ED270B * (it + 1)))
                if it >= config.warmup:
                    times.append(ms * 1e-3)
            med = statistics.median(times)
            return BenchRecord(to_string(OpKind(config.op)), variant_string(config.spec), n, m,
                               config.threshold.value, config.backend, config.elem, med, min(times),
                               float(n) * n * m / med / 1e9)
        except SingularityError:
            if attempt >= 10:
                raise
    raise AssertionError("unreachable")


def run_sweep(config: BenchConfig) -> List[BenchRecord]:
    """bench.cpp:317-331 (per-size seed config.seed + 7919 * (i + 1))."""
    _check_config(config)
    records = []
    for i, n in enumerate(config.sizes):
        m = config.fixed_m if config.m_mode == "fixed" else n
        records.append(time_one(config, n, m, config.seed + 7919 * (i + 1)))
    if config.out_path:
        write_sweep_csv(config.out_path, records)
    return records


def crossover_scan(config: BenchConfig, thresholds: List[int]) -> List[BenchRecord]:
    """bench.cpp:380-393"""
    if not thresholds:
        raise ConfigError("no thresholds given")
    out_path, config.out_path = config.out_path, ""
    allrec = []
    for t in thresholds:
        config.threshold = Threshold(t)
        allrec.extend(run_sweep(config))
    if out_path:
        write_sweep_csv(out_path, allrec)
    return allrec


def _fmt(v: float) -> str:
    return "%.9e" % v


def sweep_csv_text(records: List[BenchRecord]) -> str:
    lines = [SWEEP_CSV_HEADER]
    for r in records:
        lines.append(",".join([r.op, r.variant, str(r.n), str(r.m), str(r.threshold), r.backend, r.elem,
                               _fmt(r.median_time_s), _fmt(r.min_time_s), _fmt(r.gflops)]))
    return "\n".join(lines) + "\n"


def write_sweep_csv(path: str, records: List[BenchRecord]) -> None:
    try:
        Path(path).write_text(sweep_csv_text(records))
    except OSError as e:
        raise IoError(f"cannot write '{path}'") from e


def read_sweep_csv(path: str) -> List[BenchRecord]:
    """bench.cpp:263-296"""
    try:
        text = Path(path).read_text()
    except OSError as e:
        raise IoError(f"cannot read '{path}'") from e
    lines = text.splitlines()
    if not lines:
        raise ConfigError(f"'{path}' is empty")
    if lines[0] != SWEEP_CSV_HEADER:
        raise ConfigError(f"'{path}' has an unexpected header: {lines[0]}")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        if len(f) != 10:
            raise ConfigError(f"'{path}' has a malformed row: {line}")
        out.append(BenchRecord(f[0], f[1], int(f[2]), int(f[3]), int(f[4]), f[5], f[6], float(f[7]), float(f[8]),
                               float(f[9])))
    return out


def ratio_csv_text(records: List[RatioRecord]) -> str:
    lines = [RATIO_CSV_HEADER]
    for r in records:
        lines.append(",".join([r.op, r.variant, str(r.n), str(r.m), _fmt(r.baseline_s), _fmt(r.candidate_s),
                               _fmt(r.ratio_percent)]))
    return "\n".join(lines) + "\n"


def ratio_report(baseline_csv: str, candidate_csv: str, out_path: str = "") -> List[RatioRecord]:
    """bench.cpp:333-378: join on (op, variant, n, m); ratio = 100 * (b / c)."""
    base = read_sweep_csv(baseline_csv)
    cand = read_sweep_csv(candidate_csv)
    key = lambda r: (r.op, r.variant, r.n, r.m)  # noqa: E731
    ks = lambda k: f"{k[0]},{k[1]},{k[2]},{k[3]}"  # noqa: E731
    cand_t = {key(r): r.median_time_s for r in cand}
    seen = set()
    missing = ""
    for r in base:
        seen.add(key(r))
        if key(r) not in cand_t:
            missing += f" candidate lacks ({ks(key(r))})"
    for r in cand:
        if key(r) not in seen:
            missing += f" baseline lacks ({ks(key(r))})"
    if missing:
        raise JoinError("key mismatch:" + missing)
    out = [RatioRecord(r.op, r.variant, r.n, r.m, r.median_time_s, cand_t[key(r)],
                       100.0 * (r.median_time_s / cand_t[key(r)])) for r in base]
    if out_path:
        try:
            Path(out_path).write_text(ratio_csv_text(out))
        except OSError as e:
            raise IoError(f"cannot write '{out_path}'") from e
    return out
