#!/usr/bin/env python
"""Benchmark of the B200 recursive TRSM/TRMM path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[2], "C3"): TRSM Left/Lower/NoTrans/
NonUnit fp64, n = m = 16384 per GPU, alpha = 1, diagonally dominant random A
(src/bench.cpp:32-61 conditioning); a TRMM Left/Upper/NoTrans fp64 line on
the same sizes rides along.  GFLOP/s = n^2 * m / t (src/bench.cpp:215-217).

Multi-GPU (torchrun, one process per GPU, NCCL): A is broadcast from rank 0
inside every timed step, B is column-sharded (m = 16384 columns per GPU,
weak scaling) with values keyed by the global column; each GPU solves its
columns with the single-GPU path.  Time = max over ranks.

value : inputs resident in HBM; per-step CUDA events on the launching stream
        (B restored from a pristine copy between steps, outside the events).
e2e   : the same call through the C-ABI with pinned HOST buffers (the library
        stages H2D, computes, copies B back), wall clock per call.
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

# Under torchrun, NCCL's communicator INIT lines go to a per-process file that
# setup_dist() echoes to stderr (evidence of the rank count).  NCCL reads its
# debug settings once, when the library initialises, so they are set before
# torch is imported.
# (An inherited NCCL_DEBUG=VERSION / WARN is raised to INFO for INIT only.)
if "WORLD_SIZE" in os.environ and os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
    os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT",
                      NCCL_DEBUG_FILE=f"/tmp/rectri_bench_nccl.{os.getpid()}.log")

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TRSM/TRMM GFLOP/s (m*n^2) fp64/fp32 at n=16384, % of B200 peak, 1/2/4/8 GPU"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock and throttle reasons
    DURING the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - NVML absent
            log(f"clock sampling unavailable: {e}")
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self._nv:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- utilities
def env_int(k, d):
    return int(os.environ.get(k, d))


def spawn_ranks(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: re-launch this script as N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1 and return
    the exit code; None when already a rank (or N == 1)."""
    if "WORLD_SIZE" in os.environ or args.gpus <= 1:
        return None
    import socket
    import subprocess

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    log("bench: spawning " + " ".join(cmd))
    return subprocess.call(cmd, env=dict(os.environ))


def setup_dist(args):
    """One process per GPU.  Under torchrun (WORLD_SIZE set) the process group
    is created even at world size 1, so the NCCL init, the in-step broadcast
    of A and the max-over-ranks all-reduce run on every launch of this kind;
    NCCL's INIT lines go to stderr as evidence of the communicator size."""
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if "WORLD_SIZE" in os.environ:
        if args.dry_gloo:
            dist.init_process_group("gloo")
        else:
            nccl_log = os.environ.get("NCCL_DEBUG_FILE")  # set at import (top of this file)
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
            if nccl_log and os.path.exists(nccl_log):
                for ln in Path(nccl_log).read_text().splitlines()[:60]:
                    log("nccl: " + ln.strip())
        log(f"bench: rank {dist.get_rank()} of {dist.get_world_size()} ({dist.get_backend()}), local rank {local}")
        if args.gpus != world:
            log(f"bench: note --gpus {args.gpus} but WORLD_SIZE {world}; the launcher's world size is used")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def allmax(x: float, world: int) -> float:
    if not dist.is_initialized():
        return x
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if dist.is_initialized():
        dist.barrier()
    torch.cuda.synchronize()


def bind_to_gpu_numa_node(index: int):
    """Pins this process to the CPUs NVML reports as local to the GPU (its
    NUMA node), so pinned host buffers are first-touched on the GPU's node.
    Returns the previous affinity (restored for the CPU baseline)."""
    prev = os.sched_getaffinity(0)
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = (os.cpu_count() + 63) // 64
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, words)
        cpus = {64 * w + b for w, m in enumerate(mask) for b in range(64) if (int(m) >> b) & 1}
        cpus &= prev
        if cpus and cpus != prev:
            os.sched_setaffinity(0, cpus)
            log(f"bench: bound to the {len(cpus)} CPUs local to GPU {index}")
    except Exception as e:  # pragma: no cover - NVML absent
        log(f"bench: no NUMA binding ({e})")
    return prev


# ------------------------------------------------------------ reference arm
def run_reference(args, world, rank):
    """`--impl reference`: the reference's own CPU path (oracle/_ref, compiled
    from the untouched sources) with Backend::par() on every host core, on a
    bounded column sample of the same workload."""
    if rank != 0:
        return
    import oracle
    from oracle import ref

    n = args.n
    m_s = args.ref_cols
    cores = os.cpu_count()
    a, b = make_host_inputs(n, m_s, args.op_headline)
    spec = oracle.spec(0, 0 if args.op_headline == "trsm" else 1, 0, 0, 1.0)
    if ref.available():
        kind = "reference"

        b0 = b.copy(order="F")

        def step():
            np.copyto(b, b0)  # restore B (outside the timer: see the loop below)
            t0 = time.perf_counter()
            st, _, _, _ = ref.rec(args.op_headline, spec, a, b, args.ref_threshold, width=-1)
            assert st == 0, ref.last_error()
            return time.perf_counter() - t0
    else:  # the C restatement (single thread, naive) on a tiny slice
        kind = "port"
        m_s = 8
        b = b[:, :m_s].copy(order="F")
        cores = 1

        def step():
            t0 = time.perf_counter()
            (oracle.oracle_trsm if args.op_headline == "trsm" else oracle.oracle_trmm)(spec, a, b)
            return time.perf_counter() - t0
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    t = statistics.median(times)
    value = n * n * m_s / t / 1e9
    sample = (f"{args.op_headline} left-{'lower' if args.op_headline == 'trsm' else 'upper'}-n-nonunit fp64 "
              f"n={n}, m={m_s} column slice of the m={args.m} workload (columns independent), "
              f"threshold {args.ref_threshold}, Backend::par() ({cores} threads), median of {args.steps}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_host_inputs(n, m, op):
    """fp64 column-major host inputs, uniform [-1, 1]; TRSM A lower-dominant
    (src/bench.cpp:40-51)."""
    rng = np.random.default_rng(42)
    a = np.asfortranarray(rng.uniform(-1.0, 1.0, (n, n)))
    if op == "trsm":
        d = np.zeros(n)
        for c0 in range(0, n, 2048):  # sum |A(r, c)| over c < r, blockwise
            blk = np.abs(a[:, c0:c0 + 2048])
            for j in range(blk.shape[1]):
                c = c0 + j
                d[c + 1:] += blk[c + 1:, j]
        a[np.arange(n), np.arange(n)] = d + 1.0
    b = np.asfortranarray(rng.uniform(-1.0, 1.0, (n, m)))
    return a, b


def workload_config(args, world):
    tag = ("C5 tall-RHS" if args.config == "c5" else "C3") + f" ({args.op_headline} headline)"
    return {
        "workload": (f"{tag}: TRSM Left/Lower/NoTrans/NonUnit + TRMM Left/Upper/NoTrans "
                     f"fp64, n={args.n}, m={args.m} per GPU (m={args.m * world} total), alpha=1, "
                     "diagonally dominant random A"),
        "n": args.n, "m_per_gpu": args.m, "m_total": args.m * world, "threshold": args.threshold,
        "parallelism": f"rhs-shard x{world}" if world > 1 else "single GPU",
        "l2": "inputs (A 2 GiB + B 2 GiB per GPU) far larger than the 126 MB L2",
        "timing": "per-step CUDA events on the launching stream; B restored between steps outside the events",
    }


def run_dry(args, world, rank):
    """`--dry-gloo`: the multi-rank plumbing of the bench without a GPU --
    the spawn, the rendezvous, the in-step broadcast of A from rank 0 and the
    max-over-ranks of the step time, on gloo.  Prints a JSON line with no
    value (nothing is computed)."""
    n = 64
    A = torch.arange(n * n, dtype=torch.float64).reshape(n, n) if rank == 0 else torch.zeros(n, n, dtype=torch.float64)
    steps = []
    for _ in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if dist.is_initialized():
            dist.broadcast(A, src=0)
        steps.append(time.perf_counter() - t0)
    ok = bool(torch.equal(A, torch.arange(n * n, dtype=torch.float64).reshape(n, n)))
    oks = allmax(0.0 if ok else 1.0, world)
    ms = allmax(sum(steps[args.warmup:]) * 1e3, world)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms / max(args.steps, 1), "dry_run": True,
                          "backend": dist.get_backend() if dist.is_initialized() else None,
                          "broadcast_ok": oks == 0.0, "config": workload_config(args, world)}), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def run_c5(args, world, rank, local, rc, stream):
    """North-star strong-scaling line (BASELINE configs[4], "C5"): TRSM
    L/L/N/NU fp64, n = 8192, m = 524288 right-hand sides in TOTAL, column-
    sharded (m / N per GPU, values keyed by the global column), A broadcast
    from rank 0 inside every timed step; time = max over ranks of the summed
    per-step CUDA events.  B is regenerated between steps outside the events."""
    from paper_2504_13821_b200 import ASYNC, Backend, Diag, MatrixBuffer, Side, Threshold, Trans, TriangularSpec, Uplo

    n, m_total = 8192, 524288
    m = m_total // world
    dev = torch.device("cuda", local)
    A = MatrixBuffer(n, n, torch.float64, dev)
    if rank == 0:
        rc.fill_uniform(A.view(), 0, n, seed=11)
        rc.make_dominant(A.view(), Uplo.Lower)
    B = MatrixBuffer(n, m, torch.float64, dev)
    spec = TriangularSpec(Side.Left, Uplo.Lower, Trans.NoTrans, Diag.NonUnit, 1.0)
    be = Backend.cuda(device=local, stream=stream, flags=ASYNC)
    torch.cuda.synchronize()

    def step():
        if dist.is_initialized():
            dist.broadcast(A.data, src=0)
        rc.rec_trsm(spec, A.cview(), B.view(), Threshold(args.threshold), be)

    for _ in range(1):  # graph capture
        rc.fill_uniform(B.view(), col0=rank * m, global_rows=n, seed=12)
        step()
    rc.sync(stream)
    barrier(world)
    evs = []
    gc.collect()
    gc.disable()
    with ClockSampler(local) as clk:
        for _ in range(args.c5_steps):
            rc.fill_uniform(B.view(), col0=rank * m, global_rows=n, seed=12, backend=be)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            evs.append((e0, e1))
        rc.sync(stream)
        torch.cuda.synchronize()
    gc.enable()
    barrier(world)
    ms = allmax(sum(a.elapsed_time(b) for a, b in evs), world) / args.c5_steps
    # residual on 8 sampled columns of this rank's shard (pristine values regenerated by global column)
    cols = [k * (m // 8) for k in range(8)]
    Bs = MatrixBuffer(n, 8, torch.float64, dev)
    for j, c in enumerate(cols):
        rc.fill_uniform(Bs.view().subview(0, j, n, 1), col0=rank * m + c, global_rows=n, seed=12)
    torch.cuda.synchronize()
    X = B.data[cols].t()
    L = torch.tril(A.data.t())
    Bsd = Bs.data.t()
    resid = (L @ X - Bsd).abs().max().item()
    eta = resid / (L.abs().sum(1).max().item() * max(X.abs().max().item(), Bsd.abs().max().item(), 1.0)
                   * n * np.finfo(float).eps)
    finite = bool(torch.isfinite(X).all().item())
    eta = float(allmax(float(eta) if finite else float("inf"), world))
    del L, X, A, B, Bs
    torch.cuda.empty_cache()
    value = float(n) * n * m_total / (ms * 1e-3) / 1e9
    log(f"c5: {value:.1f} GFLOP/s over {world} GPU(s), {ms:.2f} ms/step, eta {eta:.3e}")
    return {"value": value, "unit": "GFLOP/s", "ms_per_step": ms, "steps": args.c5_steps, "n_gpus": world,
            "scaling": "strong", "clocks": clk.summary(),
            "workload": f"C5: TRSM Left/Lower/NoTrans/NonUnit fp64 n={n}, m={m_total} total, {m} per GPU, "
                        "A broadcast from rank 0 inside every step",
            "residual": {"eta": eta, "finite": eta != float("inf"), "bound": 32, "columns_per_rank": 8}}


# ----------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=["c3", "c5"], default="c3",
                    help="c3: n=m=16384 per GPU (weak scaling); c5: tall RHS n=8192, m=524288 total (strong)")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--m", type=int, default=None, help="right-hand sides per GPU")
    ap.add_argument("--no-fp32", action="store_true")
    ap.add_argument("--threshold", type=int, default=256)
    ap.add_argument("--op-headline", choices=["trsm", "trmm"], default="trsm")
    ap.add_argument("--ref-cols", type=int, default=1024,
                    help="column slice of the reference arm and of cpu_baseline (the same slice)")
    ap.add_argument("--ref-threshold", type=int, default=256)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--no-trmm", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 strong-scaling line")
    ap.add_argument("--c5-steps", type=int, default=3)
    ap.add_argument("--dry-gloo", action="store_true",
                    help="CPU-only plumbing check: spawn, gloo rendezvous, broadcast of A, max over ranks; no compute")
    args = ap.parse_args()

    rc_spawn = spawn_ranks(args)
    if rc_spawn is not None:
        sys.exit(rc_spawn)
    world, rank, local = setup_dist(args)
    if args.config == "c5":
        args.n = args.n or 8192
        args.m = args.m or 524288 // world
        args.scaling = "strong"
    else:
        args.n = args.n or 16384
        args.m = args.m or 16384
        args.scaling = "weak"
    if args.dry_gloo:
        run_dry(args, world, rank)
        return
    if args.impl == "reference":
        run_reference(args, world, rank)
        if dist.is_initialized():
            dist.destroy_process_group()
        return
    cpu_affinity = bind_to_gpu_numa_node(local)

    import paper_2504_13821_b200 as rc
    from paper_2504_13821_b200 import (ASYNC, TF32X3, Backend, Diag, MatrixBuffer, Side, Threshold, Trans,
                                       TriangularSpec, Uplo)

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    n, m = args.n, args.m
    f64 = torch.float64

    # Inputs resident in HBM. A: rank 0 generates, broadcast inside each step.
    A = MatrixBuffer(n, n, f64, dev)
    if rank == 0:
        rc.fill_uniform(A.view(), 0, n, seed=1)
    B = MatrixBuffer(n, m, f64, dev)
    B0 = MatrixBuffer(n, m, f64, dev)
    rc.fill_uniform(B0.view(), col0=rank * m, global_rows=n, seed=2)
    # TRSM reads the lower triangle (diag made dominant); TRMM the upper one.
    A_trsm = A
    if rank == 0:
        rc.make_dominant(A_trsm.view(), Uplo.Lower)
    torch.cuda.synchronize()
    if dist.is_initialized():
        dist.broadcast(A.data, src=0)
    be = Backend.cuda(device=local, stream=stream, flags=ASYNC)

    specs = {
        "trsm": TriangularSpec(Side.Left, Uplo.Lower, Trans.NoTrans, Diag.NonUnit, 1.0),
        "trmm": TriangularSpec(Side.Left, Uplo.Upper, Trans.NoTrans, Diag.NonUnit, 1.0),
    }
    flops_per_gpu = float(n) * n * m

    def one(op, Abuf=None, Bbuf=None, backend=None):
        Abuf = Abuf if Abuf is not None else A
        Bbuf = Bbuf if Bbuf is not None else B
        fn = rc.rec_trsm if op == "trsm" else rc.rec_trmm
        if dist.is_initialized():
            dist.broadcast(Abuf.data, src=0)
        fn(specs[op], Abuf.cview(), Bbuf.view(), Threshold(args.threshold), backend or be)

    def timed(op, Abuf=None, Bbuf=None, B0buf=None, backend=None):
        Bbuf = Bbuf if Bbuf is not None else B
        B0buf = B0buf if B0buf is not None else B0
        for _ in range(args.warmup):
            Bbuf.data.copy_(B0buf.data)
            one(op, Abuf, Bbuf, backend)
        rc.sync(stream)
        barrier(world)
        launches0 = rc.launch_count()
        evs = []
        gc.collect()
        gc.disable()  # no cycle collection between a step's events (see the e2e loop)
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                Bbuf.data.copy_(B0buf.data)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                one(op, Abuf, Bbuf, backend)
                e1.record(stream)
                evs.append((e0, e1))
            rc.sync(stream)
            torch.cuda.synchronize()
        gc.enable()
        launches = rc.launch_count() - launches0
        barrier(world)
        local_ms = sum(a.elapsed_time(b) for a, b in evs)
        ms = allmax(local_ms, world)
        value = flops_per_gpu * world * args.steps / (ms * 1e-3) / 1e9
        return value, ms / args.steps, launches, clk.summary()

    peak64 = rc.probe_peak("f64")
    value, ms_step, launches, clocks = timed("trsm")
    log(f"trsm: {value:.1f} GFLOP/s, {ms_step:.2f} ms/step, clocks {clocks}")

    # Residual gate on 8 sampled columns (finite check first).
    B.data.copy_(B0.data)
    one("trsm")
    rc.sync(stream)
    cols = torch.arange(0, m, max(1, m // 8), device=dev)[:8]
    X = B.data[cols].t()                          # n x 8
    Bs = B0.data[cols].t()
    L = torch.tril(A.data.t())                    # masked lower triangle incl. diag
    resid = (L @ X - Bs).abs().max().item()
    anorm = L.abs().sum(1).max().item()
    xmax = X.abs().max().item()
    eta = resid / (anorm * max(xmax, Bs.abs().max().item(), 1.0) * n * np.finfo(float).eps)
    finite = bool(torch.isfinite(X).all().item())
    del L
    torch.cuda.empty_cache()
    log(f"residual eta {eta:.3e} finite {finite}")

    # Per-kernel-class breakdown with CUDA events around every launch (extra
    # untimed calls, direct launches): the roofline's achieved figure.  Right
    # after the timed TRSM steps (before the power-hungry fp32 / 3xTF32 runs
    # can leave the GPU power-capped), best of three passes.
    prof = None
    for _ in range(3):
        B.data.copy_(B0.data)
        torch.cuda.synchronize()
        rc.profile_enable(True)
        one("trsm")
        rc.sync(stream)
        rc.profile_enable(False)
        pr = rc.profile_read()
        if prof is None or pr["gemm"]["ms"] < prof["gemm"]["ms"]:
            prof = pr
    g = prof["gemm"]
    gemm_tflops = g["flops"] / (g["ms"] * 1e-3) / 1e12 if g["ms"] else 0.0
    step_ms_prof = sum(v["ms"] for v in prof.values())
    log(f"profile: {json.dumps(prof)}")
    traffic = None
    tf = ROOT / "profiles" / "ncu_gemm_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {
        "bound": "tensor", "achieved": gemm_tflops, "peak": peak64, "unit": "TFLOP/s",
        "frac": gemm_tflops / peak64 if peak64 > 0 else None, "traffic": traffic,
        "kernel": "dgemm_tma_kernel (off-diagonal GEMM updates, TMA-fed DMMA.8x8x4)",
        "peak_source": "live DMMA.8x8x4 issue-rate probe on this GPU (rectri_cu_probe_peak; MEASURED_PEAKS.json "
                       "has no fp64 figure); cf. profiles/r01_microbench_peaks.jsonl",
        "per_launch_flops": g["flops"] / max(g["launches"], 1), "launches": g["launches"],
        "share_of_step": g["ms"] / step_ms_prof if step_ms_prof else None,
        "breakdown_ms": {k: v["ms"] for k, v in prof.items()},
        "achieved_source": "per-launch CUDA events on the launching stream in untimed steps with direct "
                           "launches on one stream (the profiling mode of the library), best of 3, right after "
                           "the timed TRSM steps",
    }
    # The same GEMM flops inside the TIMED configuration (graph, 2 right-hand-side
    # streams): the step time minus the non-GEMM kernels' profiled time.
    other_ms = step_ms_prof - g["ms"]
    roofline["achieved_in_step"] = g["flops"] / max((ms_step - other_ms) * 1e-3, 1e-9) / 1e12
    roofline["frac_in_step"] = roofline["achieved_in_step"] / peak64 if peak64 > 0 else None
    # The leaf (trsm_base per diagonal block): achieved HBM bandwidth on its
    # algorithmic bytes (nb(nb+1)/2 + 2 nb r) * 8 next to the
    # measured copy bandwidth -- it is latency / tensor bound, not HBM bound.
    lf = prof.get("leaf", {})
    if lf.get("launches"):
        nleaf = lf["launches"]
        nb = n // nleaf if n % nleaf == 0 else args.threshold
        leaf_bytes = (nb * (nb + 1) // 2 + 2 * nb * m) * 8 * nleaf
        hbm = 6450.0
        try:
            hbm = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", hbm))
        except Exception:
            pass
        roofline["leaf"] = {
            "kernel": "leaf3_kernel (fp64 trsm_base, packed-block ring, DMMA)", "launches": nleaf,
            "ms": lf["ms"], "algorithmic_bytes": leaf_bytes,
            "achieved_gbs": leaf_bytes / (lf["ms"] * 1e-3) / 1e9 if lf["ms"] else None,
            "hbm_peak_gbs": hbm, "achieved_tflops": lf["flops"] / (lf["ms"] * 1e-3) / 1e12 if lf["ms"] else None,
        }


    trmm = None
    if not args.no_trmm:
        tv, tms, tl, tclk = timed("trmm")
        trmm = {"value": tv, "unit": "GFLOP/s", "ms_per_step": tms, "pct_of_peak": tv / 1e3 / peak64 * 100,
                "gpu_launches": tl, "clocks": tclk,
                "workload": f"TRMM Left/Upper/NoTrans/NonUnit fp64 n={n}, m={m} per GPU"}
        log(f"trmm: {tv:.1f} GFLOP/s, {tms:.2f} ms/step")

    # fp32 line: TRSM L/L/N/NU on the same inputs rounded to fp32.
    fp32 = None
    if not args.no_fp32:
        A32 = MatrixBuffer(n, n, torch.float32, dev)
        A32.data.copy_(A.data)
        B32_0 = MatrixBuffer(n, m, torch.float32, dev)
        B32_0.data.copy_(B0.data)
        B32 = MatrixBuffer(n, m, torch.float32, dev)
        v32, ms32, l32, clk32 = timed("trsm", A32, B32, B32_0)
        fp32 = {"value": v32, "unit": "GFLOP/s", "ms_per_step": ms32, "gpu_launches": l32, "clocks": clk32,
                "pct_of_ffma2_peak": v32 / 1e3 / rc.probe_peak("f32") * 100,
                "workload": f"TRSM Left/Lower/NoTrans/NonUnit fp32 n={n}, m={m} per GPU (FFMA path)"}
        if not args.no_cublas and world == 1:
            try:
                fp32["cublas_strsm_LLN"] = cublas_strsm(A32, B32_0, n, m)
            except Exception as e:  # pragma: no cover
                fp32["cublas_strsm_LLN"] = {"error": str(e)}
        log(f"fp32 trsm: {v32:.1f} GFLOP/s, {ms32:.2f} ms/step")
        # Opt-in 3xTF32 variant on tcgen05 (csrc/sgemm_tf32x3.cu), reported
        # separately with its own residual on 8 sampled columns.
        be_tf = Backend.cuda(device=local, stream=stream, flags=ASYNC | TF32X3)
        vt, mst, lt, clkt = timed("trsm", A32, B32, B32_0, be_tf)
        B32.data.copy_(B32_0.data)
        one("trsm", A32, B32, be_tf)
        rc.sync(stream)
        Xt = B32.data[cols].t().double()
        L32 = torch.tril(A32.data.t().double())
        Bt = B32_0.data[cols].t().double()
        res_t = (L32 @ Xt - Bt).abs().max().item()
        eta_t = res_t / (L32.abs().sum(1).max().item() * max(Xt.abs().max().item(), Bt.abs().max().item(), 1.0)
                         * n * float(np.finfo(np.float32).eps))
        del L32, Xt, Bt
        fp32["tf32x3"] = {"value": vt, "unit": "GFLOP/s", "ms_per_step": mst, "gpu_launches": lt, "clocks": clkt,
                          "residual_eta_fp32": eta_t, "tolerance": "eta <= 32 (the fp32 criterion of the FFMA path)",
                          "workload": "same TRSM, fp32 GEMM updates as 3xTF32 (hi/lo split, 3 tcgen05 kind::tf32 "
                                      "MMAs per k-step, fp32 accumulation in TMEM); opt-in RECTRI_CU_TF32X3"}
        log(f"fp32 trsm 3xTF32: {vt:.1f} GFLOP/s, {mst:.2f} ms/step, eta {eta_t:.3e}")
        del A32, B32_0, B32
        torch.cuda.empty_cache()

    # End to end through the C-ABI with pinned host buffers.
    e2e = None
    if not args.no_e2e:
        me = min(m, 65536)  # pinned host budget: C5 uses a 65536-column slice per GPU
        Ah = torch.empty((n, n), dtype=f64, pin_memory=True)
        Ah.copy_(A.data)
        Bh0 = torch.empty((me, n), dtype=f64, pin_memory=True)
        Bh0.copy_(B0.data[:me])
        Bh = torch.empty((me, n), dtype=f64, pin_memory=True)
        Av = rc.MatrixView(Ah, n, n).as_const()
        Bv = rc.MatrixView(Bh, n, me)
        be_sync = Backend.cuda(device=local, stream=stream)
        walls = []
        # Collect now and keep the collector out of the timed steps: a cycle
        # collection that frees an earlier phase's pinned buffers (cudaFreeHost
        # unpins GBs) inside a step cost up to 200 ms on one run.
        gc.collect()
        gc.disable()
        for i in range(args.warmup + args.steps):
            Bh.copy_(Bh0)
            barrier(world)
            t0 = time.perf_counter()
            rc.rec_trsm(specs["trsm"], Av, Bv, Threshold(args.threshold), be_sync)
            w = time.perf_counter() - t0
            if i >= args.warmup:
                walls.append(w)
        gc.enable()
        wall = allmax(sum(walls), world)
        e2e = {"value": float(n) * n * me * world * args.steps / wall / 1e9, "unit": "GFLOP/s",
               # A: the recursion's leaf diagonal blocks (full squares) + off-diagonal GEMM blocks,
               # (n^2 + n t)/2 elements (driver.cu run_host_streamed); B: every element once
               "h2d_bytes_per_step": ((n * n + n * args.threshold) // 2 + n * me) * 8 * world,
               "d2h_bytes_per_step": n * me * 8 * world,
               "rhs_per_gpu": me,
               "ms_per_step": wall / args.steps * 1e3,
               "step_ms": [round(w * 1e3, 2) for w in walls],
               "median_step_ms": round(sorted(walls)[len(walls) // 2] * 1e3, 2),
               "path": "rectri_cu_rec_trsm_f64 with pinned host views: A blocks and B row chunks copied in "
                       "first-use order, each kernel gated on its own inputs, chunks copied back after their "
                       "last writer (driver.cu run_host_streamed); wall clock"}
        log(f"e2e: {e2e['value']:.1f} GFLOP/s")
        del Ah, Bh, Bh0

    # End to end through the C++ drop-in with reference-caller memory
    # (tests/cpp/dropin_bench.cpp): MatrixBuffers (the drop-in keeps their
    # bytes page-locked) and plain std::vector storage behind MatrixViews
    # (pageable, staged through bounce buffers).
    e2e_pageable = e2e_dropin = None
    if not args.no_e2e and world == 1:
        e2e_dropin = run_dropin(args, n, min(m, 65536), "buffer")
        e2e_pageable = run_dropin(args, n, min(m, 65536), "pageable")

    # cuBLAS reported comparison (same inputs, device-resident).
    cublas = None
    if not args.no_cublas and world == 1:
        try:
            cublas = cublas_compare(A, B0, n, m, args)
        except Exception as e:  # pragma: no cover
            cublas = {"error": str(e)}
    # Second roofline denominator: cuBLAS DGEMM (16384^3) measured in this run.
    dg = (cublas or {}).get("dgemm", {}).get("tflops_2n3")
    if dg:
        roofline["peak_cublas_dgemm"] = dg
        roofline["frac_vs_cublas_dgemm"] = roofline["achieved"] / dg
        roofline["achieved_in_step_frac_vs_cublas_dgemm"] = roofline["achieved_in_step"] / dg

    c5 = None
    if not args.no_c5 and args.config != "c5":
        c5 = run_c5(args, world, rank, local, rc, stream)

    cpu = None
    if not args.no_cpu_baseline and world == 1 and rank == 0:
        os.sched_setaffinity(0, cpu_affinity)  # every host core, like the reference arm
        cpu = cpu_baseline(args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-generated uniform[-1,1), dominant A)",
            "config": workload_config(args, world),
            "pct_of_peak": value / 1e3 / (peak64 * world) * 100,
            "residual": {"eta": eta, "finite": finite, "bound": 32,
                         "definition": "||tril(A) X - B||_max / (||A||_inf max(|X|,|B|,1) n eps), 8 sampled columns"},
            "trmm": trmm, "fp32": fp32, "c5_strong": c5, "e2e": e2e, "e2e_dropin": e2e_dropin,
            "e2e_pageable": e2e_pageable,
            "roofline": roofline, "cpu_baseline": cpu,
            "cublas": cublas,
            "clocks": clocks, "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def run_dropin(args, n, m, storage):
    """tests/cpp/dropin_bench: rectri::rec_trsm<double> exactly as reference
    code calls it, on rectri::MatrixBuffers (storage "buffer": the drop-in
    allocates them page-locked, the library streams them directly) or on
    plain std::vector storage behind MatrixViews ("pageable": staged through
    pinned bounce buffers by host threads overlapping the transfers,
    csrc/host_stage.h); wall clock per call with steady_clock."""
    import subprocess

    exe = ROOT / "tests" / "cpp" / "build" / "dropin_bench"
    if not exe.exists():
        return {"error": "tests/cpp/build/dropin_bench not built"}
    steps = max(1, min(args.steps, 5))
    try:
        r = subprocess.run([str(exe), str(n), str(m), str(steps), "2", storage], capture_output=True, text=True,
                           timeout=900)
        d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}
    how = ("rectri::MatrixBuffers (page-locked by the drop-in's allocator; streamed directly)"
           if storage == "buffer" else
           "std::vector storage behind MatrixViews (pageable); pinned bounce staging by host threads "
           "overlapping the streamed transfers")
    d.update({"value": float(n) * n * m / (d["ms_per_step"] * 1e-3) / 1e9, "unit": "GFLOP/s",
              "h2d_bytes_per_step": ((n * n + n * args.threshold) // 2 + n * m) * 8,
              "d2h_bytes_per_step": n * m * 8, "rc": r.returncode,
              "path": f"C++ drop-in rectri::rec_trsm<double> on {how}; wall clock per call"})
    log(f"e2e {storage}: {d['value']:.1f} GFLOP/s ({d['ms_per_step']:.1f} ms/step, eta {d['eta']:.2e})")
    return d


def cublas_compare(A, B0, n, m, args):
    """cuBLAS dtrsm / dtrmm / dgemm on the SAME device inputs (reported
    comparison only; tools/libcublas_cmp.so, best of 2 with CUDA events).
    cuBLAS trmm is out of place (C = A B); flops counted like ours (n^2 m)."""
    import ctypes

    lib = ctypes.CDLL(str(ROOT / "tools" / "libcublas_cmp.so"))
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    lib.cmp_dtrsm_lln.argtypes = [vp, i64, vp, i64, ctypes.c_int]
    lib.cmp_dtrmm_lun.argtypes = [vp, i64, vp, vp, i64, ctypes.c_int]
    lib.cmp_dgemm.argtypes = [vp, vp, vp, i64, ctypes.c_int]
    for f in (lib.cmp_dtrsm_lln, lib.cmp_dtrmm_lun, lib.cmp_dgemm):
        f.restype = ctypes.c_double
    work = B0.data.clone()
    out = torch.empty_like(work)
    torch.cuda.synchronize()
    # trsm solves in place: each timed call re-solves the previous solution,
    # which changes values but not the work.
    t_trsm = lib.cmp_dtrsm_lln(A.data.data_ptr(), n, work.data_ptr(), m, 2)
    work.copy_(B0.data)
    t_trmm = lib.cmp_dtrmm_lun(A.data.data_ptr(), n, work.data_ptr(), out.data_ptr(), m, 2)
    res = {"dtrsm_LLN": {"ms": t_trsm, "gflops": float(n) * n * m / t_trsm / 1e6},
           "dtrmm_LUN": {"ms": t_trmm, "gflops": float(n) * n * m / t_trmm / 1e6, "note": "out of place"}}
    if m == n:
        t_gemm = lib.cmp_dgemm(A.data.data_ptr(), work.data_ptr(), out.data_ptr(), n, 2)
        res["dgemm"] = {"ms": t_gemm, "tflops_2n3": 2.0 * n ** 3 / t_gemm / 1e9}
    del work, out
    torch.cuda.empty_cache()
    return res


def cublas_strsm(A32, B32_0, n, m):
    """cuBLAS strsm (Left/Lower/N/NonUnit) on the same fp32 device inputs."""
    import ctypes

    lib = ctypes.CDLL(str(ROOT / "tools" / "libcublas_cmp.so"))
    lib.cmp_strsm_lln.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
    lib.cmp_strsm_lln.restype = ctypes.c_double
    work = B32_0.data.clone()
    t = lib.cmp_strsm_lln(A32.data.data_ptr(), n, work.data_ptr(), m, 2)
    del work
    return {"ms": t, "gflops": float(n) * n * m / t / 1e6}


def cpu_baseline(args):
    """The reference's CPU path (oracle/_ref) on the host cores, bounded
    sample: the same column slice, generator, threshold and statistic (median
    of repeated calls) as the `--impl reference` arm."""
    import oracle
    from oracle import ref

    n, m_s = args.n, args.ref_cols
    a, b = make_host_inputs(n, m_s, "trsm")
    spec = oracle.spec(0, 0, 0, 0, 1.0)
    if ref.available():
        reps = 3
        ref.rec("trsm", spec, a, b[:, :16].copy(order="F"), args.ref_threshold, width=-1)  # warm
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            st, _, _, _ = ref.rec("trsm", spec, a, b, args.ref_threshold, width=-1)
            ts.append(time.perf_counter() - t0)
            assert st == 0
        t = statistics.median(ts)
        return {"value": n * n * m_s / t / 1e9, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": f"rec_trsm left-lower-n-nonunit fp64 n={n}, m={m_s} column slice (the reference arm's), "
                          f"threshold {args.ref_threshold}, Backend::par() ({os.cpu_count()} threads), "
                          f"median of {reps} calls ({t:.2f} s each)"}
    m_s = 4
    t0 = time.perf_counter()
    oracle.oracle_trsm(spec, a, b[:, :m_s].copy(order="F"))
    t = time.perf_counter() - t0
    return {"value": n * n * m_s / t / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": f"C oracle restatement, n={n}, m={m_s}"}


if __name__ == "__main__":
    main()
