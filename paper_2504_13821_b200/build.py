"""Builds the sm_100a library in-tree: paper_2504_13821_b200/lib/librectri_cu.so.

Every translation unit is compiled by nvcc for ``sm_100a`` only
(``-gencode arch=compute_100a,code=sm_100a -lineinfo``), in parallel, and
linked with a static CUDA runtime so the library is self-contained on the GPU
box.  The build is incremental (objects are rebuilt only when a source or a
header is newer).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "lib" / "obj"
LIB = PKG / "lib" / "librectri_cu.so"
SOURCES = ["gemm_f64.cu", *[f"gemm_f64_cfg{i}.cu" for i in range(2)], "gemm_f64_tma.cu",
           *[f"gemm_f64_tma_cfg{i}.cu" for i in range(4)], "gemm_f32.cu", "sgemm_tf32x3.cu", "leaf.cu", "leaf64.cu", "leaf64_v3.cu", "leaf64_v5.cu", "leaf32_v3.cu", "aux.cu",
           "driver.cu", "host_stage.cpp", "bench_host.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-Wall",
    f"-I{ROOT / 'include'}",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _headers() -> list[Path]:
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [ROOT / "include" / "rectri_cu.h"]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, obj: Path) -> None:
    cmd = [nvcc(), *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = _headers()
    jobs = []
    objs = []
    for name in SOURCES:
        src = CSRC / name
        obj = OBJ / (name.rsplit(".", 1)[0] + ".o")
        objs.append(obj)
        if _stale(obj, [src, *headers]):
            jobs.append((src, obj))
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            futs = [ex.submit(_compile, s, o) for s, o in jobs]
            for f in futs:
                f.result()
    if jobs or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {LIB}")
    return LIB


CMP_SRC = ROOT / "tools" / "cublas_cmp.cu"
CMP_LIB = ROOT / "tools" / "libcublas_cmp.so"


def build_cublas_cmp() -> Path:
    """The cuBLAS comparison shim used by bench.py (reported comparison only)."""
    if _stale(CMP_LIB, [CMP_SRC]):
        cmd = [nvcc(), *ARCH, "-O2", "-Xcompiler", "-fPIC", "-shared", str(CMP_SRC), "-o", str(CMP_LIB), "-lcublas"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"cublas_cmp failed to build:\n{r.stderr}")
    return CMP_LIB


EXAMPLE_SRC = ROOT / "tests" / "cpp" / "dropin_example.cpp"
EXAMPLE_BIN = ROOT / "tests" / "cpp" / "build" / "dropin_example"


def build_dropin_example() -> Path:
    """Compiles reference-style C++ user code against include/rectri/ (the
    drop-in headers) and links it to the in-tree library."""
    EXAMPLE_BIN.parent.mkdir(parents=True, exist_ok=True)
    deps = [EXAMPLE_SRC, LIB, ROOT / "include" / "rectri_b200.hpp", ROOT / "include" / "rectri_cu.h"]
    if _stale(EXAMPLE_BIN, deps):
        cmd = [os.environ.get("CXX", "g++"), "-std=c++17", "-O2", "-Wall", f"-I{ROOT / 'include'}",
               str(EXAMPLE_SRC), f"-L{LIB.parent}", "-lrectri_cu", "-Wl,-rpath,$ORIGIN/../../../paper_2504_13821_b200/lib",
               "-o", str(EXAMPLE_BIN)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"drop-in example failed to build:\n{r.stderr}")
    return EXAMPLE_BIN


BENCH_SRC = ROOT / "tests" / "cpp" / "dropin_bench.cpp"
BENCH_BIN = ROOT / "tests" / "cpp" / "build" / "dropin_bench"


def build_dropin_bench() -> Path:
    """The reference-caller-shaped e2e timer (std::vector MatrixBuffers
    through the C++ drop-in) that bench.py runs for its e2e_pageable line."""
    BENCH_BIN.parent.mkdir(parents=True, exist_ok=True)
    deps = [BENCH_SRC, LIB, ROOT / "include" / "rectri_b200.hpp", ROOT / "include" / "rectri_cu.h"]
    if _stale(BENCH_BIN, deps):
        cmd = [os.environ.get("CXX", "g++"), "-std=c++17", "-O2", "-Wall", "-pthread", f"-I{ROOT / 'include'}",
               str(BENCH_SRC), f"-L{LIB.parent}", "-lrectri_cu",
               "-Wl,-rpath,$ORIGIN/../../../paper_2504_13821_b200/lib", "-o", str(BENCH_BIN)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"drop-in bench failed to build:\n{r.stderr}")
    return BENCH_BIN


if __name__ == "__main__":
    build(verbose=True)
    build_dropin_example()
    build_dropin_bench()
    build_cublas_cmp()
    sys.exit(0)
