#!/bin/bash
# Sweep fp64 DGEMM configurations over the level shapes (RECTRI_CU_GEMM64_CFG).
for c in "$@"; do
  echo "== cfg $c"
  RECTRI_CU_GEMM64_CFG=$c timeout 200 python tools/gemm_bench.py f64 2>&1 | grep -v probe
done
