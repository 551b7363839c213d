#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box; never a bench number).
#   1. launch list of the bench command (per-launch device time)
#   2. DRAM bytes + time of every DGEMM launch of one C3 TRSM (roofline traffic)
#   3. full captures: level-1 DGEMM (NN 8192x16384x8192, TMA kernel), level-6
#      DGEMM (256x16384x256, cp.async kernel), TRSM leaf 256
set -x
OUT=gpurun_out
TAG=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $OUT/${TAG}_launches_bench.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-cublas --no-trmm --no-fp32 > $OUT/launches_bench.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:dgemm --csv --log-file $OUT/${TAG}_gemm_traffic.csv python tools/prof_run.py trsm 16384 16384 256 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm -c 1 -o $OUT/${TAG}_prof_gemm_l1 \
    python tools/prof_run.py gemm 8192 16384 8192 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm -c 1 -o $OUT/${TAG}_prof_gemm_l6 \
    python tools/prof_run.py gemm 256 16384 256 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf -c 1 -o $OUT/${TAG}_prof_leaf_trsm \
    python tools/prof_run.py leaf 256 16384 > /dev/null 2>&1
ls -la $OUT
