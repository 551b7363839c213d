#!/bin/bash
# C2 (BASELINE.json configs[2]): TRMM Left/Upper/NoTrans square sweep
# n = m = 256..16384 for fp64 and fp32, our recursion against cuBLAS, plus the
# leaf-size (threshold) sweep 32..256 at n = m = 4096.  Run on the GPU box.
OUT=${OUT:-gpurun_out}
TAG=${1:-r01}
SIZES=256,512,1024,2048,4096,8192,16384
for elem in f64 f32; do
  for be in cuda cublas; do
    python tools/rectri_bench.py sweep --op trmm --side left --uplo upper --trans n --diag nonunit \
      --sizes $SIZES --m square --threshold 256 --backend $be --elem $elem --reps 5 --warmup 3 \
      --out $OUT/${TAG}_c2_trmm_${elem}_${be}.csv
  done
  python tools/rectri_bench.py crossover --op trmm --side left --uplo upper --trans n --diag nonunit \
    --sizes 4096 --m square --thresholds 32,64,128,256 --elem $elem --reps 5 --warmup 3 \
    --out $OUT/${TAG}_c2_leafsweep_${elem}.csv
done
