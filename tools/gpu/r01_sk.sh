OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:sgemm -c 1 -o $OUT/prof_sgemm_k256 python tools/prof_run.py sgemm 256 16384 256 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm -c 1 -o $OUT/prof_dgemm_k256 python tools/prof_run.py gemm 256 16384 256 > /dev/null 2>&1
