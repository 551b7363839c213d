OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:sgemm -c 1 -o $OUT/prof_sgemm_v2_nn python tools/prof_run.py sgemm 8192 16384 8192 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf32 -c 1 -o $OUT/prof_leaf32 python tools/prof_run.py leaf32 256 16384 > /dev/null 2>&1
ls -la $OUT/*.ncu-rep | tail -3
