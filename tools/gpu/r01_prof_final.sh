OUT=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:sgemm -c 1 -o $OUT/prof_sgemm_v3_nn python tools/prof_run.py sgemm 8192 16384 8192 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sgemm -c 1 -o $OUT/prof_sgemm_v3_k256 python tools/prof_run.py sgemm 256 16384 256 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/strsm_launches_v2.csv python tools/prof_run.py strsm 16384 16384 256 > /dev/null 2>&1
