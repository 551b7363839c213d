set -x
OUT=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/strsm_launches.csv python tools/prof_run.py strsm 16384 16384 256 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sgemm -c 1 -o $OUT/prof_sgemm_nn_v2 python tools/prof_run.py sgemm 8192 16384 8192 > /dev/null 2>&1
timeout 1500 bash tools/c2_sweep.sh r01 > $OUT/c2.log 2>&1
tail -5 $OUT/c2.log; ls $OUT
