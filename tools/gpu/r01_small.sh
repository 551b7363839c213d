set -x
OUT=gpurun_out
for op in trmm trsm; do for e in f64 f32; do python tools/small_probe.py $op $e; done; done > $OUT/small_probe.jsonl 2> $OUT/small_probe.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/trmm1024_launches.csv python tools/prof_run.py trmm 1024 1024 256 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/trmm4096_launches.csv python tools/prof_run.py trmm 4096 4096 256 > /dev/null 2>&1
cat $OUT/small_probe.jsonl; tail -3 $OUT/small_probe.err
