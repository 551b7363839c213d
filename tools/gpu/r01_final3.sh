OUT=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > $OUT/final3_tests.log 2>&1; tail -2 $OUT/final3_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > $OUT/bench_v20.json 2> $OUT/bench_v20.err; tail -3 $OUT/bench_v20.err
for op in trmm trsm; do for e in f64 f32; do python tools/small_probe.py $op $e 256,512,1024,2048,4096,8192,16384; done; done > $OUT/small_v2.jsonl 2>&1
python tools/c4_sweep.py > $OUT/c4_v3.jsonl 2> /dev/null
timeout 1500 bash tools/c2_sweep.sh r01c > /dev/null 2>&1
ls $OUT | grep r01c
