OUT=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 600 > $OUT/final_tests.log 2>&1; tail -3 $OUT/final_tests.log
timeout 900 python bench.py > $OUT/final_bench.json 2> $OUT/final_bench.err; tail -c 600 $OUT/final_bench.json
for op in trmm trsm; do for e in f64 f32; do python tools/small_probe.py $op $e 256,512,1024,2048,4096,8192; done; done > $OUT/final_small.jsonl 2>&1
timeout 1500 bash tools/c2_sweep.sh r01b > $OUT/c2b.log 2>&1
python -c "
import json
for l in open('$OUT/final_small.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['op'],d['elem'],d['n'],round(d['pipe_us'],1),round(d['sync_us'],1),round(d['cublas_us'],1))
"
