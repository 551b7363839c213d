OUT=gpurun_out
for cfg in "2 2048" "2 1024" "2 512" "4 512" "4 256"; do
  set -- $cfg
  for op in trmm trsm; do
    RECTRI_CU_STREAMS=$1 RECTRI_CU_PANEL_MIN=$2 python tools/small_probe.py $op f64 256,512,1024,2048,4096 | sed "s/^{/{\"streams\": $1, \"panel_min\": $2, /"
  done
done > $OUT/panels.jsonl 2>&1
cat $OUT/panels.jsonl | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['streams'],d['panel_min'],d['op'],d['n'],round(d['pipe_us'],1),round(d['async_us'],1),round(d['cublas_us'],1))
"
