OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 > $OUT/conc_tests.log 2>&1
tail -5 $OUT/conc_tests.log
for c in 0 1; do for e in f64 f32; do RECTRI_CU_TRMM_CONC=$c python tools/small_probe.py trmm $e 256,512,1024,2048,4096,8192 | sed "s/^{/{\"conc\": $c, /"; done; done > $OUT/conc_probe.jsonl 2>&1
python -c "
import json
for l in open('$OUT/conc_probe.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['conc'],d['elem'],d['n'],round(d['pipe_us'],1),round(d['async_us'],1),round(d['cublas_us'],1))
"
