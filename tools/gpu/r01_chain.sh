timeout 1200 python -m pytest tests/test_gpu_leaf.py tests/test_gpu_parity.py tests/test_gpu_dropin.py -q --timeout 600 -x 2>&1 | tail -2
python tools/small_probe.py trsm f64 256,1024,2048,4096 | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('trsm', d['n'], round(d['pipe_us'],1), round(d['cublas_us'],1))"
python tools/small_probe.py trmm f64 256,1024,2048,4096,8192 | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('trmm', d['n'], round(d['pipe_us'],1), round(d['cublas_us'],1))"
timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-cublas --no-fp32 2>&1 | grep -E "profile|trsm:|trmm:" | cut -c1-200
