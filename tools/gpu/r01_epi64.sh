timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q --timeout 600 2>&1 | tail -2
python tools/gemm_bench.py f64 16384 2>&1 | grep NN
python tools/small_probe.py trsm f64 1024,4096,16384
python tools/small_probe.py trmm f64 1024,2048,4096,8192
