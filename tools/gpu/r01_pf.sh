python tools/gemm_bench.py f32 16384 2>&1 | grep NN
python tools/small_probe.py trsm f32 4096,16384
