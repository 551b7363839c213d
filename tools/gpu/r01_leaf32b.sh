OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_leaf.py tests/test_gpu_parity.py -x -q --timeout 600 2>&1 | tail -2
for m in 1024 16384; do python tools/leaf_bench.py 256 $m f32; done
python tools/small_probe.py trsm f32 1024,4096,16384
python tools/small_probe.py trmm f32 1024,4096
ncu --set full --clock-control none --import-source on -k regex:leaf32 -c 1 -o $OUT/prof_leaf32_v2 python tools/prof_run.py leaf32 256 16384 > /dev/null 2>&1
