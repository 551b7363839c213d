OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_leaf.py -x -q --timeout 600 -k widths 2>&1 | tail -2
for wm in 1 2; do echo "WM=$wm"; RECTRI_CU_LEAF_WM=$wm python tools/leaf_bench.py 256 16384 f64; RECTRI_CU_LEAF_WM=$wm timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-cublas --no-fp32 --no-trmm 2>&1 | grep -E "profile|GFLOP" | cut -c1-200; done
