OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_leaf.py -x -q --timeout 600 > $OUT/leaf32_tests.log 2>&1; tail -3 $OUT/leaf32_tests.log
echo "new"; for m in 1024 4096 16384; do python tools/leaf_bench.py 256 $m f32; done
echo "old"; cp tools/gpu/old/librectri_old.so paper_2504_13821_b200/lib/librectri_cu.so
for m in 1024 4096 16384; do python tools/leaf_bench.py 256 $m f32; done
