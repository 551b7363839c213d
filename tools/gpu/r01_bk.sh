OUT=gpurun_out
RECTRI_CU_SGEMM_BK=32 timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q --timeout 600 -k sgemm 2>&1 | tail -2
for bk in 16 32; do echo "BK=$bk"; RECTRI_CU_SGEMM_BK=$bk python tools/gemm_bench.py f32 16384 2>&1 | head -12; done
for bk in 16 32; do RECTRI_CU_SGEMM_BK=$bk python tools/small_probe.py trsm f32 4096,16384; done
