set -x
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_leaf.py -x -q --timeout 600 > $OUT/v2_tests.log 2>&1
tail -5 $OUT/v2_tests.log
for v in 1 2; do RECTRI_CU_SGEMM=$v python tools/gemm_bench.py f32 16384 > $OUT/sgemm_v$v.log 2>&1; done
for nc in 32 16 8; do RECTRI_CU_LEAF_NC=$nc python tools/small_probe.py trmm f64 256,1024,2048,4096,8192; done > $OUT/leafnc.jsonl 2>&1
python tools/small_probe.py trsm f64 256,1024,2048,4096,8192 >> $OUT/leafnc.jsonl 2>&1
RECTRI_CU_SGEMM=1 python tools/small_probe.py trsm f32 4096,8192,16384 > $OUT/strsm_v.jsonl 2>&1
RECTRI_CU_SGEMM=2 python tools/small_probe.py trsm f32 4096,8192,16384 >> $OUT/strsm_v.jsonl 2>&1
paste $OUT/sgemm_v1.log $OUT/sgemm_v2.log | cut -c1-160
cat $OUT/leafnc.jsonl $OUT/strsm_v.jsonl | cut -c1-220
