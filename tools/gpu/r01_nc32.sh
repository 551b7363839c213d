RECTRI_CU_LEAF_NC=8 python tools/small_probe.py trmm f32 512,1024,2048 | sed 's/^/nc=8 /'; RECTRI_CU_LEAF_NC=8 python tools/small_probe.py trsm f32 512,1024,2048 | sed 's/^/nc=8 /'
RECTRI_CU_LEAF_NC=16 python tools/small_probe.py trmm f32 512,1024,2048 | sed 's/^/nc=16 /'; RECTRI_CU_LEAF_NC=16 python tools/small_probe.py trsm f32 512,1024,2048 | sed 's/^/nc=16 /'
RECTRI_CU_LEAF_NC=32 python tools/small_probe.py trmm f32 512,1024,2048 | sed 's/^/nc=32 /'; RECTRI_CU_LEAF_NC=32 python tools/small_probe.py trsm f32 512,1024,2048 | sed 's/^/nc=32 /'
