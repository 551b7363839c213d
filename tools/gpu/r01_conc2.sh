for cfg in "4096 2097152" "8192 2097152" "8192 1048576" "8192 524288" "16384 1048576"; do set -- $cfg; echo "maxn=$1 elems=$2"; RECTRI_CU_TRMM_CONC_MAXN=$1 RECTRI_CU_TRMM_CONC_ELEMS=$2 python tools/small_probe.py trmm f64 2048,4096,8192,16384 | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print(' ', d['n'], round(d['pipe_us'],1), round(d['cublas_us'],1))"; done
