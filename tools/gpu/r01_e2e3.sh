for t in 1 2 4; do echo "panels=$t"; RECTRI_CU_E2E_TRACE=1 RECTRI_CU_E2E_PANELS=$t python tools/e2e_probe.py 16384 16384 0 2>&1 | grep -E "e2e|trace" | head -4; done
