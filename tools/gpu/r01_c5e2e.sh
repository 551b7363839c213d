for t in 1 2 4 8; do echo "panels=$t"; RECTRI_CU_E2E_PANELS=$t RECTRI_CU_E2E_TRACE=1 python tools/e2e_probe.py 8192 65536 0 2>&1 | grep -E "e2e (panel|trace)" | tail -2; done
