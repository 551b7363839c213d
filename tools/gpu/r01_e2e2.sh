timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "host" 2>&1 | tail -2
for t in 1 2 4; do echo "panels=$t"; RECTRI_CU_E2E_PANELS=$t python tools/e2e_probe.py 16384 16384 0 0 | grep e2e; done
echo default; python tools/e2e_probe.py 16384 16384 0 0 | grep e2e
