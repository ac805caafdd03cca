# long-piece timings + exactness checks after a k_long_sp change
set -u
for c in digits runs_a cfg4t block2; do timeout 300 python tools/lp_probe.py $c 3 2>&1 | grep -v Warn; done
timeout 600 python tools/adversarial_probe.py 2>&1 | grep -o '"case": "[a-z_0-9A-Z]*"\|"mismatches": [0-9]*' | paste - -
timeout 300 python tools/sanitize_longpieces.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_superpass.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
