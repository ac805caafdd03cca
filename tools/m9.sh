set -u
for c in digits runs_a cfg4t block2; do timeout 300 python tools/lp_probe.py $c 3 2>&1 | grep -v Warn; done
timeout 900 python bench.py --config 1 --engine block --no-extras --steps 10 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg1block', d['ms_per_step'], d['parity']['mismatches'])"
timeout 900 python bench.py --config 4 --table trained --no-extras --steps 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4t', d['ms_per_step'], d['parity']['mismatches'])"
timeout 600 python tools/adversarial_probe.py 2>&1 | grep -o '"case": "[a-z_0-9A-Z]*"\|"mismatches": [0-9]*' | paste - - 
