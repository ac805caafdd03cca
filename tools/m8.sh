set -u
O=gpurun_out
mkdir -p $O
for c in digits runs_a cfg4t block2 cfg2; do timeout 300 python tools/lp_probe.py $c 3 2>&1 | grep -v Warn; done
(timeout 400 python tools/adversarial_probe.py 2>&1 | tail -12) > $O/adv8.txt
python -c "
import json
for l in open('$O/adv8.txt'):
    try: d=json.loads(l); print(d['case'], d['kernel_ms']['k_long_pieces'], d['parity']['mismatches'])
    except Exception: print(l[:300])"
timeout 900 python bench.py --config 4 --table trained --no-extras --steps 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4t', d['ms_per_step'], d['parity']['mismatches'], d['gpu_launches'])"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_specops.py -m gpu -x -q 2>&1 | tail -2
