set -u
O=gpurun_out
mkdir -p $O
for c in digits runs_a cfg4t block2 mixed; do timeout 300 python tools/lp_probe.py $c 3 2>&1 | grep -v Warn; done
(timeout 400 python tools/adversarial_probe.py 2>&1 | tail -12) > $O/adv7.txt
python -c "
import json
for l in open('$O/adv7.txt'):
    try: d=json.loads(l); print(d['case'], d['kernel_ms']['k_long_pieces'], d['parity']['mismatches'])
    except Exception: print(l[:300])"
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
