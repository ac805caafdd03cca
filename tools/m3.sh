set -u
O=gpurun_out
mkdir -p $O
(timeout 400 python tools/adversarial_probe.py 2>&1 | tail -12) > $O/adv4.txt
timeout 900 python bench.py --config 4 --table trained --no-extras --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg4t4.json 2> $O/bench_cfg4t4.err
(timeout 900 python -m pytest tests/test_gpu_specops.py tests/test_gpu_parity.py -m gpu -x -q -k "specops or sharded or block or long or adversarial or trace" 2>&1 | tail -15) > $O/gputest4.txt
python -c "
import json
for l in open('$O/adv4.txt'):
    try: d=json.loads(l); print(d['case'], d['kernel_ms']['k_long_pieces'], d['parity']['mismatches'])
    except Exception: print(l[:300])
d=json.loads(open('$O/bench_cfg4t4.json').read().strip().splitlines()[-1]); print(d['value']/1e6, d['ms_per_step'], d['kernel_ms']['k_long_pieces'], d['parity'])"; tail -3 $O/bench_cfg4t4.err; cat $O/gputest4.txt
