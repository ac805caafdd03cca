set -u
O=gpurun_out
mkdir -p $O
(timeout 400 python tools/adversarial_probe.py 2>&1 | tail -12) > $O/adv2.txt
timeout 900 python bench.py --config 4 --table trained --no-extras --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg4t2.json 2> $O/bench_cfg4t2.err
(timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15) > $O/gputest2.txt
cut -c1-600 $O/adv2.txt; python -c "
import json; d=json.loads(open('$O/bench_cfg4t2.json').read().strip().splitlines()[-1]); print(d['value']/1e6, d['ms_per_step'], d['kernel_ms'], d['parity'])"; tail -3 $O/bench_cfg4t2.err; cat $O/gputest2.txt
