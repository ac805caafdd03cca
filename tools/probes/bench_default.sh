set -u
s=$(date +%s); python bench.py --steps 20 --warmup 5 > gpurun_out/bd_cfg2.json 2> gpurun_out/bd_cfg2.err; echo "cfg2 rc=$? $(( $(date +%s) - s ))s"
tail -3 gpurun_out/bd_cfg2.err
python -c "
import json; d=json.loads(open('gpurun_out/bd_cfg2.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['ms_per_step'], d['parity']['mismatches'])
for k,v in (d.get('workloads') or {}).items(): print(k, round(v['ms_per_step'],3), round(v['tokens_per_s']/1e9,3), v['dominant_kernel'], round(100*v['roofline_frac'],3), v['parity']['rows_checked'], v['parity']['mismatches'])"
