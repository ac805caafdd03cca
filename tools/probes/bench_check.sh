set -u
s=$(date +%s); python bench.py --steps 20 --warmup 5 > gpurun_out/bt_cfg2.json 2> gpurun_out/bt_cfg2.err; echo "cfg2 rc=$? $(( $(date +%s) - s ))s"
python -c "
import json; d=json.loads(open('gpurun_out/bt_cfg2.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['parity']['mismatches'], d['roofline']['traffic'], d['gpu_launches'])"
s=$(date +%s); BBPE_BENCH_SHARED_GPU=1 python bench.py --gpus 2 --config 5 --scale 0.02 --steps 3 --warmup 3 --no-extras > gpurun_out/bt_n2_cfg5.json 2> gpurun_out/bt_n2_cfg5.err; echo "n2 cfg5 rc=$? $(( $(date +%s) - s ))s"
tail -c 600 gpurun_out/bt_n2_cfg5.json; tail -3 gpurun_out/bt_n2_cfg5.err
s=$(date +%s); BBPE_BENCH_SHARED_GPU=1 python bench.py --gpus 2 --steps 3 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bt_n2_cfg2.json 2> gpurun_out/bt_n2_cfg2.err; echo "n2 cfg2 rc=$? $(( $(date +%s) - s ))s"
python -c "
import json; d=json.loads(open('gpurun_out/bt_n2_cfg2.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['value']/1e9, d['tokens_per_step'], d['parity']['rows_checked'], d['parity']['mismatches'], d['parallelism'])"
tail -3 gpurun_out/bt_n2_cfg2.err
s=$(date +%s); python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bt_ref.json 2>&1; echo "ref rc=$? $(( $(date +%s) - s ))s"; tail -c 300 gpurun_out/bt_ref.json
