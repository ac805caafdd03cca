#!/bin/bash
# Round-end measurement on one B200 (run under gpurun from the repo root):
# bench lines (both arms, cfg2 headline + cfg1/3/4/5), the ncu launch list of
# the headline command and one ncu --set full capture of k_pieces.
# Outputs land in gpurun_out/; copy the summaries into profiles/.
set -u
O=gpurun_out
mkdir -p $O
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --impl reference > $O/bench_ref_cfg2.json 2> $O/bench_ref_cfg2.err
for c in 1 3 4 5; do
  python bench.py --config $c > $O/bench_cfg$c.json 2> $O/bench_cfg$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pieces --launch-skip 2 -c 1 -f -o $O/k_pieces_cfg2 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
ls -la $O
