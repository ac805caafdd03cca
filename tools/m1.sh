set -u
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py --config 4 --table trained --no-extras --steps 3 --warmup 3 > $O/bench_cfg4t.json 2> $O/bench_cfg4t.err
timeout 600 python bench.py --config 1 --engine block --no-extras > $O/bench_cfg1_block.json 2> $O/bench_cfg1_block.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_long_pieces -c 1 -f -o $O/k_long_cfg4t \
  python bench.py --config 4 --table trained --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --parity none > $O/ncu_lp.log 2>&1
tail -c 3000 $O/bench_cfg4t.json; tail -3 $O/bench_cfg4t.err; tail -c 1500 $O/bench_cfg1_block.json; tail -3 $O/bench_cfg1_block.err; tail -5 $O/ncu_lp.log
