# Long-piece tier after a k_long_sp change: adversarial batches (every row
# checked against oracle/_ref), the trained cfg4 bench line and ncu of both
# k_long_sp instances on it.
set -u
O=gpurun_out/lp; mkdir -p $O
timeout 1500 python tools/adversarial_probe.py > $O/adversarial.jsonl 2> $O/adversarial.err; tail -3 $O/adversarial.err
timeout 900 python bench.py --config 4 --table trained --steps 5 > $O/r2_bench_cfg4_trained.json 2> $O/bench.err; tail -2 $O/bench.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_long_sp --launch-skip 2 -c 2 -f -o $O/r2_k_long_pieces_cfg4_zipf_trained \
  python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-extras --parity none --config 4 --table trained > $O/ncu.log 2>&1
python profiles/summarize.py $O/r2_k_long_pieces_cfg4_zipf_trained.ncu-rep $O/r2_k_long_pieces_cfg4_zipf_trained paper_2507_11941_b200/csrc/longpieces.cu > /dev/null 2>&1 || echo "summary failed"
ls $O
