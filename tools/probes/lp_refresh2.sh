# Bench lines and ncu captures touched by the long-piece tier (both k_long_sp
# instances summarised: main, then PIPE) plus the default cfg2 line.
set -u
O=gpurun_out/r2b; mkdir -p $O
B="timeout 1200 python bench.py"
$B > $O/r2_bench_cfg2.json 2> $O/cfg2.err; tail -c 300 $O/cfg2.err | grep -i -E "error|traceback"
$B --config 4 --table trained --steps 5 > $O/r2_bench_cfg4_trained.json 2> $O/t.err
$B --config 1 --engine block > $O/r2_bench_cfg1_block.json 2> $O/b1.err
$B --engine block --steps 3 --no-extras > $O/r2_bench_cfg2_block.json 2> $O/b2.err
prof() {
  local tag=$1; shift
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_long_sp --launch-skip 2 -c 2 -f -o $O/$tag \
    python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-extras --parity none "$@" > $O/$tag.log 2>&1
  python profiles/summarize.py $O/$tag.ncu-rep $O/$tag paper_2507_11941_b200/csrc/longpieces.cu > /dev/null 2>&1 || echo "summary $tag failed"
}
prof r2_k_long_pieces_cfg4_zipf_trained --config 4 --table trained
prof r2_k_long_pieces_cfg1_zipf_block --config 1 --engine block
prof r2_k_long_pieces_cfg2_zipf_block --engine block
ls $O
