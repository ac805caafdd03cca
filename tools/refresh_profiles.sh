#!/bin/bash
# Round-2 measurement on one B200 (run under gpurun from the repo root):
# bench lines (both arms on cfg2, every BASELINE config, the trained cfg4
# table, the text classes, the paper's block engine), the ncu launch list of
# the headline command, and ncu --set full summaries of each line's dominant
# kernel (the bench line's `traffic` reads them back from profiles/).
# Outputs: gpurun_out/r2/ (copy into profiles/).
set -u
O=gpurun_out/r2
R=/tmp/ncu_r2
mkdir -p $O $R
B="timeout 1200 python bench.py"
run() {  # name, bench args
  local name=$1; shift
  $B "$@" > $O/r2_bench_$name.json 2> $O/r2_bench_$name.err
  tail -c 400 $O/r2_bench_$name.err | grep -i -E "error|traceback" && echo "bench $name failed"
}
run cfg2
$B --impl reference > $O/r2_bench_reference_cfg2.json 2> $O/r2_bench_reference_cfg2.err
run cfg1 --config 1
run cfg3 --config 3
run cfg4 --config 4
run cfg4_trained --config 4 --table trained --steps 5
run cfg5 --config 5 --scale 0.125
run cfg2_corpus --text corpus
run cfg2_mixed --text mixed
run cfg1_block --config 1 --engine block
run cfg2_block --engine block --steps 3 --no-extras
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2_launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-extras --parity none > $R/launch.log 2>&1
prof() {  # kernel-regex, tag, bench args
  local k=$1 tag=$2; shift 2
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$k" --launch-skip 2 -c 1 -f -o $R/$tag \
    python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-extras --parity none "$@" > $R/$tag.log 2>&1
  python profiles/summarize.py $R/$tag.ncu-rep $O/$tag paper_2507_11941_b200/csrc/kernels.cu > /dev/null 2>&1 || echo "summary $tag failed"
}
prof k_pieces r2_k_pieces_cfg2_zipf
prof k_gather r2_k_gather_cfg2_zipf
prof "k_merge|k_refs|k_dedup" r2_merge_kernels_cfg2_zipf
prof k_pieces r2_k_pieces_cfg1_zipf --config 1
prof k_pieces r2_k_pieces_cfg3_zipf --config 3
prof k_pieces r2_k_pieces_cfg4_zipf --config 4
prof k_pieces r2_k_pieces_cfg5_zipf --config 5 --scale 0.125
prof k_pieces r2_k_pieces_cfg2_corpus --text corpus
prof k_pieces r2_k_pieces_cfg2_mixed --text mixed
prof "k_long_sp" r2_k_long_pieces_cfg4_zipf_trained --config 4 --table trained
prof "k_long_sp" r2_k_long_pieces_cfg1_zipf_block --config 1 --engine block
prof "k_long_sp" r2_k_long_pieces_cfg2_zipf_block --engine block
cp $R/r2_k_long_pieces_cfg4_zipf_trained.ncu-rep $O/ 2>/dev/null
ls -la $O
