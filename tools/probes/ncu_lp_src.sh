# ncu source-level capture of k_long_sp for one lp_probe case: bash tools/probes/ncu_lp_src.sh block2
set -u
c=$1
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_long_sp --launch-skip 2 -c 1 -f -o /tmp/lp_$c python tools/lp_probe.py $c 1 > /tmp/lp_$c.log 2>&1
ncu -i /tmp/lp_$c.ncu-rep --page source --csv --print-source=cuda,sass > $O/lp_src_$c.csv 2>/dev/null
python profiles/summarize.py /tmp/lp_$c.ncu-rep $O/lp_$c paper_2507_11941_b200/csrc/longpieces.cu > /dev/null 2>&1
head -20 $O/lp_$c.txt
