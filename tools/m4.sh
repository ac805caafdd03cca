set -u
O=gpurun_out
mkdir -p $O
for c in digits cfg4t; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_long_sp --launch-skip 1 -c 1 -f -o $O/k_long_sp_$c python tools/lp_probe.py $c 2 > $O/ncu_lp_$c.log 2>&1
tail -2 $O/ncu_lp_$c.log
done
