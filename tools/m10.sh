set -u
O=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pieces --launch-skip 2 -c 1 -f -o $O/kp_cfg2 python bench.py --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --no-extras --parity none > /tmp/kp.log 2>&1
ncu -i $O/kp_cfg2.ncu-rep --page source --csv --print-source=cuda,sass > $O/kp_src.csv 2>/dev/null
ls -la $O/kp_*
