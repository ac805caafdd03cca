# ncu --set full of k_merge / k_dedup / k_refs on the mixed-text cfg2 workload
set -u
mkdir -p gpurun_out
for k in k_merge k_dedup k_refs; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" --launch-skip 1 -c 1 -f \
    -o gpurun_out/r2_${k}_cfg2_mixed python tools/lp_probe.py mixed 1 > /dev/null 2>&1 || echo "ncu $k failed"
  python profiles/summarize.py gpurun_out/r2_${k}_cfg2_mixed.ncu-rep gpurun_out/r2_${k}_cfg2_mixed paper_2507_11941_b200/csrc/kernels.cu > /dev/null 2>&1 || echo "summary $k failed"
done
ls gpurun_out
