set -u
O=gpurun_out
mkdir -p $O
: > $O/lpvar2.txt
for lib in "" build_variants/noovf.so build_variants/lp_b4_s12288.so build_variants/lp_b6_s8192.so build_variants/lp_b8_s4096.so; do
  for c in digits runs_a cfg4t; do
    BBPE_LIB_PATH=$lib timeout 300 python tools/lp_probe.py $c 3 >> $O/lpvar2.txt 2>&1
  done
done
cat $O/lpvar2.txt | grep -v Warn
