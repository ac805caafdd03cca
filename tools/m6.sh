set -u
O=gpurun_out
mkdir -p $O
: > $O/pairvar.txt
for lib in "" build_variants/pair4.so build_variants/pair8.so; do
  for c in cfg2 mixed digits cfg4t block2; do
    BBPE_LIB_PATH=$lib timeout 300 python tools/lp_probe.py $c 3 >> $O/pairvar.txt 2>&1
  done
done
grep -v Warn $O/pairvar.txt
