set -u
for lib in "" build_variants/ge5.so build_variants/ge8.so; do
  for c in cfg2 mixed; do BBPE_LIB_PATH=$lib timeout 300 python tools/lp_probe.py $c 10 2>&1 | grep -v Warn; done
done
