set -u
for lib in "" build_variants/dd64_16.so build_variants/dd32_16.so build_variants/dd128_4.so build_variants/dd32_8.so; do
  for c in cfg2 mixed; do BBPE_LIB_PATH=$lib timeout 300 python tools/lp_probe.py $c 5 2>&1 | grep -v Warn; done
done
