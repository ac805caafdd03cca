set -u
for lib in "" build_variants/kmerge_bf.so; do
  for c in mixed cfg2; do BBPE_LIB_PATH=$lib timeout 300 python tools/lp_probe.py $c 5 2>&1 | grep -v Warn; done
done
