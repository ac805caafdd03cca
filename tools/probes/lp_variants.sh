# A/B of k_long_sp builds: bash tools/probes/lp_variants.sh lib1 lib2 ...
set -u
for lib in "" "$@"; do
  for c in block2 digits cfg4t runs_a; do BBPE_LIB_PATH=$lib timeout 300 python tools/lp_probe.py $c 3 2>&1 | grep -v Warn; done
done
