# A/B of two library builds on the cfg2 / mixed pieces path: bash tools/probes/bulk_ab.sh libA libB
set -u
for r in 1 2; do
  for lib in "$@"; do
    for c in cfg2 mixed; do BBPE_LIB_PATH=$lib timeout 300 python tools/lp_probe.py $c 5 2>&1 | grep -v Warn; done
  done
done
