# A/B of library builds on the merge-side workloads: bash tools/probes/merge_ab.sh libA libB ...
set -u
for r in 1 2; do
  for lib in "$@"; do
    for c in cfg2 mixed mixed4w cfg4w; do BBPE_LIB_PATH=$lib timeout 300 python tools/lp_probe.py $c 5 2>&1 | grep -v Warn; done
  done
done
