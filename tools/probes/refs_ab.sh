set -u
for lib in "" build_variants/refs_half.so; do
  for c in cfg2 mixed; do BBPE_LIB_PATH=$lib timeout 300 python tools/lp_probe.py $c 10 2>&1 | grep -v Warn; done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "dedup or cfg2 or sharded or text_classes or jsonl" 2>&1 | tail -1
