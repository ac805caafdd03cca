set -u
timeout 900 python -m pytest tests -m gpu -q -x -k "decode or jsonl or round_trip or cli" 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-workload-legs --parity none 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('decode', d['decode']); print('jsonl', d['jsonl'])"
