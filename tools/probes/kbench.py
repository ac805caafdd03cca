#!/usr/bin/env python3
"""Device-resident cfg2 encode, K steps: ms/step and per-kernel ms (CUDA events).
Library variant via BBPE_LIB_PATH."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_2507_11941_b200 as bb
from workloads import text as synth
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
memo = (sys.argv[2] != "nomemo") if len(sys.argv) > 2 else True
pattern = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] != "none" else None
dedup = (sys.argv[4] != "nodedup") if len(sys.argv) > 4 else True
t = bb.load_merge_table_files(os.path.join(ROOT, "tests/golden/gpt2.bbpt"), None, "binary")
if cfg == 4:
    from workloads import tables as WT
    t = bb.MergeTable.from_arrays(*WT.arrays(*WT.extend_wordlevel(*WT.gpt2_table(), 200000)))
gen = synth.TextGen(synth.word_list(t))
data, off, desc = synth.config_rows(gen, cfg, scale=1 / 16 if cfg == 5 else 1.0, seed=cfg * 1000)
n, total = off.size - 1, int(off[-1])
enc = bb.Encoder(device=0, piece_memo=memo, pattern=pattern, dedup=dedup)
enc.prepare(t)
s = torch.cuda.Stream()
d_data = torch.from_numpy(data).cuda()
d_off = torch.from_numpy(off.view(np.int64)).cuda()
d_ids = torch.empty(total, dtype=torch.int32, device="cuda")
d_oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
def step():
    enc.encode_device(t, d_data.data_ptr(), d_off.data_ptr(), n, total, d_ids.data_ptr(), d_oo.data_ptr(),
                      stream=s.cuda_stream, sync=False)
for _ in range(3):
    step()
enc.sync(); enc.kernel_times(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 5
with torch.cuda.stream(s):
    e0.record(s)
    for _ in range(K):
        step()
    e1.record(s)
enc.sync(); torch.cuda.synchronize()
kt, kc = enc.kernel_times(reset=True)
print(json.dumps({"lib": os.path.basename(os.environ.get("BBPE_LIB_PATH", "default")), "cfg": cfg, "memo": memo,
                  "ms": round(e0.elapsed_time(e1) / K, 4), "tokens": int(d_oo[-1].item()),
                  "kernels": {k: round(v / max(kc, 1), 4) for k, v in kt.items()}}), flush=True)
