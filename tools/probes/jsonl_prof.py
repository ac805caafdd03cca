"""Device JSONL writer on cfg2's output, for ncu."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_2507_11941_b200 as bb
from workloads import tables as WT, text as WX
t = bb.load_merge_table_files(WT.GPT2_VOCAB, WT.GPT2_MERGES, "gpt2")
data, off, _ = WX.config_rows(WX.TextGen(WX.word_list(WT.gpt2_table()[0])), 2)
n, total = off.size - 1, int(off[-1])
enc = bb.Encoder(0)
d = torch.from_numpy(data).cuda(); o = torch.from_numpy(off.view(np.int64)).cuda()
ids = torch.empty(total, dtype=torch.int32, device="cuda"); oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
enc.encode_device(t, d.data_ptr(), o.data_ptr(), n, total, ids.data_ptr(), oo.data_ptr(), sync=True)
ntok = int(oo[-1].item())
cap = enc.jsonl_device(ids.data_ptr(), oo.data_ptr(), n, ntok, 0, 0)
out = torch.empty(cap, dtype=torch.uint8, device="cuda")
for _ in range(3):
    assert enc.jsonl_device(ids.data_ptr(), oo.data_ptr(), n, ntok, out.data_ptr(), cap) == cap
print("ok", cap)
