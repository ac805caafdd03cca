"""Device decode of the cfg2 output, for ncu (kernel times of the decode path)."""
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
back = torch.empty(total, dtype=torch.uint8, device="cuda"); boff = torch.empty(n + 1, dtype=torch.int64, device="cuda")
for _ in range(3):
    enc.decode_device(t, ids.data_ptr(), oo.data_ptr(), n, ntok, back.data_ptr(), total, boff.data_ptr())
assert torch.equal(back, d)
print("ok")
