"""cfg2 rows ending in <|endoftext|> + BOS through the device specials path, for ncu."""
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
sp = bb.SpecialTokenSet(); sp.add("<|endoftext|>", 50256)
d = torch.from_numpy(data.copy()).cuda().view(n, 256)
d[:, -13:] = torch.tensor(list(b"<|endoftext|>"), dtype=torch.uint8, device="cuda")
o = torch.from_numpy(off.view(np.int64)).cuda()
enc.set_specials(sp)
cap = total + 2 * n
ids = torch.empty(cap, dtype=torch.int32, device="cuda"); oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
for _ in range(3):
    k = enc.encode_batch_device(t, d.data_ptr(), o.data_ptr(), n, total, ids.data_ptr(), cap, oo.data_ptr(), bos_id=50256)
print("ok", k)
