#!/usr/bin/env python3
"""cfg2 rows with specials: bbpe_encode_batch_device (device split + encode +
stitch) vs the plain encode of the same bytes; CUDA-event ms per call."""
import os, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import paper_2507_11941_b200 as bb
from workloads import text as synth
t = bb.load_merge_table_files(os.path.join(ROOT, "tests/golden/gpt2.bbpt"), None, "binary")
gen = synth.TextGen(synth.word_list(t))
data, off, _ = synth.config_rows(gen, 2, seed=2000)
n = off.size - 1
eot = np.frombuffer(b"<|endoftext|>", np.uint8)
# every row: its 256 bytes with the last 13 replaced by <|endoftext|>
d2 = data.reshape(n, 256).copy()
d2[:, -13:] = eot
data = d2.reshape(-1)
total = int(off[-1])
sp = bb.SpecialTokenSet()
sp.add("<|endoftext|>", 50256)
enc = bb.Encoder(0)
enc.prepare(t)
enc.set_specials(sp)
d_data = torch.from_numpy(data).cuda()
d_off = torch.from_numpy(off.view(np.int64)).cuda()
cap = total + 2 * n
d_ids = torch.empty(cap, dtype=torch.int32, device="cuda")
d_oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
def sp_call():
    return enc.encode_batch_device(t, d_data.data_ptr(), d_off.data_ptr(), n, total, d_ids.data_ptr(), cap,
                                   d_oo.data_ptr(), 50256, None)
def plain():
    enc.encode_device(t, d_data.data_ptr(), d_off.data_ptr(), n, total, d_ids.data_ptr(), d_oo.data_ptr())
res = {}
for name, f in [("specials_bos", sp_call), ("plain", plain)]:
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 5
    e0.record()
    for _ in range(K):
        f()
    e1.record()
    torch.cuda.synchronize()
    res[name] = e0.elapsed_time(e1) / K
res["ids"] = int(d_oo[-1].item())
print(json.dumps(res))
