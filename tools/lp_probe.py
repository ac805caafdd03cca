"""Long-piece tier probe for ncu: one workload encoded `reps` times on the
device (digits | runs_a | cfg4t | cfg4w | mixed4w | cfg2 | mixed | block1 | block2).  python tools/lp_probe.py digits 3"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2507_11941_b200 as bb
from workloads import tables as WT, text as WX

case = sys.argv[1] if len(sys.argv) > 1 else "digits"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rng = np.random.default_rng(7)
N = 256 << 20
engine = "pieces"
if case in ("cfg2", "mixed", "block2", "block1"):
    t = bb.load_merge_table_files(WT.GPT2_VOCAB, WT.GPT2_MERGES, "gpt2")
    gen = WX.make_gen("mixed" if case == "mixed" else "zipf", WT.gpt2_table()[0])
    data, off, _ = WX.config_rows(gen, 1 if case == "block1" else 2, seed=2000)
    engine = "block" if case.startswith("block") else "pieces"
elif case in ("cfg4w", "mixed4w"):  # the word-level 200k table (wide keys): zipf / mixed text
    tokens, m = WT.extend_wordlevel(*WT.gpt2_table(), 200000)
    t = bb.MergeTable.from_arrays(*WT.arrays(tokens, m))
    gen = WX.make_gen("mixed", WT.gpt2_table()[0]) if case == "mixed4w" else WX.TextGen(WX.word_list(tokens))
    data, off, _ = WX.config_rows(gen, 4 if case == "cfg4w" else 2, seed=2000)
elif case == "cfg4t":
    from workloads import train
    tokens, m, _ = train.trained_table(*WT.gpt2_table(), 200000)
    t = bb.MergeTable.from_arrays(*WT.arrays(tokens, m))
    data, off, _ = WX.config_rows(WX.TextGen(WX.word_list(WT.gpt2_table()[0])), 4)
else:
    t = bb.load_merge_table_files(WT.GPT2_VOCAB, WT.GPT2_MERGES, "gpt2")
    if case == "digits":
        data, L = rng.integers(48, 58, N, dtype=np.uint8), 4096
    else:
        data, L = np.full(N, ord("a"), np.uint8), 65536
    off = np.arange(0, N + 1, L, dtype=np.uint64)
enc = bb.Encoder(0, engine=engine)
n, total = off.size - 1, int(off[-1])
d = torch.from_numpy(data).cuda()
o = torch.from_numpy(off.view(np.int64)).cuda()
ids = torch.empty(total, dtype=torch.int32, device="cuda")
oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
enc.encode_device(t, d.data_ptr(), o.data_ptr(), n, total, ids.data_ptr(), oo.data_ptr(), sync=True)
enc.kernel_times(reset=True)
for _ in range(reps):
    enc.encode_device(t, d.data_ptr(), o.data_ptr(), n, total, ids.data_ptr(), oo.data_ptr(), sync=True)
kt, calls = enc.kernel_times(reset=True)
print(case, os.path.basename(os.environ.get("BBPE_LIB_PATH", "base")), {k: round(v / max(calls, 1), 3) for k, v in kt.items() if v > 0.05 * calls})
