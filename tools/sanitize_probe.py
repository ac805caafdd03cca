"""Small invocations of the newer device paths for compute-sanitizer memcheck:
gpt2 pattern mode (short and long rows, aligned and unaligned), specials
(in place and compacted layouts) with BOS/EOS, decode with specials, the
splitter bitmap, the chunked device encode boundary logic on a small batch."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_11941_b200 as bb
t = bb.load_merge_table_files("tests/golden/gpt2.bbpt", None, "binary")
toy = bb.MergeTable.build([(0, b"a"), (1, b"b"), (2, b"c"), (3, b"ab"), (4, b"abc")], [(0, 0, 1, 3), (1, 3, 2, 4)])
rows = [b"hello world's test", b"", b"a" * 5000, "café \xa0\xa0x".encode(), b"word " * 1500, b"x\n" * 100, b"<|a|>x<|a|>"]
d, o = bb.pack_rows(rows)
e = bb.Encoder(0, pattern="gpt2")
ids, oo, _ = e.encode_packed(t, d, o)
for shift in (0, 3):
    buf = torch.zeros(d.size + 16, dtype=torch.uint8, device="cuda")
    buf[shift:shift + d.size] = torch.from_numpy(d.copy()).cuda()
    do = torch.from_numpy(o.view(np.int64).copy()).cuda()
    di = torch.empty(d.size, dtype=torch.int32, device="cuda")
    doo = torch.empty(o.size, dtype=torch.int64, device="cuda")
    e.encode_device(t, buf.data_ptr() + shift, do.data_ptr(), o.size - 1, d.size, di.data_ptr(), doo.data_ptr())
    bits = torch.zeros((d.size + 31) // 32, dtype=torch.int32, device="cuda")
    e.pretokenize_device(buf.data_ptr() + shift, do.data_ptr(), o.size - 1, d.size, bits.data_ptr())
sp = bb.SpecialTokenSet()
sp.add("<|a|>", 60001)
sp.add("x", 60002)
sp.set_bos("<|a|>")
for tab in (t, toy):
    rr = rows if tab is t else [b"abx", b"xab", b"x", b""]
    cfg = bb.BlockConfig(256, None)
    be = bb.encode_batch(rr, tab, sp, cfg, 0, True, False)
    bb.decode_batch(be, tab, sp, True)
    bb.decode_batch(be, tab, sp, False) if tab is t else None
print("ok")
