"""Small invocations of the round-2 device paths for compute-sanitizer
(memcheck, racecheck, synccheck): the super-pass long-piece kernel on narrow
(GPT-2) and wide (trained 200k-merge) tables, in shared memory and from the
global scratch, both kernel instances (pieces <= 8K and > 8K positions), the
block engine on whole rows, the pass-by-pass engine (max_passes), the spec
ops, and the sharded encode over two contexts. Each result is checked against
the C restatement of the reference (oracle/).

  compute-sanitizer --tool memcheck python tools/sanitize_longpieces.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_11941_b200 as bb  # noqa: E402
from oracle.oracle import CRestatement  # noqa: E402
from workloads import tables as WT, text as WX  # noqa: E402

rng = np.random.default_rng(3)


def check(table, rows, engine="pieces", max_passes=None):
    _, _, _, m4 = table.export()
    orc = CRestatement(m4, [table.byte_token(b) for b in range(256)])
    d, o = bb.pack_rows(rows)
    enc = bb.Encoder(0, engine=engine, config=bb.BlockConfig(256, max_passes))
    ids, oo, _ = enc.encode_packed(table, d, o)
    wi, wo = orc.encode_packed(d, o)
    assert np.array_equal(oo, wo) and np.array_equal(ids, wi), (engine, max_passes)


gpt2 = bb.load_merge_table_files(WT.GPT2_VOCAB, WT.GPT2_MERGES, "gpt2")
digits = bytes(rng.integers(48, 58, 3000, dtype=np.uint8))
rows = [b"a" * 9000, b"." * 2100, digits, b"0" * 700, b"x" * 40, b"", bytes(rng.integers(0, 256, 500, dtype=np.uint8))]
check(gpt2, rows)                                   # k_long_sp<narrow>: smem, L2, and > 8K positions
check(gpt2, rows[2:], engine="block")               # whole rows (BBPE_ENGINE_BLOCK)
check(gpt2, [b"hello world " * 30, digits[:600]], engine="block", max_passes=100000)  # k_long_pieces

from workloads import train  # noqa: E402
toks, merges, _ = train.trained_table(*WT.gpt2_table(), 200000, text_bytes=4 << 20)
wide = bb.MergeTable.from_arrays(*WT.arrays(toks, merges))
gen = WX.TextGen(WX.word_list(WT.gpt2_table()[0]))
d, o, _ = WX.config_rows(gen, 4, scale=1 / 2048)
trows = [d[int(o[i]):int(o[i + 1])].tobytes() for i in range(o.size - 1)]
check(wide, trows + [b"the the the " * 800])        # k_long_sp<wide>

toy = bb.MergeTable.build([(0, b"a"), (1, b"b"), (2, b"c"), (3, b"ab"), (4, b"abc")], [(0, 0, 1, 3), (1, 3, 2, 4)])
assert bb.block_bpe_replay([0, 1, 2, 0, 1], toy) == [4, 3]
assert bb.compact([0, 1, 0, 1], toy, [0, 1, 0, 1], [0, 0, 1, 1]) == [3, 3]
try:
    bb.compact([2, 2], toy, [0, 1], [0, 0])
    raise SystemExit("expected ContractViolation")
except bb.ContractViolation:
    pass

dd, oo2 = bb.pack_rows([b"some text here %d " % i * 7 for i in range(3000)])
ids1, off1, _ = bb.Encoder(0).encode_packed(gpt2, dd, oo2)
ids2, off2, _ = bb.encode_sharded([bb.Encoder(0), bb.Encoder(0)], gpt2, dd, oo2, capacity=int(ids1.size))
assert np.array_equal(ids1, ids2) and np.array_equal(off1, off2)
print("ok")
