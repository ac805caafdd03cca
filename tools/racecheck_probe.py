"""compute-sanitizer --tool racecheck probe: byte-level and gpt2 pattern encodes of
mixed rows (short, long, invalid-ish bytes, digit runs) -- 0 hazards in round 1."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2507_11941_b200 as bb
from workloads import text as synth
t = bb.load_merge_table_files("tests/golden/gpt2.bbpt", None, "binary")
gen = synth.TextGen(synth.word_list(t))
data, off = synth.rows_fixed(gen, 200, 600, seed=5)
rows = [bytes(data[int(off[i]):int(off[i + 1])]) for i in range(200)] + [b"a" * 3000, b"\xff" * 40, b"12345678901234567890" * 10]
d, o = bb.pack_rows(rows)
for pat in (None, "gpt2"):
    e = bb.Encoder(0, pattern=pat)
    ids, oo, _ = e.encode_packed(t, d, o)
print("ok", ids.size)
