import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2507_11941_b200 as bb
from oracle.oracle import Reference
gpt2 = bb.load_merge_table_files(os.path.join(ROOT, "tests/golden/gpt2.bbpt"), None, "binary")
ids_, off_, blob_, m4_ = gpt2.export()
ref = Reference.from_arrays(ids_, off_, blob_, m4_)
rng = np.random.default_rng(71)
alphabet = list(b"ab cd\n\n\r\t'sll.,!0123 ") + ["é".encode(), "αβ".encode(), b"\xe3\x80\x80", b"\xc2\xa0"]
rows = []
for _ in range(60):
    n = int(rng.integers(0, 3000))
    rows.append(b"".join(alphabet[i] if isinstance(alphabet[i], bytes) else bytes([alphabet[i]]) for i in rng.integers(0, len(alphabet), n)))
rows += [b"word " * 2000, b"\n" * 500 + b"x", b"x\n" * 700, b"a" * 5000, b" \n \n  \n\t\n" * 90]
d, o = bb.pack_rows(rows)
want_ids, want_off = ref.encode_pattern(d, o, "gpt2", workers=8)
enc = bb.Encoder(0, pattern="gpt2")
ids, oo, _ = enc.encode_packed(gpt2, d, o)
single = [enc.encode_packed(gpt2, *bb.pack_rows([r]))[0] for r in rows]
for i in range(len(rows)):
    a = ids[int(oo[i]):int(oo[i+1])].tolist(); b = want_ids[int(want_off[i]):int(want_off[i+1])].tolist()
    if a != b:
        k = next(j for j in range(min(len(a), len(b))) if a[j] != b[j])
        print("row", i, "len", len(rows[i]), "first diff token", k, "got", a[k:k+4], "want", b[k:k+4],
              "alone ok:", single[i].tolist() == b)
        bpos = sum(len(gpt2.bytes_of(t)) for t in b[:k])
        print("   bytes at", bpos, repr(rows[i][max(0, bpos-10):bpos+10]))
