"""The super-pass long-piece kernel (k_long_sp, csrc/longpieces.cu) against
the oracle's block engine (oracle/bpe_oracle.c, restating
block_engine.hpp:268-310) on adversarial inputs for its rule: random
consistent AND inconsistent tables over 2-4 letters (so nearly every pair is
a merge and runs of one repeated pair are common), rows of runs up to 20k
tokens (shared-memory pieces, L2 pieces and the pipelined > 8K instance), both
engines (every row one piece, and the piece decomposition). The CPU pin of
the same rule is tests/test_superpass.py."""
import random

import numpy as np
import pytest

import paper_2507_11941_b200 as bb
from oracle.oracle import CRestatement

pytestmark = pytest.mark.gpu


def _table(rng, alphabet, merges, consistent):
    toks = {i: bytes([97 + i]) for i in range(alphabet)}
    words, used, ms, nid = set(toks.values()), set(), [], alphabet
    for _ in range(merges * 8):
        if len(ms) >= merges:
            break
        pool = list(toks)
        l = rng.choice(pool)
        r = l if rng.random() < 0.3 else rng.choice(pool)
        if (l, r) in used or toks[l] + toks[r] in words:
            continue
        used.add((l, r))
        toks[nid] = toks[l] + toks[r]
        words.add(toks[nid])
        ms.append((l, r, nid))
        nid += 1
    order = list(range(len(ms)))
    if not consistent:
        rng.shuffle(order)
    merges4 = [(order[k],) + ms[k] for k in range(len(ms))]
    return toks, merges4


def _rows(rng, alphabet, n_rows, max_len):
    rows = []
    for _ in range(n_rows):
        target = rng.choice([rng.randrange(0, 64), rng.randrange(0, max_len)])
        s = bytearray()
        while len(s) < target:
            s += bytes([97 + rng.randrange(alphabet)]) * rng.choice([1, 1, 2, 3, rng.randrange(1, 200)])
        rows.append(bytes(s[:target]))
    return rows


@pytest.mark.parametrize("consistent", [True, False])
@pytest.mark.parametrize("engine", ["block", "pieces"])
def test_superpass_kernel_vs_oracle_random_tables(consistent, engine):
    rng = random.Random(101 if consistent else 202)
    for trial in range(30):
        A = rng.randrange(2, 5)
        toks, m4 = _table(rng, A, rng.randrange(4, 60), consistent)
        table = bb.MergeTable.build(sorted(toks.items()), m4)
        orc = CRestatement(np.array(m4, np.uint32).reshape(-1, 4), list(range(A)) + [0xFFFFFFFF] * (256 - A))
        rows = _rows(rng, A, 60, 20000 if trial % 3 == 0 else 3000)
        data, off = bb.pack_rows(rows)
        ids, oo, _ = bb.Encoder(0, engine=engine).encode_packed(table, data, off)
        # the oracle's alphabet is byte - 97
        wi, wo = orc.encode_packed(np.where(data >= 97, data - 97, data).astype(np.uint8), off)
        assert np.array_equal(oo, wo), (trial, consistent, engine)
        assert np.array_equal(ids, wi), (trial, consistent, engine)
