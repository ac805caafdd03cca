"""CPU pin of the super-pass rule that k_long_sp (csrc/longpieces.cu) uses.

A super-pass applies, in one sweep, every pair that block_bpe would merge in
its passes below a cut C (see the kernel's header comment):
  * pair i merges iff rank r_i exists, a_i is even and b_i is even, where
    a_i = consecutive steps r_{j-1} <= r_j ending at i and b_i = consecutive
    steps r_{j+1} < r_j starting at i;
  * C = min over those merges of max(x, tau + 1), x the rank of a pair the
    merge creates with its neighbour token as of its pass tau;
  * the merges with r_i < C are applied, the rest wait for the next sweep.
`superpass_bpe` below is a direct Python statement of those four sweeps; the
tests check it equals the oracle's block engine (oracle/bpe_oracle.c,
restating block_engine.hpp:268-310) on random consistent AND inconsistent
tables (runs of repeated tokens included), the reference's inconsistent-table
KAT, GPT-2 text, and the adversarial run/digit rows of SURVEY §8c, and that it
needs far fewer sweeps than passes.
"""
import random

import numpy as np
import pytest

from oracle.oracle import CRestatement

NONE = 0xFFFFFFFF


def superpass_bpe(t, rank, merged, stats=None):
    t = list(t)
    sweeps = 0
    while len(t) >= 2:
        n = len(t)
        r = [rank.get((t[i], t[i + 1]), NONE) for i in range(n - 1)] + [NONE]
        a = [0] * n
        b = [0] * n
        for i in range(1, n):
            a[i] = a[i - 1] + 1 if r[i - 1] <= r[i] else 0
        for i in range(n - 2, -1, -1):
            b[i] = b[i + 1] + 1 if r[i + 1] < r[i] else 0
        mg = [r[i] != NONE and a[i] % 2 == 0 and b[i] % 2 == 0 for i in range(n)]
        if not any(mg):
            break
        C = NONE
        for i in range(n - 1):
            if not mg[i]:
                continue
            tau, M = r[i], merged[(t[i], t[i + 1])]
            if i >= 1:
                lt = merged[(t[i - 2], t[i - 1])] if i >= 2 and mg[i - 2] and r[i - 2] <= tau else t[i - 1]
                x = rank.get((lt, M), NONE)
                if x != NONE:
                    C = min(C, max(x, tau + 1))
            if i + 2 < n:
                rt = merged[(t[i + 2], t[i + 3])] if mg[i + 2] and r[i + 2] <= tau else t[i + 2]
                x = rank.get((M, rt), NONE)
                if x != NONE:
                    C = min(C, max(x, tau + 1))
        out, i = [], 0
        while i < n:
            if mg[i] and r[i] < C:
                out.append(merged[(t[i], t[i + 1])])
                i += 2
            else:
                out.append(t[i])
                i += 1
        assert len(out) < n  # progress: the global minimum is always below C
        t = out
        sweeps += 1
    if stats is not None:
        stats["sweeps"] = stats.get("sweeps", 0) + sweeps
    return t


def _dicts(m4):
    rank = {(int(l), int(r)): int(k) for k, l, r, _ in m4}
    merged = {(int(l), int(r)): int(m) for _, l, r, m in m4}
    return rank, merged


def _random_table(rng, alphabet, merges, consistent, self_pairs=0.3):
    toks = {i: bytes([97 + i]) for i in range(alphabet)}
    words, used, ms, nid = set(toks.values()), set(), [], alphabet
    for _ in range(merges * 6):
        if len(ms) >= merges:
            break
        pool = list(toks)
        l = rng.choice(pool)
        r = l if rng.random() < self_pairs else rng.choice(pool)
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
    return np.array([(order[k],) + ms[k] for k in range(len(ms))], np.uint32).reshape(-1, 4)


@pytest.mark.parametrize("consistent", [True, False])
def test_superpass_equals_block_engine_on_random_tables(consistent):
    rng = random.Random(11 if consistent else 12)
    for trial in range(150):
        A = rng.randrange(1, 5)
        m4 = _random_table(rng, A, rng.randrange(1, 40), consistent)
        if m4.shape[0] == 0:
            continue
        orc = CRestatement(m4, list(range(A)) + [0xFFFFFFFF] * (256 - A))
        rank, merged = _dicts(m4)
        for _ in range(15):
            s = []
            while len(s) < rng.randrange(0, 150):
                s += [rng.randrange(A)] * rng.randrange(1, 9)  # runs of repeated tokens
            assert superpass_bpe(s, rank, merged) == orc.block_bpe(s), (trial, s, m4.tolist())


def test_superpass_inconsistent_kat():
    # (ab, a) -> aba at rank 0, (a, b) -> ab at rank 1; block gives [ab, ab]
    m4 = np.array([[0, 3, 0, 4], [1, 0, 1, 3]], np.uint32)
    rank, merged = _dicts(m4)
    assert superpass_bpe([0, 1, 0, 1], rank, merged) == [3, 3]
    orc = CRestatement(m4, [0, 1] + [0xFFFFFFFF] * 254)
    for s in ([0, 1, 0, 1, 0], [0, 1] * 7, [0, 0, 1, 0, 1, 1, 0, 1]):
        assert superpass_bpe(s, rank, merged) == orc.block_bpe(s)


def test_superpass_gpt2_rows_and_adversarial(gpt2):
    _, _, _, m4 = gpt2.export()
    bt = [gpt2.byte_token(b) for b in range(256)]
    orc = CRestatement(m4, bt)
    rank, merged = _dicts(m4)
    rng = random.Random(3)
    corpus = open(__file__.replace("test_superpass.py", "golden/corpus.txt"), "rb").read()
    rows = [corpus[:3000], b"a" * 2000, b"." * 1500, b"0" * 999,
            bytes(rng.randrange(48, 58) for _ in range(2048)), bytes(rng.randrange(256) for _ in range(1024))]
    passes = sweeps = 0
    for row in rows:
        t0 = [bt[b] for b in row]
        want, tr = orc.block_bpe(t0, trace=True)
        st = {}
        assert superpass_bpe(t0, rank, merged, st) == want
        passes += len(tr)
        sweeps += st.get("sweeps", 0)
    assert sweeps * 10 < passes  # the point of the rule: far fewer sequential steps
