"""CPU check of the exactness argument behind the piece decomposition
(DESIGN.md "Piece decomposition"), using the oracle's block_bpe:

  block_bpe(row) == concat(block_bpe(piece) for piece in pieces(row))

where pieces are cut at every byte position whose bigram is not the junction
(last byte of left, first byte of right) of any merge. This is what licenses
the GPU's lane-per-piece tier; the property is checked on the GPT-2 table, on
training-consistent random tables and on the inconsistent table of SURVEY
Appendix A (the decomposition does not need rank consistency)."""
import zlib

import numpy as np
import pytest

from conftest import arrays_from_json


def junction_set(ids, off, blob, m4):
    first, last = {}, {}
    for k, i in enumerate(ids):
        b = bytes(blob[int(off[k]):int(off[k + 1])])
        if b:
            first[int(i)], last[int(i)] = b[0], b[-1]
    J = np.zeros((256, 256), bool)
    for _, l, r, _ in m4:
        if int(l) in last and int(r) in first:
            J[last[int(l)], first[int(r)]] = True
    return J


def pieces(s: bytes, J):
    if not s:
        return []
    cuts = [0] + [p for p in range(1, len(s)) if not J[s[p - 1], s[p]]] + [len(s)]
    return [s[a:b] for a, b in zip(cuts, cuts[1:])]


def check(orc, J, s):
    whole = orc.block_bpe(orc.initial(s))
    parts = []
    for p in pieces(s, J):
        parts += orc.block_bpe(orc.initial(p))
    assert parts == whole, s


def test_gpt2_decomposition(gpt2, oracle_for):
    J = junction_set(*gpt2.export())
    assert J.sum() == gpt2.info()["junction_bigrams"] == 2689
    orc = oracle_for("gpt2")
    rng = np.random.default_rng(5)
    for _ in range(300):
        check(orc, J, bytes(rng.integers(0, 256, rng.integers(0, 200)).astype(np.uint8)))
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    text = gen.stream(1 << 15, seed=9).tobytes()
    for i in range(0, len(text), 1024):
        check(orc, J, text[i:i + 1024])
    for s in [b"a" * 300, b"." * 257, b"0123456789" * 30, b" " * 100 + b"x", b"\n\n\n  \t\t"]:
        check(orc, J, s)


@pytest.mark.parametrize("name", ["toy8", "inconsistent", "doubling"] + [f"random{k}" for k in range(20)])
def test_toy_decomposition(name, toy_tables, oracle_for):
    arrs = arrays_from_json(toy_tables[name])
    J = junction_set(*arrs)
    orc = oracle_for(name)
    alphabet = np.frombuffer(b"abcd", np.uint8)
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    for _ in range(300):
        s = bytes(rng.choice(alphabet, rng.integers(0, 40)))
        if any(orc.byte_tokens[b] == 0xFFFFFFFF for b in s):
            continue
        check(orc, J, s)
