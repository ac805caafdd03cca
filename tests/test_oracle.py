"""The CPU oracle (oracle/bpe_oracle.c) pinned against the reference's golden
vectors and traces (tests/golden, generated from the unmodified reference by
tests/golden/make_golden.py), plus the reference tests' engine-equivalence and
pass-semantics properties (test_block_engine.cpp, acceptance_test.cpp)."""
import itertools
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, VECTOR_SETS, load_vectors


@pytest.mark.parametrize("name", VECTOR_SETS)
def test_oracle_matches_reference_vectors(name, oracle_for):
    v = load_vectors(name)
    orc = oracle_for(str(v["table"]))
    ids, off = orc.encode_packed(v["data"], v["offsets"])
    assert np.array_equal(off, v["out_offsets"])
    assert np.array_equal(ids, v["ids"])


def test_oracle_kats(oracle_for):
    with open(os.path.join(GOLDEN, "kats.json")) as f:
        kats = json.load(f)
    orc = oracle_for("gpt2")
    for s, want in kats["gpt2"]:
        assert orc.block_bpe(orc.initial(s.encode())) == want, s


def test_oracle_traces(oracle_for):
    with open(os.path.join(GOLDEN, "traces.json")) as f:
        tr = json.load(f)
    for fam, name in (("doubling", "doubling"), ("gpt2", "gpt2")):
        orc = oracle_for(name)
        for case in tr[fam]:
            out, trace = orc.block_bpe(case["tokens"], trace=True)
            assert out == case["out"]
            assert [(p, r, m) for p, r, m in trace] == [tuple(t) for t in case["trace"]]
    mp = tr["max_passes"]
    kind, partial, passes = oracle_for("doubling").block_bpe(mp["tokens"], max_passes=mp["max_passes"])
    assert kind == "max_passes" and partial == mp["partial"] and passes == mp["passes"]
    assert partial == [5, 5, 5, 5]  # test_block_engine.cpp:384-399


def test_block_equals_heap_equals_naive_on_consistent_tables(oracle_for):
    # acceptance_test.cpp:39-77 (exhaustive <= 6 on toy8) -- here <= 5 to keep it fast.
    orc = oracle_for("toy8")
    for L in range(0, 6):
        for p in itertools.product(b"abcd", repeat=L):
            t = orc.initial(bytes(p))
            b = orc.block_bpe(t)
            assert b == orc.naive_bpe(t) == orc.heap_bpe(t), bytes(p)
    g = oracle_for("gpt2")
    rng = np.random.default_rng(1001)
    for _ in range(300):
        s = bytes(rng.integers(0, 256, rng.integers(0, 257)).astype(np.uint8))
        t = g.initial(s)
        assert g.block_bpe(t) == g.heap_bpe(t) == g.naive_bpe(t)


def test_inconsistent_table_block_semantics(oracle_for):
    # block [ab, ab] vs naive/heap [aba, b] on "abab".
    orc = oracle_for("inconsistent")
    t = orc.initial(b"abab")
    assert orc.block_bpe(t) == [2, 2]
    assert orc.naive_bpe(t) == [3, 1] == orc.heap_bpe(t)


def test_per_pass_invariants(oracle_for):
    # test_block_engine.cpp:321-338
    g = oracle_for("gpt2")
    rng = np.random.default_rng(71)
    for _ in range(100):
        s = bytes(rng.integers(0, 256, rng.integers(0, 151)).astype(np.uint8))
        t = g.initial(s)
        out, trace = g.block_bpe(t, trace=True)
        total = 0
        for k, (p, r, m) in enumerate(trace):
            assert m >= 1
            total += m
            if k:
                assert trace[k - 1][1] < r
        assert len(t) - len(out) == total
        assert len(trace) <= len(t)
