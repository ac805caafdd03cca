"""Spec-level operations on the device (block_engine.hpp:189-256), mirroring
the reference's own tests (tests/test_block_engine.cpp:27-112) case by case,
plus a pass-by-pass replay equal to block_bpe and the oracle."""
import random

import pytest

import paper_2507_11941_b200 as bb
from conftest import table_from_json

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def toy(toy_tables):
    return table_from_json(toy_tables["toy"])


@pytest.fixture(scope="module")
def toy8(toy_tables):
    return table_from_json(toy_tables["toy8"])


def test_pair_ranks_toy(toy):  # test_block_engine.cpp:27-32
    assert bb.pair_ranks([0, 1, 2], toy) == [0, None]
    assert bb.pair_ranks([2, 2, 2], toy) == [None, None]
    assert bb.pair_ranks([], toy) == []


def test_single_token_and_empty(toy):
    assert bb.pair_ranks([3], toy) == []
    assert bb.mark_merges([3], toy, 0) == [0]
    assert bb.mark_merges([], toy, 0) == []
    assert bb.exclusive_scan([0]) == [0]
    assert bb.compact([3], toy, [0], [0]) == [3]
    assert bb.compact([], toy, [], []) == []
    assert bb.block_bpe_replay([], toy) == [] and bb.block_bpe_replay([2], toy) == [2]


def test_min_rank_reduce():  # :34-41
    assert bb.min_rank_reduce([5, None, 2]) == 2
    assert bb.min_rank_reduce([None, None]) is None
    assert bb.min_rank_reduce([2, 5, None]) == 2
    assert bb.min_rank_reduce([None, 2, 5]) == 2
    assert bb.min_rank_reduce([]) is None


def test_mark_merges(toy, toy8):  # :43-59
    assert bb.mark_merges([0, 1, 0, 1], toy, 0) == [0, 1, 0, 1]
    assert bb.mark_merges([0, 0, 0], toy8, 7) == [0, 1, 0]
    assert bb.mark_merges([0, 0, 0, 0], toy8, 7) == [0, 1, 0, 1]
    assert bb.mark_merges([0, 0, 0, 0, 0], toy8, 7) == [0, 1, 0, 1, 0]
    assert bb.mark_merges([0, 1, 2], toy, 0) == [0, 1, 0]


def test_mark_merges_no_adjacent_flags(toy8):  # :61-76
    rng = random.Random(41)
    for _ in range(100):
        inp = [rng.randrange(4) for _ in range(rng.randrange(20))]
        m = bb.min_rank_reduce(bb.pair_ranks(inp, toy8))
        if m is None:
            continue
        f = bb.mark_merges(inp, toy8, m)
        assert len(f) == len(inp) and (not f or f[0] == 0)
        assert not any(f[i - 1] and f[i] for i in range(1, len(f)))


def test_exclusive_scan():  # :78-87
    assert bb.exclusive_scan([0, 1, 0, 1]) == [0, 0, 1, 1]
    assert bb.exclusive_scan([0, 0, 0]) == [0, 0, 0]
    assert bb.exclusive_scan([]) == []
    with pytest.raises(bb.ContractViolation, match="adjacent merge flags at indices 1 and 2"):
        bb.exclusive_scan([0, 1, 1])
    with pytest.raises(bb.ContractViolation, match="merge flags must be 0/1, got 2 at index 1"):
        bb.exclusive_scan([0, 2, 0])
    big = [0, 1] * 3000
    assert bb.exclusive_scan(big) == [i // 2 for i in range(6000)]  # carries across 1024-element chunks


def test_compact(toy, toy8):  # :89-112
    assert bb.compact([0, 1, 0, 1], toy, [0, 1, 0, 1], [0, 0, 1, 1]) == [3, 3]
    assert bb.compact([0, 1, 2], toy, [0, 1, 0], [0, 0, 1]) == [3, 2]
    assert bb.compact([0, 1, 2], toy, [0, 0, 0], [0, 0, 0]) == [0, 1, 2]
    with pytest.raises(bb.ContractViolation, match="offsets are not the exclusive scan of flags at index 2"):
        bb.compact([0, 1, 2], toy, [0, 1, 0], [0, 0, 0])
    with pytest.raises(bb.ContractViolation, match="flags/offsets length does not match token count"):
        bb.compact([0, 1, 2], toy, [0, 1, 0], [0, 0])
    # compact_into (block_engine.hpp:174-176): (2, 2) is not a merge pair
    with pytest.raises(bb.ContractViolation, match="flags mark a pair that is not in the merge table at index 0"):
        bb.compact([2, 2], toy, [0, 1], [0, 0])
    assert bb.compact([3, 2, 3], toy8, [0, 0, 0], [0, 0, 0]) == [3, 2, 3]
    assert bb.compact([0, 0, 3, 2], toy8, [0, 1, 0, 0], [0, 0, 1, 1]) == [11, 3, 2]


def test_replay_equals_block_bpe_and_oracle(gpt2, oracle_for):
    """The pass loop driven through the device spec ops equals bbpe_block_bpe
    (and its PassTrace) and the oracle, on GPT-2 text and an adversarial run."""
    orc = oracle_for("gpt2")
    rows = [b"The quick brown fox jumps over the lazy dog, 12345 times!", b"a" * 300, b"0123456789" * 20,
            bytes(range(200))]
    for row in rows:
        t0 = orc.initial(row)
        tr = []
        got = bb.block_bpe_replay(t0, gpt2, trace=tr)
        want, want_tr = orc.block_bpe(t0, trace=True)
        assert got == want
        assert tr == want_tr
        tr2 = []
        assert bb.block_bpe(t0, gpt2, bb.BlockConfig(), trace=tr2) == want and tr2 == want_tr
