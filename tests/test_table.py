"""Table loading and validation (merge_table.hpp) through the C-ABI: the
reference's formats, error types and messages, and the device layout the
host builds (dense ids/ranks, junction bigrams). CPU only."""
import json
import os

import numpy as np
import pytest

import paper_2507_11941_b200 as bb
from conftest import extend_table, GOLDEN, arrays_from_json, table_from_json

REF_GPT2 = "/root/reference/proj/tests/testdata/gpt2/"


def test_gpt2_fixture(gpt2):
    info = gpt2.info()
    assert info["token_count"] == 50257 and info["merge_count"] == 50000 and info["base_size"] == 256
    assert info["rank_consistent"] == 1 and info["remapped_ids"] == 0 and info["junction_bigrams"] == 2689
    # test_vocab.cpp:158-167 spot ids
    assert gpt2.bytes_of(13) == b"." and gpt2.bytes_of(995) == b" world"
    assert gpt2.rank_of(220, 83) == 0 and gpt2.merged_of(220, 83) == 256
    assert gpt2.rank_of(83, 220) is None
    assert all(gpt2.byte_token(b) != 0xFFFFFFFF for b in range(256))


@pytest.mark.skipif(not os.path.exists(REF_GPT2), reason="reference tree not present")
def test_gpt2_text_format_loader_matches_fixture(gpt2):
    t = bb.load_merge_table_files(REF_GPT2 + "vocab.json", REF_GPT2 + "merges.txt", "gpt2")
    for x, y in zip(t.export(), gpt2.export()):
        assert np.array_equal(x, y)


def test_binary_header_sizes_checked_before_allocation(tmp_path):
    """A .bbpt header announcing more payload than the file holds is a
    ParseError ('truncated'), not a multi-GB allocation."""
    import struct
    p = str(tmp_path / "bad.bbpt")
    with open(p, "wb") as f:
        f.write(b"BBPT" + struct.pack("<IQQQ", 1, 1 << 31, 1 << 35, 1 << 31) + b"\0" * 64)
    with pytest.raises(bb.ParseError, match="truncated"):
        bb.load_merge_table_files(p, None, "binary")


def test_binary_round_trip(tmp_path, gpt2):
    p = str(tmp_path / "t.bbpt")
    gpt2.save_binary(p)
    t = bb.load_merge_table_files(p, None, "binary")
    for x, y in zip(t.export(), gpt2.export()):
        assert np.array_equal(x, y)


def test_canonical_json_loader(tmp_path, toy_tables):
    for name in ("toy", "toy8", "doubling"):
        p = tmp_path / f"{name}.json"
        p.write_text(json.dumps(toy_tables[name]))
        t = bb.load_merge_table_files(str(p), None, "json")
        for x, y in zip(t.export(), table_from_json(toy_tables[name]).export()):
            assert np.array_equal(x, y)


def test_parse_errors(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    with pytest.raises(bb.ParseError):
        bb.load_merge_table_files(str(bad), None, "json")
    with pytest.raises(bb.UsageError):
        bb.load_merge_table_files(str(tmp_path / "missing.json"), None, "json")
    with pytest.raises(bb.UsageError):
        bb.parse_vocab_format("yaml")
    v = tmp_path / "vocab.json"
    v.write_text(json.dumps({"a": 0, "b": 1, "ab": 2}))
    m = tmp_path / "merges.txt"
    m.write_text("#version: 0.2\na b\nb c\n")
    with pytest.raises(bb.ParseError, match="merges.txt:3"):
        bb.load_merge_table_files(str(v), str(m), "gpt2")
    m.write_text("a  b\n")
    with pytest.raises(bb.ParseError, match='expected exactly "left right"'):
        bb.load_merge_table_files(str(v), str(m), "gpt2")
    m.write_text("b a\n")
    with pytest.raises(bb.IntegrityError, match="not in vocab"):
        bb.load_merge_table_files(str(v), str(m), "gpt2")


def test_integrity_errors():
    # add_token / add_merge / finalize checks (merge_table.hpp:257-297)
    with pytest.raises(bb.IntegrityError, match="duplicate token id 0"):
        bb.MergeTable.build([(0, b"a"), (0, b"b")], [])
    with pytest.raises(bb.IntegrityError, match="duplicate merge rank 0"):
        bb.MergeTable.build([(0, b"a"), (1, b"b"), (2, b"ab"), (3, b"ba")], [(0, 0, 1, 2), (0, 1, 0, 3)])
    with pytest.raises(bb.IntegrityError, match=r"duplicate merge pair \(0, 1\)"):
        bb.MergeTable.build([(0, b"a"), (1, b"b"), (2, b"ab")], [(0, 0, 1, 2), (1, 0, 1, 2)])
    with pytest.raises(bb.IntegrityError, match="two tokens share byte value 97"):
        bb.MergeTable.build([(0, b"a"), (1, b"a")], [])
    with pytest.raises(bb.IntegrityError, match="references unknown token id"):
        bb.MergeTable.build([(0, b"a"), (1, b"b")], [(0, 0, 1, 7)])
    with pytest.raises(bb.IntegrityError, match="merged token bytes mismatch"):
        bb.MergeTable.build([(0, b"a"), (1, b"b"), (2, b"ba")], [(0, 0, 1, 2)])


def test_sparse_ranks_and_huge_ids_are_remapped():
    # Canonical tables may use any unique u32 ranks and ids (merge_table.hpp:492-493).
    big = 4_000_000_000
    t = bb.MergeTable.build([(big, b"a"), (big + 1, b"b"), (big + 7, b"ab")],
                            [(3_000_000_000, big, big + 1, big + 7)])
    info = t.info()
    assert info["remapped_ids"] == 1 and info["merge_count"] == 1
    assert t.rank_of(big, big + 1) == 3_000_000_000


def test_inconsistent_table_is_flagged(toy_tables):
    assert table_from_json(toy_tables["inconsistent"]).info()["rank_consistent"] == 0
    assert table_from_json(toy_tables["toy8"]).info()["rank_consistent"] == 1


def test_decode_and_unknown_ids(gpt2):
    sp = bb.SpecialTokenSet()
    sp.add("<|endoftext|>", 50256)
    assert bb.decode(gpt2, sp, [31373, 995]) == b"hello world"
    with pytest.raises(bb.DecodeError, match="unknown token id 60000 at index 1"):
        bb.decode(gpt2, sp, [31373, 60000])


def test_extended_large_tables(gpt2):
    from workloads import text as synth
    t, (ids, off, blob, m4) = extend_table(gpt2, 200000)
    info = t.info()
    assert info["merge_count"] == 200000 and info["rank_consistent"] == 1
    assert info["remapped_ids"] == 0 and info["id_bits"] == 18 and info["hash_slots"] == 2097152
    # regex-like: the junction set barely grows
    assert info["junction_bigrams"] < 3000
    t2, _ = extend_table(gpt2, 200000)
    assert np.array_equal(t2.export()[3], m4)  # deterministic


@pytest.fixture(scope="module")
def trained200k(tmp_path_factory):
    """GPT-2 continued by BPE training without
    pre-tokenization (workloads/train.py)."""
    from workloads import tables as WT, train
    toks, merges, how = train.trained_table(*WT.gpt2_table(), 200000)
    path = WT.write_canonical(str(tmp_path_factory.mktemp("tr") / "t.json"), toks, merges)
    return toks, merges, path


def test_trained_cfg4_table(trained200k):
    toks, merges, path = trained200k
    t = bb.load_merge_table_files(path, None, "json")
    info = t.info()
    assert info["merge_count"] == 200000
    # cross-word merges add junctions GPT-2 lacks (letter|punctuation, space), so
    # pieces span words (GPT-2 alone: 2,689 junction bigrams)
    assert info["junction_bigrams"] > 2689 + 200
    assert any(toks[m[3]].count(b" ") >= 2 for m in merges[50000:50100])
    for r, l, rr, m in merges[::997]:
        assert toks[m] == toks[l] + toks[rr]


def test_trained_cfg4_table_oracles_agree(trained200k):
    """The C restatement's block engine equals the compiled reference's
    encode_batch on rows of the cfg4 text under the trained table."""
    from oracle.oracle import CRestatement, Reference
    from workloads import text as WX
    toks, merges, path = trained200k
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    ref = Reference.load_files(path, None, canonical=True)
    data, off, _ = WX.config_rows(WX.TextGen(WX.word_list(toks)), 4, scale=1 / 2048)
    ri, ro = ref.encode_batch(data, off, workers=os.cpu_count() or 1)
    t = bb.load_merge_table_files(path, None, "json")
    _, _, _, m4 = t.export()
    orc = CRestatement(m4, [t.byte_token(b) for b in range(256)])
    ci, co = orc.encode_packed(data, off)
    assert np.array_equal(ro, co) and np.array_equal(ri, ci)
    # cross-word merges: far fewer tokens per byte than GPT-2 alone
    assert int(ro[-1]) < int(off[-1]) / 6
