"""Host-side pieces of the drop-in (no GPU): specials splitting, batch
serialisation, synthetic data determinism (pretokenize.hpp:32-57,
merge_table.hpp:309-385, batch.hpp:159-242)."""
import numpy as np
import pytest

import paper_2507_11941_b200 as bb
from workloads import text as synth


def specials():
    s = bb.SpecialTokenSet()
    s.add("<eos>", 9)
    s.add("<e>", 8)
    return s


def test_split_specials_longest_first():
    segs = bb.split_specials(b"hi<eos>x<e><eos>", specials())
    assert [(s.kind, s.bytes, s.special_id) for s in segs] == [
        ("literal", b"hi", None), ("special", b"<eos>", 9), ("literal", b"x", None), ("special", b"<e>", 8),
        ("special", b"<eos>", 9)]
    assert bb.split_specials(b"", specials()) == []
    assert b"".join(s.bytes for s in bb.split_specials(b"a<eos>b", specials())) == b"a<eos>b"


def test_special_set_errors():
    s = specials()
    with pytest.raises(bb.UsageError):
        s.add("<eos>", 3)
    with pytest.raises(bb.UsageError):
        s.add("", 3)
    with pytest.raises(bb.UsageError):
        s.set_bos("<nope>")
    s.set_bos("<e>")
    assert s.bos_id() == 8 and s.eos_id() is None


def test_validate_specials(gpt2):
    s = bb.SpecialTokenSet()
    s.add("<|endoftext|>", 50256)
    bb.validate_specials(gpt2, s)
    s2 = bb.SpecialTokenSet()
    s2.add("x", gpt2.byte_token(ord("x")))
    with pytest.raises(bb.IntegrityError, match="base byte token"):
        bb.validate_specials(gpt2, s2)
    s3 = bb.SpecialTokenSet()
    s3.add("<m>", 256)
    with pytest.raises(bb.IntegrityError, match="merge-derived"):
        bb.validate_specials(gpt2, s3)


def make_encoding():
    e = bb.BatchEncoding(batch_size=3, max_len=2, pad_id=99)
    e.ids = np.array([4, 99, 3, 3, 99, 99], np.uint32)
    e.lengths = np.array([1, 2, 0], np.uint32)
    e.mask = np.array([1, 0, 1, 1, 0, 0], np.uint8)
    return e


def test_jsonl_round_trip():
    text = bb.write_batch_jsonl(make_encoding())
    assert text.split("\n")[1] == '{"ids":[3,3],"len":2}'
    assert bb.read_jsonl_token_seqs(text, "t") == [[4], [3, 3], []]
    with pytest.raises(bb.ParseError, match="rows.jsonl:2"):
        bb.read_jsonl_token_seqs('{"ids":[1]}\nnot json\n', "rows.jsonl")


def test_binary_round_trip():
    e = make_encoding()
    blob = bb.write_batch_binary(e)
    assert blob[:4] == b"BBPE" and len(blob) == 16 + 4 * 6
    back = bb.read_batch_binary(blob, "t")
    assert back.batch_size == 3 and back.max_len == 2 and back.pad_id == 99
    assert back.lengths.tolist() == [1, 2, 0]
    with pytest.raises(bb.ParseError):
        bb.read_batch_binary(b"NOPE....", "t")


def test_pack_rows():
    d, o = bb.pack_rows([b"ab", "", b"c"])
    assert d.tobytes() == b"abc" and o.tolist() == [0, 2, 2, 3]


def test_synth_is_deterministic(gpt2):
    gen = synth.TextGen(synth.word_list(gpt2))
    a = gen.stream(10000, 5)
    b = synth.TextGen(synth.word_list(gpt2)).stream(10000, 5)
    assert np.array_equal(a, b) and a.max() < 128
    d, o, desc = synth.config_rows(gen, 2, scale=1 / 4096)
    assert o[-1] == d.size == 256 * (o.size - 1)
    d3, o3, _ = synth.config_rows(gen, 3, scale=1 / 4096)
    L = np.diff(o3.astype(np.int64))
    assert L.min() >= 8192 and L.max() <= 65536
