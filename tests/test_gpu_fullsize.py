"""Bit-exactness at FULL BASELINE.json sizes (north_star: "bit-exact ... on
every config"): every row of cfg2, cfg3, cfg4 (128k and 200k merges) and a
2 GB shard of the cfg5 corpus, against the compiled reference (oracle/_ref).
Like the reference bench's correctness gate (bench.hpp:328-353): the block
engine's encode_batch (the drop-in target) on every row where it fits the
time budget, else heap_bpe on every row (identical on these rank-consistent
tables; rows where heap differs are re-decided by the block engine) plus the
block engine on a deterministic row sample (bench.parity_check)."""
import os

import numpy as np
import pytest

import paper_2507_11941_b200 as bb
from oracle.oracle import Reference

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not Reference.available(), reason="oracle/_ref not built")]


def _encode(table, data, off):
    torch = pytest.importorskip("torch")
    enc = bb.Encoder(device=0)
    n, total = off.size - 1, int(off[-1])
    d = torch.from_numpy(data).cuda()
    o = torch.from_numpy(off.view(np.int64)).cuda()
    ids = torch.empty(max(total, 1), dtype=torch.int32, device="cuda")
    oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    enc.encode_device(table, d.data_ptr(), o.data_ptr(), n, total, ids.data_ptr(), oo.data_ptr(), sync=True)
    oo = oo.cpu().numpy().view(np.uint64)
    res = ids[: int(oo[-1])].cpu().numpy().view(np.uint32), oo, enc.piece_stats()
    del d, o, ids
    torch.cuda.empty_cache()
    return res


def _check(ref, table, data, off, budget=60.0):
    import bench
    ids, oo, st = _encode(table, data, off)
    par = bench.parity_check(ref, data, off, ids, oo, budget)
    assert par["rows_checked"] == off.size - 1
    assert par["mismatches"] == 0, par
    return par, st


@pytest.fixture(scope="module")
def gpt2_ref():
    from workloads import tables as WT
    return Reference.load_files(WT.GPT2_VOCAB, WT.GPT2_MERGES)


@pytest.fixture(scope="module")
def gen():
    from workloads import tables as WT, text as WX
    return WX.TextGen(WX.word_list(WT.gpt2_table()[0]))


def test_cfg2_every_row_vs_block_engine(gpt2, gpt2_ref, gen):
    from workloads import text as WX
    data, off, _ = WX.config_rows(gen, 2)
    par, st = _check(gpt2_ref, gpt2, data, off, budget=120.0)
    assert "block engine" in par["oracle"] and par["tokens_checked"] > 60e6
    # piece statistics of the encode (bbpe_ctx_piece_stats)
    assert st["input_bytes"] == int(off[-1]) and st["pieces"] > 0.15 * int(off[-1])
    assert 0.8 < st["memo_hit_rate"] < 1.0 and st["long_pieces"] == 0


def test_cfg3_full_size(gpt2, gpt2_ref, gen):
    from workloads import text as WX
    data, off, _ = WX.config_rows(gen, 3)
    assert off.size - 1 == 16384 and int(off[-1]) > 5.5e8
    _check(gpt2_ref, gpt2, data, off)


@pytest.mark.parametrize("merges", [128000, 200000])
def test_cfg4_full_size_wordlevel_tables(merges, tmp_path):
    from workloads import tables as WT, text as WX
    tokens, m = WT.extend_wordlevel(*WT.gpt2_table(), 200000)
    m = [x for x in m if x[0] < merges]
    path = WT.write_canonical(str(tmp_path / "t.json"), tokens, m)
    table = bb.load_merge_table_files(path, None, "json")
    ref = Reference.load_files(path, None, canonical=True)
    data, off, _ = WX.config_rows(WX.TextGen(WX.word_list(tokens)), 4)
    assert off.size - 1 == 65536
    _check(ref, table, data, off)


@pytest.mark.parametrize("merges", [128000, 200000])
def test_cfg4_full_size_trained_tables(merges, tmp_path):
    """SURVEY §8d's cfg4 table: GPT-2 continued by BPE training without
    pre-tokenization (cross-word merges: rows become long pieces)."""
    from workloads import tables as WT, text as WX, train
    tokens, m, _ = train.trained_table(*WT.gpt2_table(), merges)
    path = WT.write_canonical(str(tmp_path / "t.json"), tokens, m)
    table = bb.load_merge_table_files(path, None, "json")
    ref = Reference.load_files(path, None, canonical=True)
    data, off, _ = WX.config_rows(WX.TextGen(WX.word_list(WT.gpt2_table()[0])), 4)
    assert off.size - 1 == 65536
    par, st = _check(ref, table, data, off)
    assert st["long_pieces"] > 0


def test_cfg5_2gb_shard(gpt2, gpt2_ref, gen):
    """Shard 1 of 8 of the one 16 GB cfg5 corpus (cost-balanced bounds from the
    encoder's partitioner): ~2 GB, bit-exact on every row."""
    from workloads import text as WX
    rng = np.random.default_rng(1005)
    L = WX.cfg5_lengths(1.0, rng)
    corpus = np.zeros(L.size + 1, np.uint64)
    np.cumsum(L.astype(np.uint64), out=corpus[1:])
    bounds = bb.partition(corpus, 8).astype(np.int64)
    data, off, desc, (r0, r1), _ = WX.cfg5_shard(gen, 1.0, 8, 1, bounds=bounds)
    assert int(off[-1]) > 1.5e9
    _check(gpt2_ref, gpt2, data, off)


@pytest.mark.parametrize("text", ["corpus", "mixed"])
def test_other_text_classes_cfg2(text, gpt2, gpt2_ref):
    """The reference bench's corpus.txt rows and the mixed class (random-letter
    words, numbers, hex, code, CJK, Cyrillic) at cfg2 size."""
    from workloads import text as WX
    corpus = open(os.path.join(os.path.dirname(__file__), "golden", "corpus.txt"), "rb").read()
    data, off, _ = WX.config_rows(WX.make_gen(text, None, corpus), 2, scale=1 / 4)
    _check(gpt2_ref, gpt2, data, off)


def test_device_jsonl_equals_reference_writer(gpt2, gpt2_ref, gen):
    """The device JSON-lines writer against the reference's own
    write_batch_jsonl (batch.hpp:157-166, via oracle/_ref) on 20k rows with
    empty and long rows mixed in."""
    torch = pytest.importorskip("torch")
    from workloads import text as WX
    d0, o0 = WX.rows_lengths(gen, np.random.default_rng(8).integers(0, 3000, 20000), seed=8)
    ids, oo, _ = _encode(gpt2, d0, o0)
    enc = bb.Encoder(device=0)
    d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
    d_oo = torch.from_numpy(oo.view(np.int64)).cuda()
    cap = enc.jsonl_device(d_ids.data_ptr(), d_oo.data_ptr(), oo.size - 1, ids.size, 0, 0)
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    assert enc.jsonl_device(d_ids.data_ptr(), d_oo.data_ptr(), oo.size - 1, ids.size, out.data_ptr(), cap) == cap
    want = gpt2_ref.write_batch(d0, o0, pad_id=0, binary=False, workers=os.cpu_count() or 1)
    assert out.cpu().numpy().tobytes() == want
