"""GPU parity: the sm_100a path (through the C-ABI) against the reference's
golden vectors, the C oracle, and the reference tests' batch semantics
(test_batch.cpp, test_block_engine.cpp, acceptance_test.cpp)."""
import json
import os

import numpy as np
import pytest

import paper_2507_11941_b200 as bb
from conftest import extend_table, GOLDEN, VECTOR_SETS, load_vectors, table_from_json

pytestmark = pytest.mark.gpu

ENGINES = ["pieces", "nomemo", "block"]


def make_encoder(name, **kw):
    if name == "nomemo":
        return bb.Encoder(device=0, engine="pieces", piece_memo=False, **kw)
    return bb.Encoder(device=0, engine=name, **kw)


@pytest.fixture(scope="module")
def enc():
    return {e: make_encoder(e) for e in ENGINES}


@pytest.fixture(scope="module")
def tables(gpt2, toy_tables):
    t = {"gpt2": gpt2}
    for k, v in toy_tables.items():
        t[k] = table_from_json(v)
    return t


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("name", VECTOR_SETS)
def test_golden_vectors(name, engine, enc, tables):
    v = load_vectors(name)
    ids, off, st = enc[engine].encode_packed(tables[str(v["table"])], v["data"], v["offsets"])
    assert np.array_equal(off, v["out_offsets"])
    assert np.array_equal(ids, v["ids"])


def test_kats(enc, gpt2):
    with open(os.path.join(GOLDEN, "kats.json")) as f:
        kats = json.load(f)
    for e in ENGINES:
        rows = [s.encode() for s, _ in kats["gpt2"]]
        got = enc[e].encode_rows(gpt2, rows)
        assert got == [w for _, w in kats["gpt2"]]


def test_toy_canonical_kats(enc, tables):
    assert enc["pieces"].encode_rows(tables["toy"], [b"abc", b"ab"]) == [[4], [3]]


@pytest.mark.parametrize("engine", ENGINES)
def test_random_gpt2_vs_oracle(engine, enc, gpt2, oracle_for):
    rng = np.random.default_rng(2024)
    rows = [bytes(rng.integers(0, 256, rng.integers(0, 700)).astype(np.uint8)) for _ in range(500)]
    rows += [bytes(rng.choice(np.frombuffer(b"ab .0\n", np.uint8), rng.integers(0, 300))) for _ in range(300)]
    data, off = bb.pack_rows(rows)
    ids, oo, _ = enc[engine].encode_packed(gpt2, data, off)
    wi, wo = oracle_for("gpt2").encode_packed(data, off)
    assert np.array_equal(oo, wo) and np.array_equal(ids, wi)


def test_block_bpe_traces(enc, tables):
    with open(os.path.join(GOLDEN, "traces.json")) as f:
        tr = json.load(f)
    e = enc["block"]
    for fam in ("doubling", "gpt2"):
        for case in tr[fam]:
            out, trace = e.block_bpe(tables[fam], case["tokens"], trace=True)
            assert out == case["out"]
            assert [tuple(x) for x in trace] == [tuple(x) for x in case["trace"]]


def test_max_passes_partial_state(tables):
    with open(os.path.join(GOLDEN, "traces.json")) as f:
        mp = json.load(f)["max_passes"]
    e = bb.Encoder(device=0, config=bb.BlockConfig(256, mp["max_passes"]))
    with pytest.raises(bb.MaxPassesError) as ei:
        e.block_bpe(tables["doubling"], mp["tokens"])
    assert ei.value.partial_tokens == mp["partial"] == [5, 5, 5, 5]
    # Sufficient cap is silent (test_block_engine.cpp:401-405).
    assert e.block_bpe(tables["doubling"], [0, 1, 0, 1]) == [5]


def test_max_passes_in_batch_is_row_tagged_error(tables):
    e = bb.Encoder(device=0, config=bb.BlockConfig(256, 2))
    with pytest.raises(bb.Error) as ei:
        e.encode_rows(tables["doubling"], [b"ab", b"abab", b"ab" * 8])
    assert str(ei.value).startswith("row 2: block_bpe exceeded 2 merge passes")
    assert type(ei.value) is bb.Error  # encode_batch rethrows as plain Error


def test_row_error_names_row(enc, tables):
    # test_batch.cpp:85-94
    for e in ENGINES:
        with pytest.raises(bb.IntegrityError) as ei:
            enc[e].encode_rows(tables["toy"], [b"ab", b"ab", b"xyz"])
        assert "row 2" in str(ei.value)
        assert "byte value 120" in str(ei.value)


def test_empty_batches(enc, gpt2):
    for e in ENGINES:
        assert enc[e].encode_rows(gpt2, []) == []
        assert enc[e].encode_rows(gpt2, [b"", b"", b""]) == [[], [], []]
        assert enc[e].encode_rows(gpt2, [b"", b"hi", b""]) == [[], [5303], []]


def test_encode_batch_api(gpt2, tables):
    cfg = bb.BlockConfig(256, None)
    none = bb.SpecialTokenSet()
    toy = tables["toy"]
    enc = bb.encode_batch(["abc", "abab"], toy, none, cfg, 99, False, False)
    assert enc.max_len == 2 and enc.at(0, 0) == 4 and enc.at(0, 1) == 99
    assert enc.mask.tolist() == [1, 0, 1, 1]
    sp = bb.SpecialTokenSet()
    sp.add("<|endoftext|>", 50256)
    sp.set_bos("<|endoftext|>")
    sp.set_eos("<|endoftext|>")
    assert bb.encode_batch(["hi"], gpt2, sp, cfg, 50256, True, True).row(0) == [50256, 5303, 50256]
    assert bb.encode_single("hi<|endoftext|>", gpt2, sp, cfg) == [5303, 50256]
    lim = bb.encode_batch(["abcabc", "ab", "abcc"], toy, none, cfg, 99, False, False,
                          limits=bb.BatchLimits(1))
    assert lim.truncated_rows == 2 and lim.lengths.tolist() == [1, 1, 1]
    with pytest.raises(bb.UsageError):
        bb.encode_batch(["a"], toy, none, cfg, 0, True, False)
    with pytest.raises(bb.IntegrityError, match="row 2"):
        bb.encode_batch(["ab", "ab", "xyz"], toy, none, cfg, 99, False, False)
    inputs = ["hello world", "...."]
    e2 = bb.encode_batch(inputs, gpt2, sp, cfg, 50256, True, True)
    assert [d.decode() for d in bb.decode_batch(e2, gpt2, sp, True)] == inputs


def test_batch_independence_and_permutation(enc, gpt2):
    rng = np.random.default_rng(101)
    xs = [bytes(rng.integers(0, 256, 32).astype(np.uint8)) for _ in range(5)]
    ys = [bytes(rng.integers(0, 256, 32).astype(np.uint8)) for _ in range(7)]
    e = enc["pieces"]
    assert e.encode_rows(gpt2, xs + ys) == e.encode_rows(gpt2, xs) + e.encode_rows(gpt2, ys)
    perm = rng.permutation(12)
    both = xs + ys
    base = e.encode_rows(gpt2, both)
    assert e.encode_rows(gpt2, [both[i] for i in perm]) == [base[i] for i in perm]


def test_block_size_is_results_neutral(gpt2):
    rng = np.random.default_rng(53)
    rows = [bytes(rng.integers(0, 256, 200).astype(np.uint8)) for _ in range(50)]
    outs = []
    for bs in (32, 64, 256, 1024):
        for eng in ENGINES:
            outs.append(make_encoder(eng, config=bb.BlockConfig(bs, None)).encode_rows(gpt2, rows))
    assert all(o == outs[0] for o in outs)


def test_losslessness(enc, gpt2):
    rng = np.random.default_rng(73)
    rows = [bytes(rng.integers(0, 256, rng.integers(0, 129)).astype(np.uint8)) for _ in range(100)]
    for r, ids in zip(rows, enc["pieces"].encode_rows(gpt2, rows)):
        assert bb.decode(gpt2, bb.SpecialTokenSet(), ids) == r


def test_waves_match_single_pass(gpt2):
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off = synth.rows_fixed(gen, 3000, 256, seed=3)
    a = bb.Encoder(0).encode_packed(gpt2, data, off)
    b = bb.Encoder(0, wave_bytes=100_000).encode_packed(gpt2, data, off)
    assert b[2]["waves"] > 1
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_device_api_torch(gpt2):
    torch = pytest.importorskip("torch")
    v = load_vectors("gpt2_text")
    d = torch.from_numpy(v["data"]).cuda()
    o = torch.from_numpy(v["offsets"].astype(np.int64)).cuda()
    total = int(v["offsets"][-1])
    n = v["offsets"].size - 1
    out = torch.empty(total, dtype=torch.int32, device="cuda")
    oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    e = bb.Encoder(0)
    e.encode_device(gpt2, d.data_ptr(), o.data_ptr(), n, total, out.data_ptr(), oo.data_ptr(), sync=True)
    oo_h = oo.cpu().numpy().astype(np.uint64)
    assert np.array_equal(oo_h, v["out_offsets"])
    assert np.array_equal(out[: int(oo_h[-1])].cpu().numpy().astype(np.uint32), v["ids"])


def test_sharded_single_device_matches(gpt2):
    v = load_vectors("gpt2_random")
    encs = [bb.Encoder(0), bb.Encoder(0)]
    ids, oo, st = bb.encode_sharded(encs, gpt2, v["data"], v["offsets"])
    assert np.array_equal(oo, v["out_offsets"]) and np.array_equal(ids, v["ids"])


def test_sharded_edge_cases(gpt2):
    """Empty batch, empty rows only, fewer rows than contexts, one long row."""
    encs = [bb.Encoder(0) for _ in range(3)]
    for rows in ([], [b""], [b"", b"", b""], [b"hello"], [b"x" * 70000, b"", b"ab"]):
        data, off = bb.pack_rows(rows)
        want_ids, want_off, _ = bb.Encoder(0).encode_packed(gpt2, data, off)
        ids, oo, _ = bb.encode_sharded(encs, gpt2, data, off)
        assert np.array_equal(oo, want_off) and np.array_equal(ids, want_ids), rows[:2]


@pytest.mark.parametrize("n_ctx", [2, 3, 4])
def test_sharded_partitioned_path(gpt2, n_ctx):
    """bbpe_encode_sharded over n contexts on device 0 (the multi-GPU path
    with one GPU): cost-balanced shards, proportional output regions, the
    ordered parallel stitch (a 64 MiB batch so every move runs in waves), and
    the exact / too-small capacity cases; equal to the one-context encode."""
    from workloads import text as WX, tables as WT
    gen = WX.TextGen(WX.word_list(WT.gpt2_table()[0]))
    data, off, _ = WX.config_rows(gen, 2, scale=1 / 4)
    enc = bb.Encoder(0)
    want_ids, want_off, _ = enc.encode_packed(gpt2, data, off)
    encs = [bb.Encoder(0) for _ in range(n_ctx)]
    ids, oo, st = bb.encode_sharded(encs, gpt2, data, off)
    assert np.array_equal(oo, want_off) and np.array_equal(ids, want_ids)
    assert st["tokens"] == want_ids.size and st["n_rows"] == off.size - 1
    # capacity = the exact token count: regions are capacity shares (a shard
    # that overflows its share re-encodes into a host vector)
    ids2, oo2, _ = bb.encode_sharded(encs, gpt2, data, off, capacity=int(want_ids.size))
    assert np.array_equal(oo2, want_off) and np.array_equal(ids2, want_ids)
    ids3, oo3, _ = bb.encode_sharded(encs, gpt2, data, off, capacity=int(want_ids.size) + 1000)
    assert np.array_equal(oo3, want_off) and np.array_equal(ids3, want_ids)
    with pytest.raises(bb.UsageError, match="capacity"):
        bb.encode_sharded(encs, gpt2, data, off, capacity=int(want_ids.size) - 1)


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 1 / 128), (3, 1 / 512), (4, 1 / 256)])
def test_config_parity_vs_reference_engines(cfg, scale, gpt2, oracle_for):
    """BASELINE configs at sizes the C oracle's heap engine finishes quickly
    (heap == block on the training-consistent GPT-2 table)."""
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off, _ = synth.config_rows(gen, cfg, scale=scale)
    wi, wo = oracle_for("gpt2").encode_packed(data, off, engine=1)
    for name in ("pieces", "nomemo"):
        ids, oo, _ = make_encoder(name).encode_packed(gpt2, data, off)
        assert np.array_equal(oo, wo) and np.array_equal(ids, wi), name


def test_full_size_cfg2_properties(gpt2):
    """Full 2^20 x 256 B: round trip, determinism, and a random subsample vs the oracle."""
    from workloads import text as synth
    from oracle.oracle import CRestatement
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off, _ = synth.config_rows(gen, 2)
    e = bb.Encoder(0)
    ids, oo, _ = e.encode_packed(gpt2, data, off)
    ids2, oo2, _ = e.encode_packed(gpt2, data, off)
    assert np.array_equal(ids, ids2) and np.array_equal(oo, oo2)
    # Full-size round trip: decode(encode(x)) == x for all 256 MiB.
    tid, toff, tblob, _ = gpt2.export()
    start = np.zeros(int(tid.max()) + 1, np.int64)
    lens = np.zeros(int(tid.max()) + 1, np.int64)
    start[tid] = toff[:-1].astype(np.int64)
    lens[tid] = (toff[1:] - toff[:-1]).astype(np.int64)
    L = lens[ids]
    excl = np.zeros(ids.size, np.int64)
    np.cumsum(L[:-1], out=excl[1:])
    idx = np.repeat(start[ids] - excl, L) + np.arange(int(L.sum()), dtype=np.int64)
    assert np.array_equal(tblob[idx], data)
    # Row boundaries: every row's tokens decode to exactly its bytes.
    row_bytes = np.add.reduceat(L, oo[:-1].astype(np.int64))
    assert np.array_equal(row_bytes, np.diff(off).astype(np.int64))
    _, _, _, m4 = gpt2.export()
    orc = CRestatement(m4, [gpt2.byte_token(b) for b in range(256)])
    rng = np.random.default_rng(0)
    for r in rng.integers(0, off.size - 1, 200):
        s = data[int(off[r]):int(off[r + 1])].tobytes()
        assert ids[int(oo[r]):int(oo[r + 1])].tolist() == orc.heap_bpe(orc.initial(s))


@pytest.mark.parametrize("engine", ENGINES)
def test_remapped_ids_and_sparse_ranks(engine, toy_tables, oracle_for):
    """Canonical tables may use any unique u32 ids and ranks (merge_table.hpp:
    473-497); the device works on dense ids/ranks and maps back."""
    from oracle.oracle import CRestatement
    t = toy_tables["random3"]
    idmap = lambda i: 3_000_000_000 + 7919 * i
    toks = [(idmap(i), bytes(b)) for i, b in t["tokens"]]
    merges = [(10 * r + 5, idmap(l), idmap(rr), idmap(m)) for r, l, rr, m in t["merges"]]
    table = bb.MergeTable.build(toks, merges)
    assert table.info()["remapped_ids"] == 1
    bt = [0xFFFFFFFF] * 256
    for i, b in toks:
        if len(b) == 1:
            bt[b[0]] = i
    orc = CRestatement(np.array(merges, np.uint32), bt)
    rng = np.random.default_rng(5)
    rows = [bytes(rng.choice(np.frombuffer(b"abcd", np.uint8), rng.integers(0, 60))) for _ in range(300)]
    rows += [b"abcd" * 20, b"a" * 40]
    data, off = bb.pack_rows(rows)
    ids, oo, _ = make_encoder(engine).encode_packed(table, data, off)
    wi, wo = orc.encode_packed(data, off)
    assert np.array_equal(oo, wo) and np.array_equal(ids, wi)


@pytest.fixture(scope="module")
def big_tables(gpt2):
    from workloads import text as synth
    t200, arrs = extend_table(gpt2, 200000)
    ids, off, blob, m4 = arrs
    keep = m4[:, 0] < 128000
    t128 = bb.MergeTable.from_arrays(ids, off, blob, m4[keep])
    return {"200k": (t200, m4), "128k": (t128, m4[keep])}


@pytest.mark.parametrize("which", ["128k", "200k"])
@pytest.mark.parametrize("engine", ENGINES)
def test_large_vocab_cfg4_vs_oracle(which, engine, big_tables):
    """BASELINE config 4: 128k/200k-merge tables (wide ids, 4 MiB L2-resident
    hash), log-uniform 128 B-16 KiB rows, against the oracle's heap engine
    (identical to the block engine on these rank-consistent tables)."""
    from oracle.oracle import CRestatement
    from workloads import text as synth
    table, m4 = big_tables[which]
    assert table.info()["rank_consistent"] == 1
    gen = synth.TextGen(synth.word_list(table))
    data, off, _ = synth.config_rows(gen, 4, scale=1 / 512)
    orc = CRestatement(m4, [table.byte_token(b) for b in range(256)])
    wi, wo = orc.encode_packed(data, off, engine=1)
    ids, oo, _ = make_encoder(engine).encode_packed(table, data, off)
    assert np.array_equal(oo, wo) and np.array_equal(ids, wi)


def _pinned(a):
    torch = pytest.importorskip("torch")
    t = torch.from_numpy(a).pin_memory()
    return t, t.numpy()


@pytest.mark.parametrize("wave_bytes", [0, 50_000, 1 << 20])
def test_pinned_and_pageable_outputs_match(gpt2, wave_bytes):
    """Pinned outputs take the device-driven copy-out path (k_copy_out into
    the mapped buffer, no host round trip per wave); pageable outputs the
    host-paced path. Both equal the single-wave result and the oracle's."""
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off = synth.rows_fixed(gen, 6000, 256, seed=11)
    ref_ids, ref_off, _ = bb.Encoder(0).encode_packed(gpt2, data, off)
    e = bb.Encoder(0, wave_bytes=wave_bytes)
    ids_a, off_a, st_a = e.encode_packed(gpt2, data, off)  # pageable (numpy) outputs
    t_ids, h_ids = _pinned(np.zeros(data.size, np.uint32))
    t_off, h_off = _pinned(np.zeros(off.size, np.uint64))
    ids_b, off_b, st_b = e.encode_packed(gpt2, data, off, h_ids, h_off)
    assert np.array_equal(off_a, ref_off) and np.array_equal(ids_a, ref_ids)
    assert np.array_equal(off_b, ref_off) and np.array_equal(ids_b, ref_ids)
    if wave_bytes:
        assert st_b["waves"] > 1


def test_ramped_waves_and_odd_alignment(gpt2, oracle_for):
    """Ramped wave plan over rows of mixed length; the output buffer starts at
    an odd u32 offset so k_copy_out's aligning head/tail paths run."""
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 3000, 2500)
    data, off = synth.rows_lengths(gen, lens, seed=6)
    want_ids, want_off = oracle_for("gpt2").encode_packed(data, off)
    t_ids, h_ids = _pinned(np.zeros(data.size + 3, np.uint32))
    t_off, h_off = _pinned(np.zeros(off.size, np.uint64))
    e = bb.Encoder(0, wave_bytes=300_000)
    ids, oo, st = e.encode_packed(gpt2, data, off, h_ids[1:], h_off)
    assert st["waves"] > 4
    assert np.array_equal(oo, want_off) and np.array_equal(ids, want_ids)


@pytest.mark.parametrize("pinned", [False, True])
def test_output_capacity_too_small(gpt2, pinned):
    v = load_vectors("gpt2_text")
    n_tok = int(v["out_offsets"][-1])
    out = np.zeros(n_tok - 1, np.uint32)
    oo = np.zeros(v["offsets"].size, np.uint64)
    if pinned:
        _t1, out = _pinned(out)
        _t2, oo = _pinned(oo)
    with pytest.raises(bb.UsageError, match="capacity"):
        bb.Encoder(0).encode_packed(gpt2, v["data"], v["offsets"], out, oo)


def test_decreasing_offsets_rejected(gpt2):
    data = np.frombuffer(b"hello world, hello again", np.uint8).copy()
    off = np.array([0, 5, 3, 24], np.uint64)
    with pytest.raises(bb.UsageError, match="non-decreasing"):
        bb.Encoder(0).encode_packed(gpt2, data, off)
    torch = pytest.importorskip("torch")
    d = torch.from_numpy(data).cuda()
    o = torch.from_numpy(off.astype(np.int64)).cuda()
    out = torch.empty(24, dtype=torch.int32, device="cuda")
    oo = torch.empty(4, dtype=torch.int64, device="cuda")
    with pytest.raises(bb.UsageError, match="non-decreasing"):
        bb.Encoder(0).encode_device(gpt2, d.data_ptr(), o.data_ptr(), 3, 24, out.data_ptr(), oo.data_ptr(), sync=True)


def test_device_api_unaligned_input(gpt2):
    """Device input not 16-byte aligned: k_pieces loads its windows without
    cp.async; results unchanged."""
    torch = pytest.importorskip("torch")
    v = load_vectors("gpt2_text")
    total = int(v["offsets"][-1])
    n = v["offsets"].size - 1
    buf = torch.zeros(total + 16, dtype=torch.uint8, device="cuda")
    buf[3:3 + total] = torch.from_numpy(v["data"]).cuda()
    o = torch.from_numpy(v["offsets"].astype(np.int64)).cuda()
    out = torch.empty(total, dtype=torch.int32, device="cuda")
    oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    bb.Encoder(0).encode_device(gpt2, buf.data_ptr() + 3, o.data_ptr(), n, total, out.data_ptr(), oo.data_ptr(),
                                sync=True)
    oo_h = oo.cpu().numpy().astype(np.uint64)
    assert np.array_equal(oo_h, v["out_offsets"])
    assert np.array_equal(out[: int(oo_h[-1])].cpu().numpy().astype(np.uint32), v["ids"])


@pytest.mark.parametrize("memo", [True, False])
def test_dedupe_is_results_neutral(gpt2, oracle_for, memo):
    """Within-call dedupe of merge pieces (default) vs every piece merged on
    its own: identical ids/offsets, and equal to the oracle. Text with heavy
    repetition (numbers, capitalised words) and random bytes."""
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off = synth.rows_fixed(gen, 4000, 256, seed=21)
    rng = np.random.default_rng(22)
    rnd = rng.integers(0, 256, 200_000).astype(np.uint8)
    roff = np.arange(0, 200_001, 1000, dtype=np.uint64)
    for d, o in ((data, off), (rnd, roff)):
        a = bb.Encoder(0, piece_memo=memo, dedup=True).encode_packed(gpt2, d, o)
        b = bb.Encoder(0, piece_memo=memo, dedup=False).encode_packed(gpt2, d, o)
        want_ids, want_off = oracle_for("gpt2").encode_packed(d, o)
        assert np.array_equal(a[1], want_off) and np.array_equal(a[0], want_ids)
        assert np.array_equal(b[1], want_off) and np.array_equal(b[0], want_ids)


def test_device_decode_round_trip(gpt2):
    """Device decode inverts the device encode: lossless
    round trip (acceptance_test.cpp:111-129) on Zipf text, random bytes and
    empty rows; row byte offsets equal the input offsets."""
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off = synth.rows_fixed(gen, 3000, 256, seed=31)
    rng = np.random.default_rng(32)
    rnd = rng.integers(0, 256, 100_000).astype(np.uint8)
    roff = np.sort(np.concatenate([[0, 100_000], rng.integers(0, 100_000, 500)])).astype(np.uint64)
    enc = bb.Encoder(0)
    for d, o in ((data, off), (rnd, roff)):
        ids, oo, _ = enc.encode_packed(gpt2, d, o)
        b, bo = enc.decode_packed(gpt2, ids, oo)
        assert np.array_equal(bo, o - o[0])
        assert np.array_equal(b, d)


def test_device_decode_matches_host_decode_and_errors(gpt2):
    v = load_vectors("gpt2_text")
    enc = bb.Encoder(0)
    b, bo = enc.decode_packed(gpt2, v["ids"], v["out_offsets"])
    for r in range(0, v["out_offsets"].size - 1, 7):
        ids = v["ids"][int(v["out_offsets"][r]):int(v["out_offsets"][r + 1])]
        assert bytes(b[int(bo[r]):int(bo[r + 1])]) == bb.decode(gpt2, bb.SpecialTokenSet(), ids)
    # Unknown id: DecodeError naming the row and the index in the row (decode_batch).
    ids = np.array([31373, 995, 13, 99999999, 5], np.uint32)
    off = np.array([0, 2, 5], np.uint64)
    with pytest.raises(bb.DecodeError, match=r"row 1: unknown token id 99999999 at index 1"):
        enc.decode_packed(gpt2, ids, off)


def test_device_decode_device_api(gpt2):
    torch = pytest.importorskip("torch")
    v = load_vectors("gpt2_random")
    ids = torch.from_numpy(v["ids"].astype(np.int32)).cuda()
    off = torch.from_numpy(v["out_offsets"].astype(np.int64)).cuda()
    n = v["out_offsets"].size - 1
    cap = int(v["offsets"][-1])
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    tot = bb.Encoder(0).decode_device(gpt2, ids.data_ptr(), off.data_ptr(), n, int(v["ids"].size), out.data_ptr(),
                                      cap, oo.data_ptr())
    assert tot == cap
    assert np.array_equal(out.cpu().numpy(), v["data"])
    assert np.array_equal(oo.cpu().numpy().astype(np.uint64), v["offsets"])


@pytest.mark.parametrize("max_len", [None, 0, 1, 17, 64])
def test_device_epilogue_matches_host_padding(gpt2, max_len):
    """encode_batch's padded BatchEncoding built on the device
    equals the host padding of the same CSR (batch.hpp:98-125): widest or
    fixed max_len with right truncation, pad ids, lengths, mask, truncated
    row count; empty rows included."""
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    rng = np.random.default_rng(41)
    lens = rng.integers(0, 400, 700)
    lens[::50] = 0
    data, off = synth.rows_lengths(gen, lens, seed=42)
    rows = [bytes(data[int(off[i]):int(off[i + 1])]) for i in range(lens.size)]
    cfg = bb.BlockConfig(256, None)
    none = bb.SpecialTokenSet()
    lim = bb.BatchLimits(max_len) if max_len is not None else None
    d = bb.encode_batch(rows, gpt2, none, cfg, 7, limits=lim, device_epilogue=True)
    h = bb.encode_batch(rows, gpt2, none, cfg, 7, limits=lim, device_epilogue=False)
    assert d.max_len == h.max_len and d.truncated_rows == h.truncated_rows
    assert np.array_equal(d.lengths, h.lengths)
    assert np.array_equal(d.ids, h.ids) and np.array_equal(d.mask, h.mask)


def test_pad_device_bos_eos(gpt2):
    """bbpe_pad_device with BOS/EOS ids: [bos] + ids + [eos], truncation may
    cut the EOS (batch.hpp:76-79, 100-104)."""
    torch = pytest.importorskip("torch")
    import ctypes as C
    from paper_2507_11941_b200._lib import LIB
    ids = np.arange(1, 11, dtype=np.uint32)
    off = np.array([0, 3, 3, 10], np.uint64)
    d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    enc = bb.Encoder(0)
    w = C.c_uint64()
    assert LIB.bbpe_batch_widest_device(enc.handle, C.c_void_p(d_off.data_ptr()), 3, 1, 1, C.byref(w)) == 0
    assert w.value == 9
    for L in (9, 5):
        o = torch.empty(3 * L, dtype=torch.int32, device="cuda")
        m = torch.empty(3 * L, dtype=torch.uint8, device="cuda")
        ln = torch.empty(3, dtype=torch.int32, device="cuda")
        tr = C.c_uint64()
        assert LIB.bbpe_pad_device(enc.handle, C.c_void_p(d_ids.data_ptr()), C.c_void_p(d_off.data_ptr()), 3, 0,
                                   100, 200, L, C.c_void_p(o.data_ptr()), C.c_void_p(ln.data_ptr()),
                                   C.c_void_p(m.data_ptr()), C.byref(tr)) == 0
        want = [[100, 1, 2, 3, 200], [100, 200], [100, 4, 5, 6, 7, 8, 9, 10, 200]]
        want = [r[:L] + [0] * (L - len(r[:L])) for r in want]
        assert o.cpu().numpy().reshape(3, L).tolist() == want
        assert ln.cpu().numpy().tolist() == [min(5, L), 2, min(9, L)]
        assert tr.value == (1 if L == 5 else 0)
        assert m.cpu().numpy().reshape(3, L).sum(1).tolist() == [min(5, L), 2, min(9, L)]


@pytest.mark.parametrize("cfg", [3, 5])
def test_full_size_long_row_configs(gpt2, cfg):
    """BASELINE configs 3 (16,384 rows of 8-64 KiB, 604 MB) and 5 (log-uniform
    128 B-64 KiB, 1 GB here): full-size encode through the pipelined host API,
    device-resident encode agrees, device decode round trip is lossless, and
    sampled long rows equal the oracle (heap engine = block engine on GPT-2)."""
    torch = pytest.importorskip("torch")
    from oracle.oracle import CRestatement
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off, _ = synth.config_rows(gen, cfg, scale=1.0 if cfg == 3 else 1 / 16)
    e = bb.Encoder(0)
    ids, oo, st = e.encode_packed(gpt2, data, off)
    assert st["waves"] > 1
    n, total = off.size - 1, int(off[-1])
    d_data = torch.from_numpy(data).cuda()
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    d_ids = torch.empty(total, dtype=torch.int32, device="cuda")
    d_oo = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    e.encode_device(gpt2, d_data.data_ptr(), d_off.data_ptr(), n, total, d_ids.data_ptr(), d_oo.data_ptr(), sync=True)
    assert np.array_equal(d_oo.cpu().numpy().view(np.uint64), oo)
    assert torch.equal(d_ids[: int(oo[-1])].cpu(), torch.from_numpy(ids.view(np.int32)))
    back = torch.empty(total, dtype=torch.uint8, device="cuda")
    boff = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    assert e.decode_device(gpt2, d_ids.data_ptr(), d_oo.data_ptr(), n, int(oo[-1]), back.data_ptr(), total,
                           boff.data_ptr()) == total
    assert torch.equal(back, d_data) and torch.equal(boff, d_off)
    _, _, _, m4 = gpt2.export()
    orc = CRestatement(m4, [gpt2.byte_token(b) for b in range(256)])
    for r in np.random.default_rng(cfg).integers(0, n, 12):
        s = data[int(off[r]):int(off[r + 1])].tobytes()
        assert ids[int(oo[r]):int(oo[r + 1])].tolist() == orc.heap_bpe(orc.initial(s))


def test_device_jsonl_matches_reference_format(gpt2):
    """JSON-lines text on the device is byte-identical to
    write_batch_jsonl (batch.hpp:157-166: compact {"ids":[...],"len":n} per
    row, as the host mirror writes it), including empty rows; a capacity
    shorter than the text reports the full length."""
    torch = pytest.importorskip("torch")
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    rng = np.random.default_rng(51)
    lens = rng.integers(0, 300, 900)
    lens[::37] = 0
    data, off = synth.rows_lengths(gen, lens, seed=52)
    enc = bb.Encoder(0)
    ids, oo, _ = enc.encode_packed(gpt2, data, off)
    be = bb.BatchEncoding(batch_size=lens.size, pad_id=0)
    L = int(np.diff(oo.astype(np.int64)).max())
    be.max_len = L
    be.ids = np.zeros(lens.size * L, np.uint32)
    be.mask = np.zeros(lens.size * L, np.uint8)
    be.lengths = np.diff(oo.astype(np.int64)).astype(np.uint32)
    for r in range(lens.size):
        row = ids[int(oo[r]):int(oo[r + 1])]
        be.ids[r * L: r * L + row.size] = row
        be.mask[r * L: r * L + row.size] = 1
    want = bb.write_batch_jsonl(be).encode()
    d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
    d_oo = torch.from_numpy(oo.view(np.int64)).cuda()
    out = torch.empty(len(want) + 64, dtype=torch.uint8, device="cuda")
    n = enc.jsonl_device(d_ids.data_ptr(), d_oo.data_ptr(), lens.size, ids.size, out.data_ptr(), out.numel())
    assert n == len(want)
    assert bytes(out[:n].cpu().numpy()) == want
    assert enc.jsonl_device(d_ids.data_ptr(), d_oo.data_ptr(), lens.size, ids.size, out.data_ptr(), 10) == len(want)


def test_device_outputs_on_empty_and_degenerate_batches(gpt2):
    """Decode / JSONL / padding of empty batches, all-empty rows, a single
    empty row, and an unknown id in an otherwise empty batch."""
    torch = pytest.importorskip("torch")
    import ctypes as C
    from paper_2507_11941_b200._lib import LIB
    enc = bb.Encoder(0)
    for n in (0, 1, 5):
        off = np.zeros(n + 1, np.uint64)
        b, bo = enc.decode_packed(gpt2, np.zeros(0, np.uint32), off)
        assert b.size == 0 and np.array_equal(bo, off)
        d_ids = torch.zeros(1, dtype=torch.int32, device="cuda")
        d_off = torch.from_numpy(off.view(np.int64)).cuda()
        out = torch.empty(128, dtype=torch.uint8, device="cuda")
        t = enc.jsonl_device(d_ids.data_ptr(), d_off.data_ptr(), n, 0, out.data_ptr(), 128)
        assert t <= 128 and bytes(out[:t].cpu().numpy()) == b'{"ids":[],"len":0}\n' * n
        w = C.c_uint64()
        assert LIB.bbpe_batch_widest_device(enc.handle, C.c_void_p(d_off.data_ptr()), n, 0, 0, C.byref(w)) == 0
        assert w.value == 0
        ln = torch.full((max(n, 1),), 7, dtype=torch.int32, device="cuda")
        tr = C.c_uint64(9)
        assert LIB.bbpe_pad_device(enc.handle, C.c_void_p(d_ids.data_ptr()), C.c_void_p(d_off.data_ptr()), n, 0,
                                   0xFFFFFFFF, 0xFFFFFFFF, 0, None, C.c_void_p(ln.data_ptr()), None, C.byref(tr)) == 0
        assert tr.value == 0 and (n == 0 or ln[:n].cpu().tolist() == [0] * n)
    with pytest.raises(bb.DecodeError, match="row 2: unknown token id 60000 at index 0"):
        enc.decode_packed(gpt2, np.array([60000], np.uint32), np.array([0, 0, 0, 1], np.uint64))
    rows = bb.encode_batch([], gpt2, bb.SpecialTokenSet(), bb.BlockConfig(256, None), 0)
    assert rows.batch_size == 0 and rows.max_len == 0


PATTERN_CASES = [
    b"Hello world's test", b"it's we're they've I'm you'll he'd 'S 'tis", b"  leading and trailing  ",
    b"a\n\nb\n \nc\t\t x", b"x" * 40 + b"   " + b"1234567890" * 5, b"emoji \xf0\x9f\x98\x80 ok",
    "café naïve Ångström".encode(), "αβγ абв 中文 가나".encode(),
    "١٢ ²³  thin　ideo".encode(), b"\xaa\xb5\xba\x80\xff\xfe broken utf8 \xe2\x82",
    b"...!!!???", b"'", b" ", b"'ll", b"", b"don't stop-believin' 2023/24 $5.00",
    # the reference's pattern_pretokenize KAT inputs (test_pretokenize.cpp:114-150)
    b"1000", b"hello world", b"can't", b"a\n\nb", b"hi  ", b"hello  world", b"I'll be 42 today!", b" leading",
    b"tab\there", b"...wait", b"$3.14", "naïve café".encode(), b"a\r\nb", b"it's'll", b"don''t", b"100abc",
    b"A1b2", "a\xa0b".encode(), "a\xa0\xa0b".encode(), "a \xa0b".encode(), "a\xa0".encode(), "1½2".encode(),
    "x\u2003\u2003y".encode(),
]


@pytest.mark.parametrize("engine", ["pieces", "nomemo"])
def test_gpt2_pattern_mode_vs_reference(gpt2, engine):
    """encode_reference's pattern mode (ref_engines.hpp:119-146) with the gpt2
    splitter on the device: identical ids to the reference
    (oracle/_ref: pattern_pretokenize + heap_bpe) on contractions, whitespace
    runs and backoff, unicode letters/numbers/spaces, broken UTF-8, and Zipf
    text; the chunk starts equal the reference splitter's."""
    from oracle.oracle import Reference
    from workloads import text as synth
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    ids_, off_, blob_, m4_ = gpt2.export()
    ref = Reference.from_arrays(ids_, off_, blob_, m4_)
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off = synth.rows_fixed(gen, 2000, 256, seed=61)
    rows = PATTERN_CASES + [bytes(data[int(off[i]):int(off[i + 1])]) for i in range(off.size - 1)]
    d, o = bb.pack_rows(rows)
    want_ids, want_off = ref.encode_pattern(d, o, "gpt2", workers=8)
    enc = bb.Encoder(0, pattern="gpt2", piece_memo=(engine == "pieces"))
    ids, oo, _ = enc.encode_packed(gpt2, d, o)
    assert np.array_equal(oo, want_off)
    assert np.array_equal(ids, want_ids)
    # Byte-level and pattern mode differ somewhere on this input (the split is real).
    b_ids, b_oo, _ = bb.Encoder(0).encode_packed(gpt2, d, o)
    assert not np.array_equal(b_oo, oo) or not np.array_equal(b_ids, ids)


def test_gpt2_pattern_mode_rules(gpt2):
    with pytest.raises(bb.UsageError, match="only the gpt2 split pattern"):
        bb.Encoder(0, pattern=r"\w+")
    with pytest.raises(bb.UsageError, match="pieces engine"):
        bb.Encoder(0, pattern="gpt2", engine="block")
    enc = bb.Encoder(0, pattern=bb.api.GPT2_PATTERN)
    ids, oo, _ = enc.encode_packed(gpt2, *bb.pack_rows([b"hello world"]))
    assert ids.tolist() == [31373, 995]


def test_gpt2_pattern_mode_long_rows_and_newline_runs(gpt2):
    """The span-parallel splitter restarts after newlines: long rows with and
    without newlines, newline runs, CR/LF, and rows of one character class,
    against the reference splitter (chunk starts) and pattern encode."""
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    ids_, off_, blob_, m4_ = gpt2.export()
    ref = Reference.from_arrays(ids_, off_, blob_, m4_)
    rng = np.random.default_rng(71)
    alphabet = list(b"ab cd\n\n\r\t'sll.,!0123 ") + ["é".encode(), "αβ".encode(), b"\xe3\x80\x80", b"\xc2\xa0"]
    rows = []
    for _ in range(60):
        n = int(rng.integers(0, 3000))
        rows.append(b"".join(alphabet[i] if isinstance(alphabet[i], bytes) else bytes([alphabet[i]])
                             for i in rng.integers(0, len(alphabet), n)))
    rows += [b"word " * 2000, b"\n" * 500 + b"x", b"x\n" * 700, b"a" * 5000, b" \n \n  \n\t\n" * 90]
    # Short and long rows (threshold 4 KiB) interleaved so long rows start at
    # arbitrary offsets inside the splitter's 1 KiB spans.
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    tdata, toff = synth.rows_fixed(gen, 40, 9000, seed=72)
    for i in range(40):
        n = int(rng.integers(1000, 9000))
        if i % 2:
            rows.append(bytes(tdata[int(toff[i]):int(toff[i]) + n]))
        else:
            rows.append(b"".join(alphabet[j] if isinstance(alphabet[j], bytes) else bytes([alphabet[j]])
                                 for j in rng.integers(0, len(alphabet), n // 2)))
    d, o = bb.pack_rows(rows)
    want_ids, want_off = ref.encode_pattern(d, o, "gpt2", workers=8)
    ids, oo, _ = bb.Encoder(0, pattern="gpt2").encode_packed(gpt2, d, o)
    assert np.array_equal(oo, want_off) and np.array_equal(ids, want_ids)
    # Device API on an unaligned byte pointer (the splitter's row kernel needs
    # 16-byte alignment; unaligned input takes the tile kernel for every row).
    import torch
    enc = bb.Encoder(0, pattern="gpt2")
    for shift in (0, 3):
        buf = torch.zeros(d.size + 16, dtype=torch.uint8, device="cuda")
        buf[shift:shift + d.size] = torch.from_numpy(d.copy()).cuda()
        d_off = torch.from_numpy(o.view(np.int64).copy()).cuda()
        d_ids = torch.empty(d.size, dtype=torch.int32, device="cuda")
        d_oo = torch.empty(o.size, dtype=torch.int64, device="cuda")
        enc.encode_device(gpt2, buf.data_ptr() + shift, d_off.data_ptr(), o.size - 1, d.size, d_ids.data_ptr(),
                          d_oo.data_ptr())
        k = int(d_oo[-1].item())
        assert np.array_equal(d_oo.cpu().numpy().view(np.uint64), want_off)
        assert np.array_equal(d_ids[:k].cpu().numpy().view(np.uint32), want_ids)


SPECIALS = [(b"<|endoftext|>", 50256), (b"<|pad|>", 50300), (b"<|a|>", 60001), (b"<|a|>x", 60002),
            (b"\n\n", 60003), ("é".encode(), 60004), (b"zz", 60005)]
SPECIAL_CASES = [b"", b"<|endoftext|>", b"hi<|endoftext|>there", b"<|a|>x<|a|><|a|>xx", b"zzzzz", b"a\n\n\nb",
                 b"<|endofte", b"xt|>", b"<|endof", b"text|>", "café é\n\n".encode(), b"<|pad|><|pad|>",
                 b"plain text without any", b"<|a|", b"zz"]


def _special_rows(gpt2):
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    rng = np.random.default_rng(83)
    data, off = synth.rows_fixed(gen, 1500, 256, seed=84)
    rows = list(SPECIAL_CASES)
    for i in range(off.size - 1):
        r = bytes(data[int(off[i]):int(off[i + 1])])
        for _ in range(int(rng.integers(0, 4))):  # sprinkle specials in
            p = int(rng.integers(0, len(r) + 1))
            r = r[:p] + SPECIALS[int(rng.integers(0, len(SPECIALS)))][0] + r[p:]
        rows.append(r)
    long = b"".join(rows[15:60])  # long rows: many specials, incl. the common "\n\n"
    rows += [long * 3, b"\n\n" * 3000 + b"x", long]
    return rows


@pytest.mark.parametrize("bos_eos", [(False, False), (True, False), (False, True), (True, True)])
def test_device_specials_vs_reference(gpt2, bos_eos):
    """encode_batch with special tokens: the device split
    (bbpe_encode_batch_device: greedy longest-first split_specials,
    pretokenize.hpp:32-57, literal segments encoded, ids passed through,
    BOS/EOS) equals the compiled reference's encode_batch row for row, and
    the host split of the same rows."""
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    add_bos, add_eos = bos_eos
    ids_, off_, blob_, m4_ = gpt2.export()
    ref = Reference.from_arrays(ids_, off_, blob_, m4_)
    sp = bb.SpecialTokenSet()
    for b, i in SPECIALS:
        ref.add_special(b, i)
        sp.add(b, i)
    ref.add_special(b"<|endoftext|>", 50256, 1)
    ref.add_special(b"<|pad|>", 50300, 2)
    sp.set_bos("<|endoftext|>")
    sp.set_eos("<|pad|>")
    rows = _special_rows(gpt2)
    d, o = bb.pack_rows(rows)
    want_ids, want_off = ref.encode_batch(d, o, workers=8, add_bos=add_bos, add_eos=add_eos)
    cfg = bb.BlockConfig(256, None)
    ids, oo = bb.encode_batch_csr(rows, gpt2, sp, cfg, add_bos, add_eos)
    assert np.array_equal(oo, want_off)
    assert np.array_equal(ids, want_ids)
    h_ids, h_oo = bb.encode_batch_csr(rows, gpt2, sp, cfg, add_bos, add_eos, device_split=False)
    assert np.array_equal(h_oo, oo) and np.array_equal(h_ids, ids)
    # The padded BatchEncoding from the device equals the host assembly.
    dv = bb.encode_batch(rows[:300], gpt2, sp, cfg, 7, add_bos, add_eos, device_epilogue=True)
    hv = bb.encode_batch(rows[:300], gpt2, sp, cfg, 7, add_bos, add_eos, device_epilogue=False)
    assert dv.max_len == hv.max_len and np.array_equal(dv.ids, hv.ids) and np.array_equal(dv.mask, hv.mask)
    assert np.array_equal(dv.lengths, hv.lengths)


def test_device_specials_errors_and_rules(gpt2, tables):
    """Special bytes are never BPE-encoded (a special may hold a byte with no
    token); an invalid byte in a literal segment names the INPUT row; the set
    rejects empty and duplicate strings (SpecialTokenSet::add)."""
    toy = tables["toy"]
    cfg = bb.BlockConfig(256, None)
    sp = bb.SpecialTokenSet()
    sp.add("x", 900)
    ids, oo = bb.encode_batch_csr([b"abx", b"xab", b"x"], toy, sp, cfg)
    plain = bb.Encoder(0).encode_rows(toy, [b"ab"])[0]
    assert [ids[int(oo[i]):int(oo[i + 1])].tolist() for i in range(3)] == [plain + [900], [900] + plain, [900]]
    with pytest.raises(bb.IntegrityError, match=r"^row 2: .*byte value 121"):
        bb.encode_batch_csr([b"abx", b"xab", b"xay", b"ab"], toy, sp, cfg)

    class Raw:
        def __init__(self, e):
            self.e = e

        def entries(self):
            return self.e

    # Host entry (bbpe_encode_batch) as the FIRST call of a fresh ctx: the
    # lazy memo build must not clobber the staged input.
    fresh = bb.Encoder(0)
    d0, o0 = bb.pack_rows([b"abc", b"ab", b"cab"])
    ids0, oo0 = fresh.encode_batch_packed(toy, d0, o0)
    assert [ids0[int(oo0[i]):int(oo0[i + 1])].tolist() for i in range(3)] == [[4], [3], [2, 3]]
    fresh.set_specials(sp)
    ids0, oo0 = fresh.encode_batch_packed(toy, *bb.pack_rows([b"abx", b"xabc"]), bos_id=900, eos_id=900)
    assert ids0.tolist() == [900, 3, 900, 900, 900, 900, 4, 900] and oo0.tolist() == [0, 4, 8]
    enc = bb.Encoder(0)
    with pytest.raises(bb.UsageError, match="duplicate special"):
        enc.set_specials(Raw([(b"ab", 1), (b"ab", 2)]))
    with pytest.raises(bb.UsageError, match="may not be empty"):
        enc.set_specials(Raw([(b"", 1)]))
    # Longest first whatever the insertion order; n = 0 clears.
    enc.set_specials(Raw([(b"a", 1), (b"abc", 3), (b"ab", 2)]))
    import torch
    d = torch.tensor(list(b"abcabxa"), dtype=torch.uint8, device="cuda")
    o = torch.tensor([0, 7], dtype=torch.int64, device="cuda")
    out = torch.empty(16, dtype=torch.int32, device="cuda")
    oo = torch.empty(2, dtype=torch.int64, device="cuda")
    n = enc.encode_batch_device(gpt2, d.data_ptr(), o.data_ptr(), 1, 7, out.data_ptr(), 16, oo.data_ptr())
    assert n == 4 and out[:4].tolist() == [3, 2, gpt2.byte_token(ord("x")), 1] and oo.tolist() == [0, 4]
    with pytest.raises(bb.UsageError, match="output capacity"):
        enc.encode_batch_device(gpt2, d.data_ptr(), o.data_ptr(), 1, 7, out.data_ptr(), 3, oo.data_ptr())
    enc.set_specials(None)
    n = enc.encode_batch_device(gpt2, d.data_ptr(), o.data_ptr(), 1, 7, out.data_ptr(), 16, oo.data_ptr())
    assert out[:n].tolist() == bb.Encoder(0).encode_rows(gpt2, [b"abcabxa"])[0]


def test_encode_tensors_zero_copy(gpt2):
    """Zero-copy CSR hand-off: torch device tensors in and out,
    DLPack export shares the memory; a row window (offsets[0] != 0) works."""
    import torch
    from torch.utils.dlpack import from_dlpack, to_dlpack
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off = synth.rows_fixed(gen, 3000, 200, seed=91)
    enc = bb.Encoder(0)
    want_ids, want_off, _ = enc.encode_packed(gpt2, data, off)
    d = torch.from_numpy(data.copy()).cuda()
    o = torch.from_numpy(off.view(np.int64).copy()).cuda()
    ids, oo = enc.encode_tensors(gpt2, d, o)
    assert ids.is_cuda and ids.dtype == torch.int32 and oo.dtype == torch.int64
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), want_ids)
    assert np.array_equal(oo.cpu().numpy().view(np.uint64), want_off)
    assert from_dlpack(to_dlpack(ids)).data_ptr() == ids.data_ptr()
    sub_ids, sub_oo = enc.encode_tensors(gpt2, d, o[100:201])
    a, b = int(want_off[100]), int(want_off[200])
    assert np.array_equal(sub_ids.cpu().numpy().view(np.uint32), want_ids[a:b])
    assert np.array_equal(sub_oo.cpu().numpy(), (want_off[100:201] - want_off[100]).astype(np.int64))
    with pytest.raises(bb.UsageError):
        enc.encode_tensors(gpt2, d.cpu(), o)


def test_device_call_over_4_gib(gpt2):
    """One device-API call over 4 GiB of input (20 x the cfg2 batch, 5.4 GB):
    no 32-bit tile / slot / record index overflows -- the ids and offsets are
    exactly the single batch's, repeated (rows are independent)."""
    import torch
    from workloads import text as synth
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off, _ = synth.config_rows(gen, 2)
    e = bb.Encoder(0)
    ids1, oo1, _ = e.encode_packed(gpt2, data, off)
    R, n, B, T = 20, off.size - 1, int(off[-1]), int(oo1[-1])
    assert R * B > (1 << 32)
    d1 = torch.from_numpy(data).cuda()
    d = d1.repeat(R)
    o1 = torch.from_numpy(off.view(np.int64)).cuda()
    o = torch.cat([o1[:-1] + k * B for k in range(R)] + [torch.tensor([R * B], device="cuda")])
    del d1
    ids = torch.empty(R * B, dtype=torch.int32, device="cuda")
    oo = torch.empty(R * n + 1, dtype=torch.int64, device="cuda")
    e.encode_device(gpt2, d.data_ptr(), o.data_ptr(), R * n, R * B, ids.data_ptr(), oo.data_ptr())
    del d
    assert int(oo[-1].item()) == R * T
    want_ids = torch.from_numpy(ids1.view(np.int32)).cuda()
    want_oo = torch.from_numpy(oo1.view(np.int64)).cuda()
    for k in range(R):
        assert torch.equal(ids[k * T:(k + 1) * T], want_ids)
        assert torch.equal(oo[k * n:(k + 1) * n + 1] - k * T, want_oo)


def test_pattern_mode_with_specials_vs_reference(gpt2):
    """gpt2 pattern mode together with special tokens: specials split first,
    each literal segment pattern-split and encoded (encode_reference,
    ref_engines.hpp:119-146) -- device split + segment rows in pattern mode."""
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    ids_, off_, blob_, m4_ = gpt2.export()
    ref = Reference.from_arrays(ids_, off_, blob_, m4_)
    enc = bb.Encoder(0, pattern="gpt2")
    sp = bb.SpecialTokenSet()
    for b, i in SPECIALS:
        ref.add_special(b, i)
        sp.add(b, i)
    enc.set_specials(sp)
    rows = _special_rows(gpt2)[:400] + PATTERN_CASES
    d, o = bb.pack_rows(rows)
    want_ids, want_off = ref.encode_pattern(d, o, "gpt2", workers=8)
    ids, oo = enc.encode_batch_packed(gpt2, d, o)
    assert np.array_equal(oo, want_off)
    assert np.array_equal(ids, want_ids)


@pytest.mark.parametrize("skip", [False, True])
def test_device_decode_batch_with_specials(gpt2, skip):
    """decode_batch (batch.hpp:128-154) on the GPU with special tokens: ids the
    table lacks decode to their special's bytes, skip_specials drops special
    ids (a special id that is also a table token -- GPT-2's end of text -- is
    dropped too); the unknown-id error counts the index among kept ids."""
    sp = bb.SpecialTokenSet()
    for b, i in SPECIALS:
        sp.add(b, i)
    rows = _special_rows(gpt2)[:300]
    cfg = bb.BlockConfig(256, None)
    be = bb.encode_batch(rows, gpt2, sp, cfg, 0)
    got = bb.decode_batch(be, gpt2, sp, skip)
    for r in range(0, be.batch_size, 5):  # the host mirror of decode, merge_table.hpp:565-579
        ids = be.row(r)
        if skip:
            ids = [i for i in ids if not sp.contains_id(i)]
        assert got[r] == bb.decode(gpt2, sp, ids), r
    if not skip:
        assert got == [bytes(x) for x in rows]  # lossless round trip through the specials
    bad = bb.BatchEncoding(batch_size=2, max_len=4, pad_id=0)
    bad.ids = np.array([31373, 0, 0, 0, 50300, 60001, 70000, 995], np.uint32)
    bad.lengths = np.array([1, 4], np.uint32)
    bad.mask = np.ones(8, np.uint8)
    with pytest.raises(bb.DecodeError, match=f"row 1: unknown token id 70000 at index {0 if skip else 2}"):
        bb.decode_batch(bad, gpt2, sp, skip)


def test_gpt2_splitter_chunk_starts_vs_reference(gpt2):
    """The device splitter itself (bbpe_pretokenize_device): chunk starts equal
    pattern_pretokenize("gpt2")'s (pretokenize.hpp:79-264, oracle/_ref) on the
    reference's KAT strings, mixed-alphabet rows, and long rows (> 4 KiB, the
    span kernel) interleaved with short ones; an encode on the same ctx after
    it still matches (the splitter's scratch is re-zeroed)."""
    import torch
    from oracle.oracle import Reference
    from workloads import text as synth
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    ids_, off_, blob_, m4_ = gpt2.export()
    ref = Reference.from_arrays(ids_, off_, blob_, m4_)
    rng = np.random.default_rng(29)
    alphabet = [bytes([c]) for c in b"ab cd\n\n\r\t'sll.,!0123 "] + ["é".encode(), "αβ".encode(), b"\xe3\x80\x80",
                                                                    b"\xc2\xa0", b"\xe2\x80\x83", b"\xff"]
    rows = list(PATTERN_CASES)
    for n in rng.integers(0, 9000, 60):
        rows.append(b"".join(alphabet[j] for j in rng.integers(0, len(alphabet), int(n) // 2)))
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off = synth.rows_fixed(gen, 30, 7000, seed=30)
    rows += [bytes(data[int(off[i]):int(off[i + 1])]) for i in range(30)]
    d, o = bb.pack_rows(rows)
    total = int(o[-1])
    enc = bb.Encoder(0)
    dd = torch.from_numpy(d.copy()).cuda()
    do = torch.from_numpy(o.view(np.int64).copy()).cuda()
    bits = torch.zeros((total + 31) // 32, dtype=torch.int32, device="cuda")
    enc.pretokenize_device(dd.data_ptr(), do.data_ptr(), len(rows), total, bits.data_ptr())
    b = bits.cpu().numpy().view(np.uint32)
    flags = ((b[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool).reshape(-1)[:total]
    starts = np.nonzero(flags)[0]
    for r, s in enumerate(rows):
        lo, hi = int(o[r]), int(o[r + 1])
        got = (starts[(starts >= lo) & (starts < hi)] - lo).tolist()
        assert got == list(ref.pretokenize(s, "gpt2")), (r, s[:60])
    ids, oo, _ = enc.encode_packed(gpt2, d, o)
    want, wo, _ = bb.Encoder(0).encode_packed(gpt2, d, o)
    assert np.array_equal(ids, want) and np.array_equal(oo, wo)


def test_splitter_unaligned_and_decode_device_skip(gpt2):
    """bbpe_pretokenize_device on an unaligned byte pointer (plain-load kernels)
    equals the aligned result; bbpe_decode_device_ex with skip_specials on
    device buffers equals the host-buffer decode."""
    import torch
    rows = list(PATTERN_CASES) + [b"word " * 1200, b"x\n" * 3000]
    d, o = bb.pack_rows(rows)
    total = int(o[-1])
    enc = bb.Encoder(0)
    do = torch.from_numpy(o.view(np.int64).copy()).cuda()
    outs = []
    for shift in (0, 5):
        buf = torch.zeros(total + 16, dtype=torch.uint8, device="cuda")
        buf[shift:shift + total] = torch.from_numpy(d.copy()).cuda()
        bits = torch.zeros((total + 31) // 32, dtype=torch.int32, device="cuda")
        enc.pretokenize_device(buf.data_ptr() + shift, do.data_ptr(), len(rows), total, bits.data_ptr())
        outs.append(bits.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    sp = bb.SpecialTokenSet()
    for b, i in SPECIALS:
        sp.add(b, i)
    sp.set_bos("<|endoftext|>")
    srows = _special_rows(gpt2)[:200]
    ids, oo = bb.encode_batch_csr(srows, gpt2, sp, bb.BlockConfig(256, None), True, False)
    enc.set_specials(sp)
    want, woff = enc.decode_packed(gpt2, ids, oo, skip_specials=True)
    d_ids = torch.from_numpy(ids.view(np.int32)).cuda()
    d_oo = torch.from_numpy(oo.view(np.int64)).cuda()
    cap = int(woff[-1]) + 64
    d_out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    d_boff = torch.empty(len(srows) + 1, dtype=torch.int64, device="cuda")
    n = enc.decode_device(gpt2, d_ids.data_ptr(), d_oo.data_ptr(), len(srows), ids.size, d_out.data_ptr(), cap,
                          d_boff.data_ptr(), skip_specials=True)
    assert n == int(woff[-1])
    assert bytes(d_out[:n].cpu().numpy()) == bytes(want)
    assert np.array_equal(d_boff.cpu().numpy().view(np.uint64), woff)


def test_splitter_full_size_cfg3_vs_reference(gpt2):
    """The gpt2 splitter at full cfg3 size (16,384 rows of U[8, 64] KiB, the
    span kernel): chunk starts of 120 random rows equal the reference
    pattern_pretokenize's."""
    import torch
    from oracle.oracle import Reference
    from workloads import text as synth
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    ids_, off_, blob_, m4_ = gpt2.export()
    ref = Reference.from_arrays(ids_, off_, blob_, m4_)
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off, _ = synth.config_rows(gen, 3, seed=3000)
    n, total = off.size - 1, int(off[-1])
    enc = bb.Encoder(0)
    dd = torch.from_numpy(data).cuda()
    do = torch.from_numpy(off.view(np.int64)).cuda()
    bits = torch.zeros((total + 31) // 32, dtype=torch.int32, device="cuda")
    enc.pretokenize_device(dd.data_ptr(), do.data_ptr(), n, total, bits.data_ptr())
    b = bits.cpu().numpy().view(np.uint32)
    rng = np.random.default_rng(3)
    for r in rng.integers(0, n, 120):
        lo, hi = int(off[r]), int(off[r + 1])
        w0, w1 = lo // 32, (hi + 31) // 32
        flags = ((b[w0:w1, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool).reshape(-1)
        got = (np.nonzero(flags[lo - 32 * w0:hi - 32 * w0])[0]).tolist()
        assert got == list(ref.pretokenize(data[lo:hi].tobytes(), "gpt2")), int(r)
