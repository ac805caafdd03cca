#!/usr/bin/env python3
"""Generates tests/golden/* from the UNMODIFIED reference (oracle/_ref).

Run in the container that has /root/reference (the GPU box does not):
    make -C oracle && python tests/golden/make_golden.py

Outputs (committed):
  gpt2.bbpt            GPT-2 table (50,257 tokens / 50,000 merges) exported by
                       the reference loader (load_merge_table_files,
                       merge_table.hpp:513) and written in this repo's .bbpt
                       format by THIS script (independent of the product loader)
  toy_tables.json      toy / toy8 / doubling / inconsistent tables in the
                       reference's canonical JSON layout (tests/helpers.hpp:19-80)
  vectors_*.npz        row sets + expected CSR ids from the reference's
                       encode_batch (block engine, batch.hpp:64-126)
  traces.json          block_bpe pass traces (block_engine.hpp:42-47, 303-304)
  kats.json            the hard-coded id vectors of the reference tests
"""
import json
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference, pack  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
GPT2 = "/root/reference/proj/tests/testdata/gpt2/"


def write_bbpt(path, ids, off, blob, m4):
    with open(path, "wb") as f:
        f.write(b"BBPT")
        f.write(struct.pack("<IQQQ", 1, len(ids), len(blob), len(m4)))
        f.write(np.asarray(ids, "<u4").tobytes())
        f.write(np.asarray(off, "<u8").tobytes())
        f.write(np.asarray(blob, np.uint8).tobytes())
        f.write(np.asarray(m4, "<u4").reshape(-1, 4).tobytes())


# ---- toy tables (restating tests/helpers.hpp:19-114) ----
def toy():
    return {"tokens": [[0, b"a"], [1, b"b"], [2, b"c"], [3, b"ab"], [4, b"abc"]],
            "merges": [[0, 0, 1, 3], [1, 3, 2, 4]]}


def toy8():
    toks = [b"a", b"b", b"c", b"d", b"ab", b"abc", b"cd", b"dd", b"abab", b"ba", b"ddd", b"aa"]
    return {"tokens": [[i, t] for i, t in enumerate(toks)],
            "merges": [[0, 0, 1, 4], [1, 4, 2, 5], [2, 2, 3, 6], [3, 3, 3, 7], [4, 4, 4, 8], [5, 1, 0, 9],
                       [6, 7, 3, 10], [7, 0, 0, 11]]}


def doubling():
    toks = [[0, b"a"], [1, b"b"], [3, b"ab"]]
    merges = [[0, 0, 1, 3]]
    word, prev = b"ab", 3
    for r in range(1, 7):
        merged = prev + 2
        word = word + word
        toks.append([merged, word])
        merges.append([r, prev, prev, merged])
        prev = merged
    return {"tokens": toks, "merges": merges}


def inconsistent():
    # (ab, a) -> aba @0, (a, b) -> ab @1. naive/heap give
    # [aba, b] on "abab", the block engine gives [ab, ab].
    return {"tokens": [[0, b"a"], [1, b"b"], [2, b"ab"], [3, b"aba"]],
            "merges": [[0, 2, 0, 3], [1, 0, 1, 2]]}


def random_table(rng, base, count):
    toks = [[i, bytes([ord("a") + i])] for i in range(base)]
    by_id = {i: bytes([ord("a") + i]) for i in range(base)}
    pool = list(range(base))
    used, words = set(), set(by_id.values())
    merges, nxt, rank, attempts = [], base, 0, 0
    while rank < count and attempts < count * 50:
        attempts += 1
        l, r = pool[rng.integers(len(pool))], pool[rng.integers(len(pool))]
        if (l, r) in used:
            continue
        w = by_id[l] + by_id[r]
        if w in words:
            continue
        used.add((l, r))
        words.add(w)
        toks.append([nxt, w])
        by_id[nxt] = w
        merges.append([rank, l, r, nxt])
        pool.append(nxt)
        nxt += 1
        rank += 1
    return {"tokens": toks, "merges": merges}


def table_arrays(t):
    toks = sorted(t["tokens"])
    ids = np.array([x[0] for x in toks], np.uint32)
    off = np.zeros(len(toks) + 1, np.uint64)
    np.cumsum([len(x[1]) for x in toks], out=off[1:])
    blob = np.frombuffer(b"".join(x[1] for x in toks), np.uint8)
    return ids, off, blob, np.array(t["merges"], np.uint32).reshape(-1, 4)


def ref_of(t):
    return Reference.from_arrays(*table_arrays(t))


def json_table(t):
    return {"tokens": [[i, list(b)] for i, b in t["tokens"]], "merges": t["merges"]}


def save_vectors(name, ref, rows, table_name, **extra):
    data, off = pack(rows)
    ids, oo = ref.encode_batch(data, off, workers=8)
    np.savez_compressed(os.path.join(OUT, f"vectors_{name}.npz"), data=data, offsets=off, ids=ids,
                        out_offsets=oo, table=np.array(table_name), **extra)
    print(f"vectors_{name}: {len(rows)} rows, {data.size} bytes, {ids.size} tokens")


def random_bytes(rng, max_len):
    return bytes(rng.integers(0, 256, rng.integers(0, max_len + 1)).astype(np.uint8))


def random_utf8(rng, max_len):
    budget = int(rng.integers(0, max_len + 1))
    out = b""
    while len(out) < budget:
        k = int(rng.integers(4))
        if k == 0:
            cp = int(rng.integers(0x80))
        elif k == 1:
            cp = 0x80 + int(rng.integers(0x800 - 0x80))
        elif k == 2:
            cp = 0x800 + int(rng.integers(0x10000 - 0x800))
            if 0xD800 <= cp <= 0xDFFF:
                cp = 0x4E00
        else:
            cp = 0x10000 + int(rng.integers(0x110000 - 0x10000))
        out += chr(cp).encode("utf-8")
    return out[:budget]


def main():
    ref = Reference.load_files(GPT2 + "vocab.json", GPT2 + "merges.txt")
    ids, off, blob, m4 = ref.export()
    write_bbpt(os.path.join(OUT, "gpt2.bbpt"), ids, off, blob, m4)
    print("gpt2.bbpt:", len(ids), "tokens", len(m4), "merges")

    # KATs (test_cli.cpp:47-108, test_ref_engines.cpp:124-160,
    # test_batch.cpp:68-76), checked against the reference here.
    kats = [["hello world", [31373, 995]], ["....", [1106]], ["1000", [12825]], ["hi", [5303]],
            [".'t", [13, 470]], ["a\n\nb", [64, 628, 65]]]
    for s, want in kats:
        d, o = pack([s.encode()])
        got = ref.encode_batch(d, o)[0].tolist()
        assert got == want, (s, got, want)
    ref_sp = Reference.load_files(GPT2 + "vocab.json", GPT2 + "merges.txt")
    ref_sp.add_special(b"<|endoftext|>", 50256)
    ref_sp.add_special(b"<|endoftext|>", 50256, 1)
    ref_sp.add_special(b"<|endoftext|>", 50256, 2)
    d, o = pack([b"hi"])
    bos = ref_sp.encode_batch(d, o, add_bos=True, add_eos=True)[0].tolist()
    assert bos == [50256, 5303, 50256], bos
    d, o = pack([b"hi<|endoftext|>"])
    sp = ref_sp.encode_batch(d, o)[0].tolist()
    assert sp == [5303, 50256], sp
    with open(os.path.join(OUT, "kats.json"), "w") as f:
        json.dump({"gpt2": kats, "gpt2_bos_eos": [["hi", bos]], "gpt2_special": [["hi<|endoftext|>", sp]],
                   "toy_canonical": [["abc", [4]], ["ab", [3]]]}, f, indent=1)

    tables = {"toy": toy(), "toy8": toy8(), "doubling": doubling(), "inconsistent": inconsistent()}
    rng = np.random.default_rng(47)
    for k in range(20):
        tables[f"random{k}"] = random_table(rng, 4, 12)
    with open(os.path.join(OUT, "toy_tables.json"), "w") as f:
        json.dump({k: json_table(v) for k, v in tables.items()}, f)

    rng = np.random.default_rng(43)
    rows = [random_bytes(rng, 128) for _ in range(300)] + [random_utf8(rng, 128) for _ in range(100)] + \
           [random_bytes(rng, 256) for _ in range(200)]
    save_vectors("gpt2_random", ref, rows, "gpt2")

    from paper_2507_11941_b200 import load_merge_table_files
    from workloads import text as synth
    t = load_merge_table_files(os.path.join(OUT, "gpt2.bbpt"), None, "binary")
    gen = synth.TextGen(synth.word_list(t))
    d1, o1, _ = synth.config_rows(gen, 1, scale=1 / 16)
    text_rows = [bytes(d1[int(o1[i]):int(o1[i + 1])]) for i in range(len(o1) - 1)]
    d3 = gen.stream(8 * 8192, seed=33)
    text_rows += [bytes(d3[i * 8192:(i + 1) * 8192]) for i in range(8)]
    corpus = open("/root/reference/proj/tests/testdata/corpus.txt", "rb").read()
    text_rows += [corpus[i:i + 1024] for i in range(0, 32 * 1024, 1024)]
    save_vectors("gpt2_text", ref, text_rows, "gpt2")

    rng = np.random.default_rng(7)
    adv = [b"a" * 65536, b"." * 65536, b"0" * 65536, b" " * 65536,
           bytes(rng.integers(0, 256, 65536).astype(np.uint8)),
           bytes(rng.choice(np.frombuffer(b"0123456789 ", np.uint8), 65536)),
           b"ab" * 2000, b"\n" * 300, b"!" * 33, b"a" * 33, b"a" * 32, b"a" * 31, b"1" * 40,
           b"  " * 50 + b"x", b"", b"x"]
    save_vectors("gpt2_adversarial", ref, adv, "gpt2")

    # toy8 exhaustive (<= 5 symbols over abcd, test_block_engine.cpp:187-202)
    import itertools
    rows = [b""]
    for L in range(1, 6):
        rows += [bytes(p) for p in itertools.product(b"abcd", repeat=L)]
    save_vectors("toy8_exhaustive", ref_of(tables["toy8"]), rows, "toy8")

    rng = np.random.default_rng(11)
    rows = [b"abab", b"ababab", b"aab", b"abba"] + \
           [bytes(rng.choice(np.frombuffer(b"ab", np.uint8), rng.integers(0, 20))) for _ in range(200)]
    save_vectors("inconsistent", ref_of(tables["inconsistent"]), rows, "inconsistent")

    rng = np.random.default_rng(53)
    for k in range(4):
        rows = [bytes(rng.choice(np.frombuffer(b"abcd", np.uint8), rng.integers(0, 15))) for _ in range(100)]
        save_vectors(f"random{k}", ref_of(tables[f"random{k}"]), rows, f"random{k}")

    rows = [b"ab" * k for k in range(1, 65)] + [b"ab" * 3 + b"a"]
    save_vectors("doubling", ref_of(tables["doubling"]), rows, "doubling")

    # Pass traces (block_bpe with PassTrace) for the doubling family and a few
    # GPT-2 inputs, plus a MaxPassesError partial state (test_block_engine.cpp:384-399).
    dref = ref_of(tables["doubling"])
    traces = {"doubling": [], "gpt2": []}
    for k in range(1, 65):
        toks = [0, 1] * k
        out, tr = dref.block_bpe(toks)
        traces["doubling"].append({"tokens": toks, "out": out, "trace": tr})
    rng = np.random.default_rng(67)
    bt = ref.byte_tokens()
    for _ in range(30):
        s = random_bytes(rng, 80)
        toks = [bt[b] for b in s]
        out, tr = ref.block_bpe(toks)
        traces["gpt2"].append({"tokens": toks, "out": out, "trace": tr})
    try:
        dref.block_bpe([0, 1] * 8, max_passes=2)
        raise AssertionError("expected MaxPassesError")
    except RuntimeError as e:
        code, partial, passes = e.args
        assert code == 6
        traces["max_passes"] = {"tokens": [0, 1] * 8, "max_passes": 2, "partial": partial, "passes": passes}
    with open(os.path.join(OUT, "traces.json"), "w") as f:
        json.dump(traces, f)
    print("traces.json written")


if __name__ == "__main__":
    main()
