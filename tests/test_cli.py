"""tools/bbpe_cli.cpp: the reference CLI's `tokenize` (blockbpe_cli.cpp:73-127,
219-230) on the B200 encoder. CPU: it builds and maps usage errors to exit
code 1. GPU: its JSONL and binary output is byte-identical to the reference's
encode_batch + write_batch_jsonl / write_batch_binary (oracle/_ref), with
specials, BOS/EOS and the default pad id (eos if set, else 0)."""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

EXE = os.path.join(ROOT, "build", "bbpe_cli")
NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"


def build_cli():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    lib = os.path.join(ROOT, "paper_2507_11941_b200")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), "-I" + NLOHMANN,
           os.path.join(ROOT, "tools", "bbpe_cli.cpp"), "-L" + lib, "-lbbpe_b200", "-Wl,-rpath," + lib, "-o", EXE]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def run(*args):
    return subprocess.run([EXE, *args], capture_output=True, timeout=300)


def test_cli_builds_and_usage_errors():
    build_cli()
    assert run("--help").returncode == 0
    assert run("tokenize", "--vocab", "v.json").returncode == 1                      # no input
    assert run("tokenize", "--vocab", "v", "--engine", "gpu", "in").returncode == 1  # test_bench.cpp:176
    assert run("tokenize", "--vocab", "v", "--out", "xml", "in").returncode == 1
    assert run("tokenize", "--vocab", "v", "--block-size", "abc", "in").returncode == 1
    assert run("encode").returncode == 1
    assert run("tokenize", "--vocab", "v.json", "--format", "gpt2", "in").returncode == 1  # gpt2 needs --merges


@pytest.mark.gpu
@pytest.mark.parametrize("out,specials,bos_eos", [("jsonl", False, False), ("bin", False, False),
                                                  ("jsonl", True, True), ("bin", True, True)])
def test_cli_tokenize_matches_reference(tmp_path, gpt2, out, specials, bos_eos):
    from oracle.oracle import Reference
    import paper_2507_11941_b200 as bb
    from paper_2507_11941_b200 import synth
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    build_cli()
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off = synth.rows_fixed(gen, 300, 200, seed=97)
    rows = [bytes(data[int(off[i]):int(off[i + 1])]).replace(b"\n", b" ") for i in range(300)]
    rows[::17] = [b""] * len(rows[::17])
    rows[5] = b"hi<|endoftext|>there<|pad|>"
    src = tmp_path / "in.txt"
    src.write_bytes(b"\n".join(rows) + b"\n")
    ids_, off_, blob_, m4_ = gpt2.export()
    ref = Reference.from_arrays(ids_, off_, blob_, m4_)
    args = ["tokenize", "--vocab", os.path.join(GOLDEN, "gpt2.bbpt"), "--format", "binary", "--out", out,
            "--output", str(tmp_path / "out")]
    pad = 0
    if specials:
        (tmp_path / "sp.json").write_text(json.dumps({"specials": [["<|endoftext|>", 50256], ["<|pad|>", 50300]],
                                                      "bos": "<|endoftext|>", "eos": "<|pad|>"}))
        args += ["--specials", str(tmp_path / "sp.json")]
        ref.add_special(b"<|endoftext|>", 50256)
        ref.add_special(b"<|pad|>", 50300)
        ref.add_special(b"<|endoftext|>", 50256, 1)
        ref.add_special(b"<|pad|>", 50300, 2)
        pad = 50300  # the CLI's default pad id: eos if set
    if bos_eos:
        args += ["--bos", "--eos"]
    r = run(*args, str(src))
    assert r.returncode == 0, r.stderr.decode()
    d, o = bb.pack_rows(rows)
    want = ref.write_batch(d, o, pad, out == "bin", workers=8, add_bos=bos_eos, add_eos=bos_eos)
    assert (tmp_path / "out").read_bytes() == want


@pytest.mark.gpu
def test_cli_errors_are_row_tagged(tmp_path):
    """An input byte with no token: exit 2 and the reference's row-tagged message."""
    build_cli()
    toy = {"tokens": [[0, [97]], [1, [98]], [2, [97, 98]]], "merges": [[0, 0, 1, 2]]}  # README.md:159-173
    vocab = tmp_path / "toy.json"
    vocab.write_text(json.dumps(toy))
    src = tmp_path / "in.txt"
    src.write_bytes(b"ab\nab\nxab\n")
    r = run("tokenize", "--vocab", str(vocab), "--format", "json", str(src))
    assert r.returncode == 2, r.stderr.decode()
    assert b"row 2" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("as_json", [False, True])
def test_cli_compare_matches_reference(tmp_path, gpt2, as_json):
    """`compare --pattern gpt2` (both encodes on the GPU: byte-level rows vs the
    gpt2 split-pattern mode) prints the reference's divergence report
    (eval.hpp:147-273, oracle/_ref/ref_compare) byte for byte."""
    import paper_2507_11941_b200 as bb
    from paper_2507_11941_b200 import synth
    ref_bin = os.path.join(ROOT, "oracle", "_ref", "ref_compare")
    if not os.path.exists(ref_bin):
        pytest.skip("oracle/_ref not built")
    build_cli()
    ids_, off_, blob_, m4_ = gpt2.export()
    canon = {"tokens": [[int(i), [int(b) for b in blob_[int(off_[k]):int(off_[k + 1])]]] for k, i in enumerate(ids_)],
             "merges": np.asarray(m4_).reshape(-1, 4).astype(np.int64).tolist()}
    vocab = tmp_path / "gpt2_canonical.json"
    vocab.write_text(json.dumps(canon))
    gen = synth.TextGen(synth.word_list(gpt2))
    data, off = synth.rows_fixed(gen, 200, 160, seed=99)
    rows = [bytes(data[int(off[i]):int(off[i + 1])]).replace(b"\n", b" ") for i in range(200)]
    rows += [b"", b"hello!!! world", b"it's 12345 and 678", b"don't   stop\t now", "café ünïcode 中文".encode(),
             b"...???!!!", b"a'll b're c've", b"\xff\xfe broken", b"   ", b"x" * 300,
             # NBSP runs: GPT-2's byte-level merges and its split pattern disagree here
             b"\xc2\xa0\xc2\xa0x", b"x\xc2\xa0\xc2\xa0\xc2\xa0y", b"\xc2\xa0\xc2\xa0z"]
    src = tmp_path / "in.txt"
    src.write_bytes(b"\n".join(rows) + b"\n")
    flag = ["--json"] if as_json else []
    r = run("compare", "--vocab", os.path.join(GOLDEN, "gpt2.bbpt"), "--format", "binary", "--pattern", "gpt2",
            *flag, str(src))
    assert r.returncode == 0, r.stderr.decode()
    want = subprocess.run([ref_bin, str(vocab), "gpt2", "1" if as_json else "0", str(src)], capture_output=True,
                          timeout=600)
    assert want.returncode == 0, want.stderr.decode()
    assert r.stdout == want.stdout
    assert (b'"divergent": true' if as_json else b"DIVERGE [") in r.stdout  # items that differ are reported
