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
    from workloads import text as synth
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
    from workloads import text as synth
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


# ---- the reference's own CLI tests (proj/tests/test_cli.cpp), same inputs and
# expectations; the GPT-2 table comes from tests/golden/gpt2.bbpt (--format binary).

def gpt2_args():
    return ["--vocab", os.path.join(GOLDEN, "gpt2.bbpt"), "--format", "binary"]


def test_ref_cli_exit_codes_and_eval(tmp_path):
    """test_cli.cpp: ExitCodeOneOnUsageErrors, ExitCodeTwoOnIntegrityErrors,
    EvalComputesSimilarity (no GPU involved)."""
    build_cli()
    inp = tmp_path / "in6.txt"
    inp.write_text("x\n")
    assert run("tokenize").returncode == 1
    assert run("tokenize", "--vocab", "/nonexistent.json", "--merges", "/nonexistent.txt", str(inp)).returncode == 1
    assert run("nonsense-subcommand").returncode == 1
    refs = tmp_path / "refs2.jsonl"
    refs.write_text('{"ids":[1]}\n')
    lens0 = tmp_path / "lens2.txt"
    lens0.write_text("0\n")
    assert run("eval", "--refs", str(refs), "--cands", str(refs), "--source-lens", str(lens0)).returncode == 1
    (tmp_path / "dv.json").write_text('{"a":0,"b":1,"ab":2}')
    (tmp_path / "dm.txt").write_text("#version: 0.2\na b\na b\n")
    (tmp_path / "in7.txt").write_text("ab\n")
    r = run("tokenize", "--vocab", str(tmp_path / "dv.json"), "--merges", str(tmp_path / "dm.txt"),
            str(tmp_path / "in7.txt"))
    assert r.returncode == 2
    (tmp_path / "refs.jsonl").write_text('{"ids":[1,2]}\n{"ids":[3]}\n')
    (tmp_path / "cands.jsonl").write_text('{"ids":[1]}\n{"ids":[3]}\n')
    (tmp_path / "lens.txt").write_text("4\n2\n")
    r = run("eval", "--json", "--refs", str(tmp_path / "refs.jsonl"), "--cands", str(tmp_path / "cands.jsonl"),
            "--source-lens", str(tmp_path / "lens.txt"))
    assert r.returncode == 0
    j = json.loads(r.stdout)
    assert j["count"] == 2 and abs(j["aggregate_sim"] - 0.875) < 1e-12


@pytest.mark.gpu
def test_ref_cli_tokenize_cases(tmp_path):
    """test_cli.cpp: TokenizeJsonl, TokenizeBinary, TokenizeWithSpecialsAndBosEos,
    TokenizeCanonicalJsonFormat."""
    build_cli()
    (tmp_path / "in.txt").write_text("hello world\n....\n")
    r = run("tokenize", *gpt2_args(), str(tmp_path / "in.txt"))
    assert r.returncode == 0
    assert r.stdout == b'{"ids":[31373,995],"len":2}\n{"ids":[1106],"len":1}\n'
    (tmp_path / "in3.txt").write_text("hi\n")
    out = tmp_path / "out.bbpe"
    assert run("tokenize", "--out", "bin", "--output", str(out), *gpt2_args(), str(tmp_path / "in3.txt")).returncode == 0
    blob = out.read_bytes()
    assert len(blob) >= 16 and blob[:4] == b"BBPE"
    (tmp_path / "sp.json").write_text('{"specials": [["<|endoftext|>", 50256]], '
                                      '"bos": "<|endoftext|>", "eos": "<|endoftext|>"}')
    r = run("tokenize", "--bos", "--eos", "--specials", str(tmp_path / "sp.json"), *gpt2_args(),
            str(tmp_path / "in3.txt"))
    assert r.returncode == 0 and r.stdout == b'{"ids":[50256,5303,50256],"len":3}\n'
    (tmp_path / "canon.json").write_text('{"tokens": [[0, [97]], [1, [98]], [2, [99]], [3, [97, 98]], '
                                         '[4, [97, 98, 99]]], "merges": [[0, 0, 1, 3], [1, 3, 2, 4]]}')
    (tmp_path / "in5.txt").write_text("abc\nab\n")
    r = run("tokenize", "--vocab", str(tmp_path / "canon.json"), "--format", "json", str(tmp_path / "in5.txt"))
    assert r.returncode == 0 and r.stdout == b'{"ids":[4],"len":1}\n{"ids":[3],"len":1}\n'


@pytest.mark.gpu
def test_ref_cli_compare_cases(tmp_path):
    """test_cli.cpp: CompareReportsDivergence, CompareTextOutput."""
    build_cli()
    (tmp_path / "cmp.txt").write_text(".'t\nhello\n")
    r = run("compare", "--pattern", "gpt2", "--json", *gpt2_args(), str(tmp_path / "cmp.txt"))
    assert r.returncode == 0
    j = json.loads(r.stdout)
    assert j["count"] == 2 and j["divergent_count"] == 1
    assert j["items"][0]["divergent"] is True
    assert j["items"][0]["reference_tokens"] == [2637, 83] and j["items"][0]["block_tokens"] == [13, 470]
    assert j["items"][1]["divergent"] is False
    (tmp_path / "cmp2.txt").write_text(".'t\n")
    r = run("compare", "--pattern", "gpt2", *gpt2_args(), str(tmp_path / "cmp2.txt"))
    assert r.returncode == 0 and b"DIVERGE" in r.stdout
