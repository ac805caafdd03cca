"""The SURVEY.md §8(d) cfg4 table: GPT-2 continued by BPE training WITHOUT
pre-tokenization, then random training-consistent fill.

WORKLOAD GENERATION ONLY (bench.py `--config 4 --table trained`, tests): the
trainer is plain C (workloads/bpe_train.c, built by workloads/Makefile or on
first use); nothing here imports the product package.

Recipe: continue BPE training from GPT-2's 50,000 merges on
generator text (the Zipf text of the bench, a different seed), taking the most
frequent adjacent pair each step; when frequencies drop below 2, fill with
random merges of existing tokens whose byte strings are unique (like the
reference's tests/helpers.hpp:85-114); where left+right already is a token,
the merge points at it (add_merge needs a unique rank and pair only,
merge_table.hpp:263-269; finalize checks concatenation, :284-296). Merges
cross word boundaries ("e" + " the", "," + " and" ...), so almost every bigram
becomes a merge junction: the adversarial case for the piece decomposition.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, List, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libbpe_train.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        src = os.path.join(HERE, "bpe_train.c")
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        _lib = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        _lib.bbt_train.argtypes = [P, I, P, P, I, P, I, I, I, ctypes.c_uint64, ctypes.c_int32, P, P, I, P, P]
        _lib.bbt_train.restype = ctypes.c_int
    return _lib


def train(text: np.ndarray, tokens: Dict[int, bytes], merges, new_merges: int, fill: bool = True,
          seed: int = 4, max_len: int = 128):
    """Runs the trainer. Returns (tokens, merges, stats) with the new merges
    appended at ranks after the base table's."""
    lib = _load()
    ids = sorted(tokens)
    if ids != list(range(len(ids))):
        raise ValueError("trainer needs dense token ids")
    tok_off = np.zeros(len(ids) + 1, np.uint64)
    np.cumsum([len(tokens[i]) for i in ids], out=tok_off[1:])
    blob = np.frombuffer(b"".join(tokens[i] for i in ids), np.uint8).copy()
    base = sorted((tuple(int(x) for x in m) for m in merges), key=lambda m: m[0])
    forced = np.array([(m[1], m[2], m[3]) for m in base], np.uint32).reshape(-1, 3)
    text = np.ascontiguousarray(text, np.uint8)
    out_m = np.zeros((max(new_merges, 1), 3), np.uint32)
    cap = new_merges * max_len + 1
    out_blob = np.zeros(cap, np.uint8)
    out_off = np.zeros(new_merges + 2, np.uint64)
    counts = np.zeros(4, np.int64)
    rc = lib.bbt_train(text.ctypes.data, text.size, blob.ctypes.data, tok_off.ctypes.data, len(ids),
                       forced.ctypes.data, forced.shape[0], new_merges, int(fill), seed, max_len,
                       out_m.ctypes.data, out_blob.ctypes.data, cap, out_off.ctypes.data, counts.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"bbt_train failed ({rc})")
    trained, filled, new_tok, last = (int(x) for x in counts)
    toks = dict(tokens)
    nid = len(ids)
    for k in range(new_tok):
        toks[nid + k] = out_blob[int(out_off[k]):int(out_off[k + 1])].tobytes()
    rank = (base[-1][0] + 1) if base else 0
    out = list(base)
    for k in range(trained + filled):
        l, r, m = (int(x) for x in out_m[k])
        assert toks[m] == toks[l] + toks[r]
        out.append((rank + k, l, r, m))
    return toks, out, {"trained": trained, "filled": filled, "new_tokens": new_tok, "last_pair_count": last}


def trained_table(tokens: Dict[int, bytes], merges: List[Tuple[int, int, int, int]], total_merges: int,
                  text_bytes: int = 16 << 20):
    """(tokens, merges, description) of the cfg4 trained table with
    `total_merges` merges in all."""
    from . import text as WX
    gen = WX.TextGen(WX.word_list(tokens))
    corpus = gen.stream(text_bytes, seed=4004)
    toks, out, st = train(corpus, tokens, merges, total_merges - len(merges))
    how = (f"continued BPE training without pre-tokenization on {text_bytes >> 20} MiB of Zipf text "
           f"(seed 4004): {st['trained']:,} trained merges (last pair count {st['last_pair_count']}), "
           f"{st['filled']:,} random consistent fill merges; {st['new_tokens']:,} new tokens")
    return toks, out, how
