"""Merge tables for the workloads, built WITHOUT the product package.

WORKLOAD GENERATION ONLY. A table here is plain data: `tokens` (dict id ->
bytes) and `merges` (list of (rank, left, right, merged)). Both bench arms
load the same table from files: the B200 arm through its own loader, the
reference arm through the reference's `load_merge_table_files`
(merge_table.hpp:513-522; gpt2 format :399-459, canonical JSON :473-497).
"""
from __future__ import annotations

import json
import os
import re
from typing import Dict, List, Tuple

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GPT2_DIR = os.path.join(ROOT, "tests", "golden", "gpt2")
GPT2_VOCAB = os.path.join(GPT2_DIR, "vocab.json")
GPT2_MERGES = os.path.join(GPT2_DIR, "merges.txt")

Merge = Tuple[int, int, int, int]


def _byte_unicode():
    """The GPT-2 byte <-> codepoint bijection (merge_table.hpp:30-53): bytes
    33-126, 161-172, 174-255 map to themselves, the rest to 256+k in order."""
    bs = list(range(33, 127)) + list(range(161, 173)) + list(range(174, 256))
    cs = bs[:]
    k = 0
    for b in range(256):
        if b not in bs:
            bs.append(b)
            cs.append(256 + k)
            k += 1
    return {chr(c): b for b, c in zip(bs, cs)}


def gpt2_table(vocab: str = GPT2_VOCAB, merges: str = GPT2_MERGES) -> Tuple[Dict[int, bytes], List[Merge]]:
    """tokens, merges of the GPT-2 files (rank = line order, merged = the
    vocab entry of left+right), as the reference's gpt2 loader reads them."""
    inv = _byte_unicode()
    with open(vocab, encoding="utf-8") as f:
        v = json.load(f)
    tokens = {int(i): bytes(inv[ch] for ch in s) for s, i in v.items()}
    out = []
    with open(merges, encoding="utf-8") as f:
        lines = f.read().split("\n")
    rank = 0
    for k, line in enumerate(lines):
        line = line.rstrip("\r")
        if (k == 0 and line.startswith("#version")) or not line:
            continue
        a, b = line.split(" ")
        out.append((rank, v[a], v[b], v[a + b]))
        rank += 1
    return tokens, out


def write_canonical(path: str, tokens: Dict[int, bytes], merges: List[Merge]) -> str:
    """Canonical JSON (README "File formats"; merge_table.hpp:473-497)."""
    doc = {"tokens": [[i, list(tokens[i])] for i in sorted(tokens)],
           "merges": [list(map(int, m)) for m in merges]}
    with open(path, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
    return path


def arrays(tokens: Dict[int, bytes], merges: List[Merge]):
    """(ids u32, tok_off u64, tok_bytes u8, merges4 u32 [M,4]) -- the layout of
    bbpe_table_create / the oracle's table builders."""
    items = sorted(tokens.items())
    ids = np.array([i for i, _ in items], np.uint32)
    off = np.zeros(len(items) + 1, np.uint64)
    np.cumsum([len(b) for _, b in items], out=off[1:])
    blob = np.frombuffer(b"".join(b for _, b in items), np.uint8).copy()
    m4 = np.array(merges, np.uint32).reshape(-1, 4)
    return ids, off, blob, m4


_WORDISH_L = re.compile(rb"^ ?[a-z]+$")
_WORDISH_R = re.compile(rb"^[a-z]+$")


def extend_wordlevel(tokens: Dict[int, bytes], merges: List[Merge], total_merges: int, seed: int = 4,
                     max_len: int = 16):
    """Large-vocabulary table, word-level variant (round 1's cfg4 table).

    Continues a base table with training-consistent, word-like merges: each
    new merge joins an existing " ?[a-z]+" token with an existing "[a-z]+"
    token (both created at lower ranks, so the table stays rank-consistent
    like tests/helpers.hpp:85-114) whose concatenation is not yet a token.
    Merges stay inside words, so the junction-bigram set is essentially
    unchanged (the easy case for the piece decomposition). Deterministic."""
    toks = dict(tokens)
    by_bytes = set(toks.values())
    left = sorted(i for i, b in toks.items() if _WORDISH_L.match(b) and len(b) <= max_len - 1)
    right = sorted(i for i, b in toks.items() if _WORDISH_R.match(b) and len(b) <= max_len - 1)
    rng = np.random.default_rng(seed)
    out = [tuple(int(x) for x in m) for m in merges]
    pairs = set((m[1], m[2]) for m in out)
    next_id = max(toks) + 1
    rank = max(m[0] for m in out) + 1 if out else 0
    attempts = 0
    while len(out) < total_merges and attempts < 40 * total_merges:
        attempts += 1
        li = left[min(int(rng.pareto(1.2) * 300), len(left) - 1)]
        ri = right[min(int(rng.pareto(1.2) * 300), len(right) - 1)]
        if (li, ri) in pairs:
            continue
        w = toks[li] + toks[ri]
        if len(w) > max_len or w in by_bytes:
            continue
        toks[next_id] = w
        by_bytes.add(w)
        pairs.add((li, ri))
        out.append((rank, li, ri, next_id))
        if _WORDISH_L.match(w):
            left.append(next_id)
        if _WORDISH_R.match(w):
            right.append(next_id)
        next_id += 1
        rank += 1
    return toks, out
