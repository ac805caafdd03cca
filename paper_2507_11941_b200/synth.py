"""Deterministic synthetic inputs for the BASELINE.json configs.

Text: words drawn Zipf(s=1.1) from the table's " [a-z]{2,}" tokens (GPT-2:
19,655 words), 3% numbers 0-99999, sentence punctuation and capitals, newlines
with probability ~0.1, then cut into rows of the requested lengths. Fully
vectorised (numpy) so 256 MiB-16 GB corpora are generated in seconds per GB.
"""
from __future__ import annotations

import re
from typing import Optional, Tuple

import numpy as np

_WORD_RE = re.compile(rb"^ [a-z]{2,}$")


def word_list(table) -> list:
    toks = table.token_bytes()
    # Ordered by token id: BPE ids follow merge order, a proxy for frequency.
    return [toks[i] for i in sorted(toks) if _WORD_RE.match(toks[i])]


class TextGen:
    def __init__(self, words, s: float = 1.1):
        self.words = list(words)
        # Variants per word: " word", " Word" (sentence start), " word." etc.
        punct = [b".", b",", b"!", b"?", b";", b":"]
        variants = []
        for w in self.words:
            core = w[1:]
            variants.append(w)                                   # 0 plain
            variants.append(b" " + core[:1].upper() + core[1:])  # 1 capitalised
            variants.append(b"\n" + core)                        # 2 newline
            for p in punct:                                      # 3..8 punctuated
                variants.append(w + p)
        self.nvar = 3 + len(punct)
        self.n_word_var = len(variants)
        for k in range(100000):                                  # numbers 0..99999
            variants.append(b" " + str(k).encode())
        lens = np.array([len(v) for v in variants], np.int64)
        self.var_off = np.zeros(len(variants) + 1, np.int64)
        np.cumsum(lens, out=self.var_off[1:])
        self.var_blob = np.frombuffer(b"".join(variants), np.uint8)
        self.var_len = lens
        r = np.arange(1, len(self.words) + 1, dtype=np.float64)
        p = r ** -s
        self.p = p / p.sum()
        self.cdf = np.cumsum(self.p)

    def _chunk(self, rng: np.random.Generator, n_items: int) -> np.ndarray:
        w = np.searchsorted(self.cdf, rng.random(n_items) * self.cdf[-1])
        w = np.minimum(w, len(self.words) - 1)
        u = rng.random(n_items)
        var = np.zeros(n_items, np.int64)
        var[u < 0.08] = 1
        var[(u >= 0.08) & (u < 0.11)] = 2
        pm = (u >= 0.11) & (u < 0.19)
        var[pm] = 3 + rng.integers(0, self.nvar - 3, pm.sum())
        items = w * self.nvar + var
        num = rng.random(n_items) < 0.03
        items[num] = self.n_word_var + rng.integers(0, 100000, int(num.sum()))
        lens = self.var_len[items]
        starts = self.var_off[items]
        total = int(lens.sum())
        out_off = np.zeros(n_items, np.int64)
        np.cumsum(lens[:-1], out=out_off[1:])
        idx = np.repeat(starts - out_off, lens) + np.arange(total, dtype=np.int64)
        text = self.var_blob[idx]
        return text

    def stream(self, total_bytes: int, seed: int) -> np.ndarray:
        rng = np.random.default_rng(seed)
        parts = []
        have = 0
        while have < total_bytes:
            need = total_bytes - have
            n_items = max(1024, min(1 << 22, need // 6 + 64))
            c = self._chunk(rng, n_items)
            parts.append(c)
            have += c.size
        return np.concatenate(parts)[:total_bytes].copy()


def rows_fixed(gen: TextGen, n: int, length: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    data = gen.stream(n * length, seed)
    offsets = np.arange(n + 1, dtype=np.uint64) * np.uint64(length)
    return data, offsets


def rows_lengths(gen: TextGen, lengths: np.ndarray, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    lengths = np.asarray(lengths, np.uint64)
    offsets = np.zeros(lengths.size + 1, np.uint64)
    np.cumsum(lengths, out=offsets[1:])
    data = gen.stream(int(offsets[-1]), seed)
    return data, offsets


def config_rows(gen: TextGen, cfg: int, scale: float = 1.0, seed: Optional[int] = None):
    """(data, offsets, description) for BASELINE.json configs 1..5 (1-based).
    scale < 1 shrinks the row count (parity tests); lengths keep their law."""
    seed = cfg if seed is None else seed
    rng = np.random.default_rng(1000 + seed)
    if cfg == 1:
        n = max(1, int(1024 * scale))
        d, o = rows_fixed(gen, n, 1024, seed)
        return d, o, f"{n} x 1 KiB"
    if cfg == 2:
        n = max(1, int((1 << 20) * scale))
        d, o = rows_fixed(gen, n, 256, seed)
        return d, o, f"{n} x 256 B"
    if cfg == 3:
        n = max(1, int(16384 * scale))
        L = rng.integers(8192, 65536 + 1, n)
        d, o = rows_lengths(gen, L, seed)
        return d, o, f"{n} x U[8 KiB, 64 KiB]"
    if cfg == 4:
        n = max(1, int(65536 * scale))
        L = np.exp(rng.uniform(np.log(128), np.log(16384), n)).astype(np.int64)
        d, o = rows_lengths(gen, L, seed)
        return d, o, f"{n} x logU[128 B, 16 KiB]"
    if cfg == 5:
        total = int(16e9 * scale)
        mean = (65536 - 128) / np.log(65536 / 128)
        n = max(1, int(total / mean))
        L = np.exp(rng.uniform(np.log(128), np.log(65536), n)).astype(np.int64)
        d, o = rows_lengths(gen, L, seed)
        return d, o, f"{n} x logU[128 B, 64 KiB] ({int(o[-1]) / 1e9:.2f} GB)"
    raise ValueError(cfg)


_WORDISH_L = re.compile(rb"^ ?[a-z]+$")
_WORDISH_R = re.compile(rb"^[a-z]+$")


def extend_table(table, total_merges: int, seed: int = 4, max_len: int = 16):
    """Large-vocabulary table for BASELINE config 4 (128k-200k merges).

    Continues a base table with training-consistent, word-like merges: each
    new merge joins an existing " ?[a-z]+" token with an existing "[a-z]+"
    token (both created at lower ranks, so the table stays rank-consistent
    like tests/helpers.hpp:85-114) whose concatenation is not yet a token.
    Merges stay inside words, as in regex-trained vocabularies, so the
    junction-bigram set is essentially unchanged. Deterministic in `seed`.
    Returns (MergeTable, (ids, tok_off, tok_bytes, merges4))."""
    from .api import MergeTable
    ids, off, blob, m4 = table.export()
    raw = blob.tobytes()
    toks = {int(i): raw[int(off[k]):int(off[k + 1])] for k, i in enumerate(ids)}
    by_bytes = set(toks.values())
    left = [i for i, b in toks.items() if _WORDISH_L.match(b) and len(b) <= max_len - 1]
    right = [i for i, b in toks.items() if _WORDISH_R.match(b) and len(b) <= max_len - 1]
    left.sort()
    right.sort()
    rng = np.random.default_rng(seed)
    merges = [tuple(int(x) for x in row) for row in m4]
    pairs = set((m[1], m[2]) for m in merges)
    next_id = max(toks) + 1
    rank = max(m[0] for m in merges) + 1 if merges else 0
    attempts = 0
    while len(merges) < total_merges and attempts < 40 * total_merges:
        attempts += 1
        # Zipf-ish preference for low ids (frequent tokens) on both sides.
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
        merges.append((rank, li, ri, next_id))
        if _WORDISH_L.match(w):
            left.append(next_id)
        if _WORDISH_R.match(w):
            right.append(next_id)
        next_id += 1
        rank += 1
    items = sorted(toks.items())
    nids = np.array([i for i, _ in items], np.uint32)
    noff = np.zeros(len(items) + 1, np.uint64)
    np.cumsum([len(b) for _, b in items], out=noff[1:])
    nblob = np.frombuffer(b"".join(b for _, b in items), np.uint8).copy()
    nm4 = np.array(merges, np.uint32)
    return MergeTable.from_arrays(nids, noff, nblob, nm4), (nids, noff, nblob, nm4)
