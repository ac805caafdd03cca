"""Deterministic synthetic inputs for the BASELINE.json configs.

WORKLOAD GENERATION ONLY (tests and bench.py): pure numpy, imports nothing
from the product package, so the reference arm of bench.py generates the same
bytes without loading the B200 library.

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
    """The table's " [a-z]{2,}" tokens ordered by id (BPE ids follow merge
    order, a proxy for frequency). `table`: a dict id -> bytes, or any object
    with token_bytes() returning one."""
    toks = table if isinstance(table, dict) else table.token_bytes()
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

    BLOCK = 1 << 24  # the stream is generated in independently seeded 16 MiB blocks

    def _block(self, seed: int, b: int) -> np.ndarray:
        rng = np.random.default_rng([seed, b])
        parts, have = [], 0
        while have < self.BLOCK:
            c = self._chunk(rng, max(1024, (self.BLOCK - have) // 6 + 64))
            parts.append(c)
            have += c.size
        return np.concatenate(parts)[: self.BLOCK]

    def stream_range(self, start: int, end: int, seed: int) -> np.ndarray:
        """Bytes [start, end) of the stream for `seed`; any range is generated
        without the bytes before it (sharded corpora: each rank makes its own)."""
        out = np.empty(max(end - start, 0), np.uint8)
        pos = start
        while pos < end:
            b = pos // self.BLOCK
            blk = self._block(seed, b)
            lo = pos - b * self.BLOCK
            hi = min(self.BLOCK, end - b * self.BLOCK)
            out[pos - start: pos - start + hi - lo] = blk[lo:hi]
            pos += hi - lo
        return out

    def stream(self, total_bytes: int, seed: int) -> np.ndarray:
        return self.stream_range(0, total_bytes, seed)


def _rows(gen, offsets: np.ndarray, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    if hasattr(gen, "rows"):  # CorpusGen: ingest_corpus semantics
        return gen.rows(offsets)
    return gen.stream(int(offsets[-1]), seed), offsets


def rows_fixed(gen, n: int, length: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    offsets = np.arange(n + 1, dtype=np.uint64) * np.uint64(length)
    return _rows(gen, offsets, seed)


def rows_lengths(gen, lengths: np.ndarray, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    lengths = np.asarray(lengths, np.uint64)
    offsets = np.zeros(lengths.size + 1, np.uint64)
    np.cumsum(lengths, out=offsets[1:])
    return _rows(gen, offsets, seed)


def cfg5_lengths(scale: float, rng: np.random.Generator) -> np.ndarray:
    """Row lengths of the cfg5 corpus: 16e9 * scale bytes, logU[128 B, 64 KiB]."""
    total = int(16e9 * scale)
    mean = (65536 - 128) / np.log(65536 / 128)
    n = max(1, int(total / mean))
    return np.exp(rng.uniform(np.log(128), np.log(65536), n)).astype(np.int64)


def cfg5_shard(gen, scale: float, parts: int, part: int, bounds=None, seed: int = 5):
    """Shard `part` of `parts` of ONE cfg5 corpus (strong scaling): the row
    lengths of the whole corpus, contiguous row bounds (byte-balanced unless
    `bounds` is given, e.g. from the encoder's cost-balanced partitioner) and
    only this shard's bytes. Returns (data, offsets from 0, description,
    (r0, r1), corpus offsets)."""
    rng = np.random.default_rng(1000 + seed)
    L = cfg5_lengths(scale, rng)
    off = np.zeros(L.size + 1, np.uint64)
    np.cumsum(L.astype(np.uint64), out=off[1:])
    if bounds is None:
        tgt = (np.arange(parts + 1, dtype=np.float64) * float(off[-1]) / parts)
        bounds = np.searchsorted(off, tgt.astype(np.uint64), side="left").astype(np.int64)
        bounds[0], bounds[-1] = 0, L.size
    r0, r1 = int(bounds[part]), int(bounds[part + 1])
    b0, b1 = int(off[r0]), int(off[r1])
    so = (off[r0:r1 + 1] - off[r0]).astype(np.uint64)
    if hasattr(gen, "rows"):
        data, so = gen.rows(so)  # (cyclic corpus: shard-relative rows)
    else:
        data = gen.stream_range(b0, b1, seed)
    desc = (f"rows [{r0}, {r1}) of {L.size} x logU[128 B, 64 KiB] ({int(off[-1]) / 1e9:.2f} GB corpus, "
            f"shard {part + 1}/{parts}: {(b1 - b0) / 1e9:.2f} GB)")
    return data, so, desc, (r0, r1), off


def config_rows(gen, cfg: int, scale: float = 1.0, seed: Optional[int] = None):
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
        L = cfg5_lengths(scale, rng)
        d, o = rows_lengths(gen, L, seed)
        return d, o, f"{L.size} x logU[128 B, 64 KiB] ({int(o[-1]) / 1e9:.2f} GB)"
    raise ValueError(cfg)


# ---------------------------------------------------------------------------
# Further text classes (bench legs; SURVEY.md §8d "a second, easier text class")


def _trim_utf8_tail(data: np.ndarray, offsets: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Drops an incomplete UTF-8 sequence at the end of each row, as
    ingest_corpus does (reference bench.hpp:149-158)."""
    n = offsets.size - 1
    keep = np.diff(offsets.astype(np.int64))
    starts = offsets[:-1].astype(np.int64)
    ends = starts + keep
    p = ends - 1
    back = np.zeros(n, np.int64)
    for _ in range(3):  # step back over continuation bytes (at most 3)
        ok = (p > starts) & (back < 3) & ((data[np.maximum(p, 0)] & 0xC0) == 0x80)
        p = np.where(ok, p - 1, p)
        back += ok
    lead = data[np.maximum(p, 0)]
    need = np.where((lead & 0x80) == 0, 1, np.where((lead & 0xE0) == 0xC0, 2,
                    np.where((lead & 0xF0) == 0xE0, 3, np.where((lead & 0xF8) == 0xF0, 4, 1))))
    cut = (keep > 0) & (need > ends - p)
    new_len = np.where(cut, p - starts, keep)
    if not cut.any():
        return data, offsets
    mask = np.ones(data.size, bool)
    for s, e, l in zip(starts[cut], ends[cut], new_len[cut]):
        mask[s + l:e] = False
    out_off = np.zeros(n + 1, np.uint64)
    np.cumsum(new_len.astype(np.uint64), out=out_off[1:])
    return data[mask], out_off


class CorpusGen:
    """The reference's own bench input (ingest_corpus, bench.hpp:120-160): rows
    cut cyclically from tests/testdata/corpus.txt (committed as
    tests/golden/corpus.txt), row i of a fixed-length batch starting at
    (i * seq_len) mod |corpus|; a trailing incomplete UTF-8 sequence is dropped."""

    def __init__(self, corpus: bytes):
        self.c = np.frombuffer(corpus, np.uint8)

    def stream_range(self, start: int, end: int, seed: int = 0) -> np.ndarray:
        idx = np.arange(start, end, dtype=np.int64) % self.c.size
        return self.c[idx]

    def stream(self, total_bytes: int, seed: int = 0) -> np.ndarray:
        return self.stream_range(0, total_bytes)

    def rows(self, offsets: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
        data = self.stream(int(offsets[-1]))
        return _trim_utf8_tail(data, offsets)


def _items(rng, lens: np.ndarray, alphabet: np.ndarray, prefix: np.ndarray = None):
    """Items of random symbols from `alphabet` (uint8 array), item k of
    lens[k] symbols, optionally preceded by one prefix byte each."""
    body = alphabet[rng.integers(0, alphabet.size, int(lens.sum()))]
    if prefix is None:
        return body, lens
    out_len = lens + 1
    out = np.empty(int(out_len.sum()), np.uint8)
    st = np.zeros(lens.size, np.int64)
    np.cumsum(out_len[:-1], out=st[1:])
    out[st] = prefix
    m = np.ones(out.size, bool)
    m[st] = False
    out[m] = body
    return out, out_len


class MixedGen:
    """Text the table's vocabulary does not hand to the encoder: random-letter
    words (not vocabulary entries), capitalised words, long numbers, hex
    literals, source-code-like identifiers and punctuation, CJK (3-byte UTF-8)
    runs and Cyrillic (2-byte) words. Items are drawn independently and
    uniformly, so repetition is rare (few pieces hit the piece memo or repeat
    within a call). Deterministic per (seed, 16 MiB block)."""

    BLOCK = 1 << 24
    LOWER = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", np.uint8)
    DIGITS = np.frombuffer(b"0123456789", np.uint8)
    HEX = np.frombuffer(b"0123456789abcdef", np.uint8)
    IDENT = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz_ABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789", np.uint8)
    PUNCT = [b"(", b")", b" = ", b";\n", b"\n    ", b"->", b" {\n", b"}\n", b", ", b".", b"[", b"]", b" + ", b"::",
             b" == ", b"\n\n", b"\t", b"  ", b" */", b" // "]

    def _cjk(self, rng, n):
        lens = rng.integers(2, 13, n)
        cp = rng.integers(0x4E00, 0xA000, int(lens.sum()))
        b = np.stack([0xE0 | (cp >> 12), 0x80 | ((cp >> 6) & 0x3F), 0x80 | (cp & 0x3F)], 1).astype(np.uint8)
        return b.reshape(-1), lens * 3

    def _cyr(self, rng, n):
        lens = rng.integers(3, 11, n)
        cp = rng.integers(0x430, 0x450, int(lens.sum()))
        b = np.stack([0xC0 | (cp >> 6), 0x80 | (cp & 0x3F)], 1).astype(np.uint8)
        body, bl = b.reshape(-1), lens * 2
        out_len = bl + 1
        out = np.empty(int(out_len.sum()), np.uint8)
        st = np.zeros(n, np.int64)
        np.cumsum(out_len[:-1], out=st[1:])
        out[st] = 0x20
        m = np.ones(out.size, bool)
        m[st] = False
        out[m] = body
        return out, out_len

    def _chunk(self, rng, n):
        kinds = rng.choice(8, n, p=[0.32, 0.05, 0.08, 0.04, 0.2, 0.13, 0.12, 0.06])
        parts = []
        for k in range(8):
            m = int((kinds == k).sum())
            if k == 0:    # random lowercase words
                b, l = _items(rng, rng.integers(2, 11, m), self.LOWER, np.uint8(0x20))
            elif k == 1:  # capitalised random words
                b, l = _items(rng, rng.integers(2, 11, m), self.LOWER, np.uint8(0x20))
                st = np.zeros(m, np.int64)
                np.cumsum(l[:-1], out=st[1:])
                b[st + 1] -= 32
            elif k == 2:  # long numbers
                b, l = _items(rng, rng.integers(5, 21, m), self.DIGITS, np.uint8(0x20))
            elif k == 3:  # hex literals (" 0" + "x..." )
                b, l = _items(rng, rng.integers(8, 17, m), self.HEX, np.uint8(ord("x")))
                b, l = _items_prefix(b, l, b" 0")
            elif k == 4:  # identifiers
                b, l = _items(rng, rng.integers(3, 15, m), self.IDENT)
            elif k == 5:  # code punctuation
                sel = rng.integers(0, len(self.PUNCT), m)
                pl = np.array([len(p) for p in self.PUNCT], np.int64)
                pb = np.frombuffer(b"".join(self.PUNCT), np.uint8)
                po = np.zeros(len(self.PUNCT), np.int64)
                np.cumsum(pl[:-1], out=po[1:])
                l = pl[sel]
                oo = np.zeros(m, np.int64)
                np.cumsum(l[:-1], out=oo[1:])
                b = pb[np.repeat(po[sel] - oo, l) + np.arange(int(l.sum()))]
            elif k == 6:
                b, l = self._cjk(rng, m)
            else:
                b, l = self._cyr(rng, m)
            parts.append((b, l, np.nonzero(kinds == k)[0]))
        # interleave items in the drawn order
        lens = np.zeros(n, np.int64)
        src_start = np.zeros(n, np.int64)
        blob = np.concatenate([p[0] for p in parts])
        base = 0
        for b, l, pos in parts:
            st = np.zeros(l.size, np.int64)
            if l.size:
                np.cumsum(l[:-1], out=st[1:])
            lens[pos] = l
            src_start[pos] = st + base
            base += b.size
        oo = np.zeros(n, np.int64)
        np.cumsum(lens[:-1], out=oo[1:])
        return blob[np.repeat(src_start - oo, lens) + np.arange(int(lens.sum()))]

    def _block(self, seed: int, b: int) -> np.ndarray:
        rng = np.random.default_rng([seed, 7, b])
        parts, have = [], 0
        while have < self.BLOCK:
            c = self._chunk(rng, max(1024, (self.BLOCK - have) // 6 + 64))
            parts.append(c)
            have += c.size
        return np.concatenate(parts)[: self.BLOCK]

    stream_range = TextGen.stream_range
    stream = TextGen.stream


def _items_prefix(b: np.ndarray, l: np.ndarray, prefix: bytes):
    p = np.frombuffer(prefix, np.uint8)
    out_len = l + p.size
    out = np.empty(int(out_len.sum()), np.uint8)
    st = np.zeros(l.size, np.int64)
    if l.size:
        np.cumsum(out_len[:-1], out=st[1:])
    m = np.ones(out.size, bool)
    for j in range(p.size):
        out[st + j] = p[j]
        m[st + j] = False
    out[m] = b
    return out, out_len


def make_gen(kind: str, tokens=None, corpus: bytes = None):
    """Text generator by class name: 'zipf' (the table's words),
    'corpus' (the reference bench's corpus.txt), 'mixed' (MixedGen)."""
    if kind == "zipf":
        return TextGen(word_list(tokens))
    if kind == "corpus":
        return CorpusGen(corpus)
    if kind == "mixed":
        return MixedGen()
    raise ValueError(kind)
