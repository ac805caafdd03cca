"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU checkers.

* ``CRestatement``  -> oracle/libbpe_oracle.so, the plain-C restatement of the
  reference hot path (oracle/bpe_oracle.c, every function cites its
  reference file:line).
* ``Reference``     -> oracle/_ref/libbbpe_ref.so, the UNMODIFIED reference
  headers compiled by oracle/Makefile (present wherever it was built; the
  GPU box receives the prebuilt .so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB = os.path.join(HERE, "libbpe_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libbbpe_ref.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
NO_RANK = 0xFFFFFFFF


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def build():
    """Compile the checkers (make -C oracle)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def pack(rows: Sequence[bytes]) -> Tuple[np.ndarray, np.ndarray]:
    off = np.zeros(len(rows) + 1, np.uint64)
    if rows:
        np.cumsum([len(r) for r in rows], out=off[1:])
    data = np.frombuffer(b"".join(rows), np.uint8) if rows else np.zeros(0, np.uint8)
    return np.ascontiguousarray(data), off


class CRestatement:
    """Plain-C restatement: block_bpe / heap_bpe / naive_bpe / encode_batch."""

    def __init__(self, merges4: np.ndarray, byte_tokens: Sequence[int]):
        lib = C.CDLL(C_LIB)
        lib.orc_table_new.restype = C.c_void_p
        lib.orc_table_new.argtypes = [C.c_size_t, u32p, u32p, u32p, u32p, u32p]
        lib.orc_table_free.argtypes = [C.c_void_p]
        lib.orc_rank_of.restype = C.c_uint32
        lib.orc_rank_of.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, u32p]
        lib.orc_block_bpe.restype = C.c_int64
        lib.orc_block_bpe.argtypes = [C.c_void_p, u32p, C.c_size_t, u32p, C.c_size_t, u32p, C.c_size_t,
                                      C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        lib.orc_naive_bpe.restype = C.c_int64
        lib.orc_naive_bpe.argtypes = [C.c_void_p, u32p, C.c_size_t, u32p]
        lib.orc_heap_bpe.restype = C.c_int64
        lib.orc_heap_bpe.argtypes = [C.c_void_p, u32p, C.c_size_t, u32p]
        lib.orc_encode_batch.restype = C.c_int64
        lib.orc_encode_batch.argtypes = [C.c_void_p, u8p, u64p, C.c_size_t, u32p, u64p, C.c_uint64, C.c_int,
                                         C.POINTER(C.c_int64)]
        self.lib = lib
        m = np.ascontiguousarray(np.asarray(merges4, np.uint32).reshape(-1, 4))
        cols = [np.ascontiguousarray(m[:, i]) for i in range(4)]
        self._cols = cols
        bt = np.ascontiguousarray(np.asarray(byte_tokens, np.uint32))
        self.byte_tokens = bt
        self.h = lib.orc_table_new(m.shape[0], *[_p(c, C.c_uint32) for c in cols], _p(bt, C.c_uint32))
        if not self.h:
            raise ValueError("duplicate merge pair")

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_table_free(self.h)

    def rank_of(self, l: int, r: int) -> Optional[int]:
        v = self.lib.orc_rank_of(self.h, l, r, None)
        return None if v == NO_RANK else v

    def initial(self, data: bytes) -> List[int]:
        return [int(self.byte_tokens[b]) for b in data]

    def block_bpe(self, tokens: Sequence[int], max_passes: int = 0, trace: bool = False):
        t = np.ascontiguousarray(np.asarray(tokens, np.uint32))
        out = np.zeros(max(t.size, 1), np.uint32)
        tr = np.zeros(2 * (t.size + 1), np.uint32)
        npass, pn = C.c_size_t(), C.c_size_t()
        k = self.lib.orc_block_bpe(self.h, _p(t, C.c_uint32), t.size, _p(out, C.c_uint32), max_passes,
                                   _p(tr, C.c_uint32), t.size + 1, C.byref(npass), C.byref(pn))
        if k == -1:
            return ("max_passes", out[: pn.value].tolist(), npass.value)
        if k < 0:
            raise RuntimeError(f"orc_block_bpe failed ({k})")
        res = out[:k].tolist()
        if trace:
            return res, [(p + 1, int(tr[2 * p]), int(tr[2 * p + 1])) for p in range(npass.value)]
        return res

    def naive_bpe(self, tokens):
        t = np.ascontiguousarray(np.asarray(tokens, np.uint32))
        out = np.zeros(max(t.size, 1), np.uint32)
        k = self.lib.orc_naive_bpe(self.h, _p(t, C.c_uint32), t.size, _p(out, C.c_uint32))
        return out[:k].tolist()

    def heap_bpe(self, tokens):
        t = np.ascontiguousarray(np.asarray(tokens, np.uint32))
        out = np.zeros(max(t.size, 1), np.uint32)
        k = self.lib.orc_heap_bpe(self.h, _p(t, C.c_uint32), t.size, _p(out, C.c_uint32))
        return out[:k].tolist()

    def encode_packed(self, data: np.ndarray, offsets: np.ndarray, engine: int = 0):
        """CSR (ids, offsets); raises ValueError('row r') on an invalid byte."""
        data = np.ascontiguousarray(data, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        cap = max(int(offsets[-1]), 1)
        ids = np.zeros(cap, np.uint32)
        oo = np.zeros(n + 1, np.uint64)
        bad = C.c_int64(-1)
        k = self.lib.orc_encode_batch(self.h, _p(data, C.c_uint8) if data.size else None, _p(offsets, C.c_uint64),
                                      n, _p(ids, C.c_uint32), _p(oo, C.c_uint64), cap, engine, C.byref(bad))
        if k == -3:
            raise ValueError(f"row {bad.value}")
        if k < 0:
            raise RuntimeError(f"orc_encode_batch failed ({k})")
        return ids[:k], oo


class Reference:
    """The unmodified reference library (oracle/_ref/libbbpe_ref.so)."""

    def __init__(self, handle, lib):
        self.h = handle
        self.lib = lib

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_LIB)

    @staticmethod
    def _lib():
        lib = C.CDLL(REF_LIB)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_table_load_files.restype = C.c_void_p
        lib.ref_table_load_files.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        lib.ref_table_build.restype = C.c_void_p
        lib.ref_table_build.argtypes = [C.c_size_t, u32p, u64p, u8p, C.c_size_t, u32p]
        lib.ref_table_free.argtypes = [C.c_void_p]
        lib.ref_table_export.restype = C.c_int
        lib.ref_table_export.argtypes = [C.c_void_p, u32p, u64p, u8p, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                         u32p, C.POINTER(C.c_size_t)]
        lib.ref_add_special.restype = C.c_int
        lib.ref_add_special.argtypes = [C.c_void_p, C.c_char_p, C.c_uint32, C.c_int]
        lib.ref_encode_batch.restype = C.c_int64
        lib.ref_encode_batch.argtypes = [C.c_void_p, u8p, u64p, C.c_size_t, C.c_uint32, C.c_uint, C.c_int, C.c_int,
                                         u32p, u64p, C.c_uint64, C.c_size_t, C.c_int64]
        lib.ref_encode_heap.restype = C.c_int64
        lib.ref_encode_heap.argtypes = [C.c_void_p, u8p, u64p, C.c_size_t, C.c_uint, u32p, u64p, C.c_uint64]
        lib.ref_write_batch.restype = C.c_int64
        lib.ref_write_batch.argtypes = [C.c_void_p, u8p, u64p, C.c_size_t, C.c_uint, C.c_int, C.c_int, C.c_uint32,
                                        C.c_int, u8p, C.c_uint64]
        lib.ref_encode_pattern.restype = C.c_int64
        lib.ref_encode_pattern.argtypes = [C.c_void_p, u8p, u64p, C.c_size_t, C.c_uint, C.c_char_p, u32p, u64p,
                                           C.c_uint64]
        lib.ref_pretokenize.restype = C.c_int64
        lib.ref_pretokenize.argtypes = [u8p, C.c_size_t, C.c_char_p, u64p, C.c_size_t]
        lib.ref_block_bpe_trace.restype = C.c_int64
        lib.ref_block_bpe_trace.argtypes = [C.c_void_p, u32p, C.c_size_t, C.c_uint32, C.c_int64, u32p, u64p,
                                            C.c_size_t, C.POINTER(C.c_size_t)]
        lib.ref_naive_bpe.restype = C.c_int64
        lib.ref_naive_bpe.argtypes = [C.c_void_p, u32p, C.c_size_t, u32p]
        lib.ref_byte_token.restype = C.c_uint32
        lib.ref_byte_token.argtypes = [C.c_void_p, C.c_uint]
        lib.ref_partial.restype = C.c_size_t
        lib.ref_partial.argtypes = [u32p, C.c_size_t, C.POINTER(C.c_size_t)]
        return lib

    @classmethod
    def load_files(cls, vocab: str, merges: Optional[str], canonical: bool = False) -> "Reference":
        lib = cls._lib()
        h = lib.ref_table_load_files(vocab.encode(), merges.encode() if merges else None, 1 if canonical else 0)
        if not h:
            raise RuntimeError(lib.ref_last_error().decode())
        return cls(h, lib)

    @classmethod
    def from_arrays(cls, ids, tok_off, tok_bytes, merges4) -> "Reference":
        lib = cls._lib()
        ids = np.ascontiguousarray(ids, np.uint32)
        tok_off = np.ascontiguousarray(tok_off, np.uint64)
        tok_bytes = np.ascontiguousarray(tok_bytes, np.uint8)
        if tok_bytes.size == 0:
            tok_bytes = np.zeros(1, np.uint8)
        m = np.ascontiguousarray(np.asarray(merges4, np.uint32).reshape(-1, 4))
        h = lib.ref_table_build(ids.size, _p(ids, C.c_uint32), _p(tok_off, C.c_uint64), _p(tok_bytes, C.c_uint8),
                                m.shape[0], _p(m, C.c_uint32) if m.size else None)
        if not h:
            raise RuntimeError(lib.ref_last_error().decode())
        return cls(h, lib)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_table_free(self.h)

    def export(self):
        nt, nb, nm = C.c_size_t(), C.c_size_t(), C.c_size_t()
        self.lib.ref_table_export(self.h, None, None, None, C.byref(nt), C.byref(nb), None, C.byref(nm))
        ids = np.zeros(nt.value, np.uint32)
        off = np.zeros(nt.value + 1, np.uint64)
        blob = np.zeros(max(nb.value, 1), np.uint8)
        m4 = np.zeros((max(nm.value, 1), 4), np.uint32)
        self.lib.ref_table_export(self.h, _p(ids, C.c_uint32), _p(off, C.c_uint64), _p(blob, C.c_uint8),
                                  C.byref(nt), C.byref(nb), _p(m4, C.c_uint32), C.byref(nm))
        return ids, off, blob[: nb.value], m4[: nm.value]

    def byte_tokens(self) -> List[int]:
        return [self.lib.ref_byte_token(self.h, b) for b in range(256)]

    def add_special(self, b: bytes, tid: int, role: int = 0):
        rc = self.lib.ref_add_special(self.h, b, tid, role)
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())

    def encode_batch(self, data, offsets, workers: int = 1, block_size: int = 256, add_bos=False, add_eos=False,
                     rows_per_call: int = 65536, max_passes: int = 0):
        """encode_batch (block engine) -> CSR. Raises RuntimeError(status, msg)."""
        data = np.ascontiguousarray(data, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        cap = int(offsets[-1]) + 2 * n + 1
        ids = np.zeros(max(cap, 1), np.uint32)
        oo = np.zeros(n + 1, np.uint64)
        k = self.lib.ref_encode_batch(self.h, _p(data, C.c_uint8) if data.size else None, _p(offsets, C.c_uint64),
                                      n, block_size, workers, int(add_bos), int(add_eos), _p(ids, C.c_uint32),
                                      _p(oo, C.c_uint64), cap, rows_per_call, max_passes)
        if k < 0:
            raise RuntimeError(-k, self.lib.ref_last_error().decode())
        return ids[:k], oo

    def write_batch(self, data, offsets, pad_id: int, binary: bool, workers: int = 1, add_bos=False,
                    add_eos=False) -> bytes:
        """The reference CLI's tokenize output (blockbpe_cli.cpp:73-127): encode_batch
        with pad_id, then write_batch_jsonl / write_batch_binary (batch.hpp:157-213)."""
        data = np.ascontiguousarray(data, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        lib = self.lib
        k = lib.ref_write_batch(self.h, _p(data, C.c_uint8) if data.size else None, _p(offsets, C.c_uint64), n,
                                workers, int(add_bos), int(add_eos), pad_id, int(binary), None, 0)
        if k < 0:
            raise RuntimeError(-k, lib.ref_last_error().decode())
        out = np.zeros(max(k, 1), np.uint8)
        lib.ref_write_batch(self.h, _p(data, C.c_uint8) if data.size else None, _p(offsets, C.c_uint64), n,
                            workers, int(add_bos), int(add_eos), pad_id, int(binary), _p(out, C.c_uint8), k)
        return out[:k].tobytes()

    def encode_pattern(self, data, offsets, pattern: str = "gpt2", workers: int = 1):
        """encode_reference in pattern mode (ref_engines.hpp:119-146), heap engine."""
        data = np.ascontiguousarray(data, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        cap = max(int(offsets[-1]), 1)
        ids = np.zeros(cap, np.uint32)
        oo = np.zeros(n + 1, np.uint64)
        k = self.lib.ref_encode_pattern(self.h, _p(data, C.c_uint8) if data.size else None,
                                        _p(offsets, C.c_uint64), n, workers, pattern.encode(), _p(ids, C.c_uint32),
                                        _p(oo, C.c_uint64), cap)
        if k < 0:
            raise RuntimeError(-k, self.lib.ref_last_error().decode())
        return ids[:k], oo

    def pretokenize(self, s: bytes, pattern: str = "gpt2") -> List[int]:
        """Chunk start offsets of pattern_pretokenize (pretokenize.hpp:252-258)."""
        buf = np.frombuffer(s, np.uint8) if s else np.zeros(1, np.uint8)
        starts = np.zeros(max(len(s), 1), np.uint64)
        k = self.lib.ref_pretokenize(_p(buf, C.c_uint8), len(s), pattern.encode(), _p(starts, C.c_uint64),
                                     starts.size)
        if k < 0:
            raise RuntimeError(-k, self.lib.ref_last_error().decode())
        return starts[:k].tolist()

    def encode_heap(self, data, offsets, workers: int = 1):
        data = np.ascontiguousarray(data, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        n = offsets.size - 1
        cap = max(int(offsets[-1]), 1)
        ids = np.zeros(cap, np.uint32)
        oo = np.zeros(n + 1, np.uint64)
        k = self.lib.ref_encode_heap(self.h, _p(data, C.c_uint8) if data.size else None, _p(offsets, C.c_uint64),
                                     n, workers, _p(ids, C.c_uint32), _p(oo, C.c_uint64), cap)
        if k < 0:
            raise RuntimeError(-k, self.lib.ref_last_error().decode())
        return ids[:k], oo

    def block_bpe(self, tokens, block_size: int = 256, max_passes: int = 0):
        """-> (ids, trace[(pass, min_rank, merges)]) or raises RuntimeError((6, partial, passes))."""
        t = np.ascontiguousarray(np.asarray(tokens, np.uint32))
        out = np.zeros(max(t.size, 1), np.uint32)
        tr = np.zeros(3 * (t.size + 1), np.uint64)
        npass = C.c_size_t()
        k = self.lib.ref_block_bpe_trace(self.h, _p(t, C.c_uint32), t.size, block_size, max_passes,
                                         _p(out, C.c_uint32), _p(tr, C.c_uint64), t.size + 1, C.byref(npass))
        if k == -6:
            passes = C.c_size_t()
            m = self.lib.ref_partial(None, 0, C.byref(passes))
            part = np.zeros(max(m, 1), np.uint32)
            self.lib.ref_partial(_p(part, C.c_uint32), m, C.byref(passes))
            raise RuntimeError(6, part[:m].tolist(), passes.value)
        if k < 0:
            raise RuntimeError(-k, self.lib.ref_last_error().decode())
        return out[:k].tolist(), [tuple(int(x) for x in tr[3 * p:3 * p + 3]) for p in range(npass.value)]

    def naive_bpe(self, tokens):
        t = np.ascontiguousarray(np.asarray(tokens, np.uint32))
        out = np.zeros(max(t.size, 1), np.uint32)
        k = self.lib.ref_naive_bpe(self.h, _p(t, C.c_uint32), t.size, _p(out, C.c_uint32))
        return out[:k].tolist()
