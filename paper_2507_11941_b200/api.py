"""Python mirror of the reference's batch-encode API over the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference library
(`namespace blockbpe`, /root/reference/proj/include/blockbpe):

  load_merge_table_files  merge_table.hpp:513-522    MergeTable   merge_table.hpp:223-305
  SpecialTokenSet         merge_table.hpp:309-369    validate_specials 374-385
  split_specials          pretokenize.hpp:32-57      bytes_to_initial_tokens 60-71
  BlockConfig             block_engine.hpp:18-32     block_bpe    block_engine.hpp:268-310
  BatchEncoding/Limits    batch.hpp:21-42            encode_single/encode_batch 46-126
  decode / decode_batch   merge_table.hpp:565-579, batch.hpp:128-154
  write/read_batch_jsonl, write/read_batch_binary    batch.hpp:159-242

All token merging runs on the GPU through libbbpe_b200.so; the host side here
only packs rows, splits specials, and assembles padding/masks exactly like
encode_batch does. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import json
import re
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence, Tuple, Union

import numpy as np

from . import _lib
from ._lib import LIB, Config, Stats, TableInfo

# ---------------------------------------------------------------------------
# Errors (types.hpp:32-70)


class Error(RuntimeError):
    pass


class UsageError(Error):
    pass


class ParseError(Error):
    pass


class IntegrityError(Error):
    pass


class DecodeError(Error):
    pass


class ContractViolation(Error):
    pass


class MaxPassesError(Error):
    def __init__(self, what: str, partial_tokens: Sequence[int], passes_run: int):
        super().__init__(what)
        self.partial_tokens = list(partial_tokens)
        self.passes_run = passes_run


_STATUS = {1: UsageError, 2: ParseError, 3: IntegrityError, 4: DecodeError, 5: ContractViolation,
           6: MaxPassesError, 7: Error}


def _check(rc: int):
    if rc != 0:
        msg = LIB.bbpe_last_error().decode(errors="replace")
        cls = _STATUS.get(rc, Error)
        if cls is MaxPassesError:
            raise MaxPassesError(msg, [], 0)
        raise cls(msg)


def _p(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


NO_RANK = 0xFFFFFFFF
INVALID_TOKEN = 0xFFFFFFFF

# ---------------------------------------------------------------------------
# Config


@dataclass
class BlockConfig:
    """block_engine.hpp:18-32. block_size never changes results."""

    block_size: int = 256
    max_passes: Optional[int] = None

    def validate(self):
        bs = self.block_size
        if bs < 32 or bs > 1024 or (bs & (bs - 1)) != 0:
            raise UsageError(f"block_size must be a power of two in [32, 1024], got {bs}")
        if self.max_passes is not None and self.max_passes < 1:
            raise UsageError("max_passes must be >= 1")


def coarsening_factor(seq_len: int, config: BlockConfig) -> int:
    """block_engine.hpp:36-39: d = ceil(n / block_size)."""
    config.validate()
    return (seq_len + config.block_size - 1) // config.block_size


@dataclass
class BatchLimits:
    max_len: Optional[int] = None


# ---------------------------------------------------------------------------
# Merge table


_FORMATS = {"gpt2": 0, "json": 1, "canonical_json": 1, "binary": 2, "bbpt": 2}


def parse_vocab_format(name: str) -> int:
    if name not in _FORMATS:
        raise UsageError(f'unknown vocab format "{name}"')
    return _FORMATS[name]


class MergeTable:
    """Immutable merge table (merge_table.hpp:223-305) owned by the C-ABI.

    Device replicas are uploaded lazily, once per GPU."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        self._tokens = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            LIB.bbpe_table_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @classmethod
    def load_files(cls, vocab_path: str, merges_path: Optional[str] = None,
                   fmt: Union[str, int] = "gpt2") -> "MergeTable":
        f = parse_vocab_format(fmt) if isinstance(fmt, str) else int(fmt)
        h = C.c_void_p()
        _check(LIB.bbpe_table_load_files(vocab_path.encode(), merges_path.encode() if merges_path else None,
                                         f, C.byref(h)))
        return cls(h)

    @classmethod
    def build(cls, tokens: Iterable[Tuple[int, bytes]],
              merges: Iterable[Tuple[int, int, int, int]]) -> "MergeTable":
        """tokens: (id, bytes); merges: (rank, left, right, merged).
        Same checks as add_token/add_merge/finalize (merge_table.hpp:257-297)."""
        toks = list(tokens)
        ids = np.array([t[0] for t in toks], dtype=np.uint32)
        lens = np.array([len(t[1]) for t in toks], dtype=np.uint64)
        off = np.zeros(len(toks) + 1, dtype=np.uint64)
        if len(toks):
            np.cumsum(lens, out=off[1:])
        blob = np.frombuffer(b"".join(t[1] for t in toks), dtype=np.uint8).copy() if toks else np.zeros(1, np.uint8)
        m = np.array(list(merges), dtype=np.uint32).reshape(-1, 4)
        return cls.from_arrays(ids, off, blob, m)

    @classmethod
    def from_arrays(cls, ids, tok_off, tok_bytes, merges4) -> "MergeTable":
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        tok_off = np.ascontiguousarray(tok_off, dtype=np.uint64)
        tok_bytes = np.ascontiguousarray(tok_bytes, dtype=np.uint8)
        if tok_bytes.size == 0:
            tok_bytes = np.zeros(1, np.uint8)
        merges4 = np.ascontiguousarray(merges4, dtype=np.uint32).reshape(-1, 4)
        h = C.c_void_p()
        _check(LIB.bbpe_table_create(len(ids), _p(ids, C.c_uint32), _p(tok_off, C.c_uint64),
                                     _p(tok_bytes, C.c_uint8), merges4.shape[0],
                                     _p(merges4, C.c_uint32) if merges4.size else None, C.byref(h)))
        return cls(h)

    def info(self) -> dict:
        i = TableInfo()
        _check(LIB.bbpe_table_get_info(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in i._fields_}

    def token_count(self) -> int:
        return self.info()["token_count"]

    def merge_count(self) -> int:
        return self.info()["merge_count"]

    def base_size(self) -> int:
        return self.info()["base_size"]

    def byte_token(self, b: int) -> int:
        return LIB.bbpe_table_byte_token(self._h, b)

    def rank_of(self, left: int, right: int) -> Optional[int]:
        r = LIB.bbpe_table_rank_of(self._h, left, right, None)
        return None if r == NO_RANK else r

    def merged_of(self, left: int, right: int) -> Optional[int]:
        m = C.c_uint32()
        r = LIB.bbpe_table_rank_of(self._h, left, right, C.byref(m))
        return None if r == NO_RANK else m.value

    def save_binary(self, path: str):
        _check(LIB.bbpe_table_save_binary(self._h, path.encode()))

    def export(self):
        """(ids u32[T], tok_off u64[T+1], tok_bytes u8[B], merges u32[M,4]) sorted by id / rank."""
        nt, nb, nm = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(LIB.bbpe_table_export(self._h, None, None, None, C.byref(nt), C.byref(nb), None, C.byref(nm)))
        ids = np.zeros(nt.value, np.uint32)
        off = np.zeros(nt.value + 1, np.uint64)
        blob = np.zeros(max(nb.value, 1), np.uint8)
        m4 = np.zeros((max(nm.value, 1), 4), np.uint32)
        _check(LIB.bbpe_table_export(self._h, _p(ids, C.c_uint32), _p(off, C.c_uint64), _p(blob, C.c_uint8),
                                     C.byref(nt), C.byref(nb), _p(m4, C.c_uint32), C.byref(nm)))
        return ids, off, blob[: nb.value], m4[: nm.value]

    def token_bytes(self) -> dict:
        if self._tokens is None:
            ids, off, blob, _ = self.export()
            raw = blob.tobytes()
            self._tokens = {int(i): raw[int(off[k]):int(off[k + 1])] for k, i in enumerate(ids)}
        return self._tokens

    def bytes_of(self, tid: int) -> Optional[bytes]:
        return self.token_bytes().get(tid)

    def max_token_bytes(self) -> int:
        """Length of the longest token (bounds a decode's output)."""
        if getattr(self, "_max_tok", None) is None:
            _, off, _, _ = self.export()
            self._max_tok = int((off[1:] - off[:-1]).max()) if off.size > 1 else 1
        return self._max_tok


def load_merge_table_files(vocab_path: str, merges_path: Optional[str], fmt: Union[str, int] = "gpt2") -> MergeTable:
    return MergeTable.load_files(vocab_path, merges_path, fmt)


# ---------------------------------------------------------------------------
# Specials (host side; merge_table.hpp:309-385, pretokenize.hpp:16-57)


class SpecialTokenSet:
    def __init__(self):
        self._entries: List[Tuple[bytes, int]] = []
        self._bos: Optional[int] = None
        self._eos: Optional[int] = None

    def add(self, b: Union[bytes, str], tid: int):
        b = b.encode() if isinstance(b, str) else bytes(b)
        if not b:
            raise UsageError("special token byte string may not be empty")
        if any(e[0] == b for e in self._entries):
            raise UsageError(f'duplicate special token "{b.decode(errors="replace")}"')
        i = 0
        while i < len(self._entries) and len(self._entries[i][0]) >= len(b):
            i += 1
        self._entries.insert(i, (b, tid))

    def empty(self) -> bool:
        return not self._entries

    def size(self) -> int:
        return len(self._entries)

    def entries(self):
        return list(self._entries)

    def bytes_of(self, tid: int) -> Optional[bytes]:
        for b, i in self._entries:
            if i == tid:
                return b
        return None

    def contains_id(self, tid: int) -> bool:
        return any(i == tid for _, i in self._entries)

    def match(self, text: bytes, pos: int):
        for b, i in self._entries:
            if text.startswith(b, pos):
                return len(b), i
        return None

    def _require(self, b, what):
        b = b.encode() if isinstance(b, str) else bytes(b)
        for e, i in self._entries:
            if e == b:
                return i
        raise UsageError(f'{what} token "{b.decode(errors="replace")}" is not in the special token set')

    def set_bos(self, b):
        self._bos = self._require(b, "bos")

    def set_eos(self, b):
        self._eos = self._require(b, "eos")

    def bos_id(self):
        return self._bos

    def eos_id(self):
        return self._eos


def validate_specials(table: MergeTable, specials: SpecialTokenSet):
    """merge_table.hpp:374-385."""
    _, _, _, m4 = table.export()
    merged = set(int(x) for x in m4[:, 3]) if len(m4) else set()
    for b, tid in specials.entries():
        tb = table.bytes_of(tid)
        if tb is not None and len(tb) == 1 and table.byte_token(tb[0]) == tid:
            raise IntegrityError(f"special id {tid} is a base byte token")
    for b, tid in specials.entries():
        if tid in merged:
            raise IntegrityError(f"special id {tid} collides with a merge-derived token")


@dataclass
class Segment:
    kind: str  # "literal" | "special"
    bytes: bytes
    special_id: Optional[int] = None


def split_specials(data: bytes, specials: SpecialTokenSet) -> List[Segment]:
    """pretokenize.hpp:32-57: greedy longest-first special matching."""
    out: List[Segment] = []
    pending = bytearray()
    pos = 0
    if specials.empty():
        return [Segment("literal", bytes(data))] if data else []
    while pos < len(data):
        m = specials.match(data, pos)
        if m:
            if pending:
                out.append(Segment("literal", bytes(pending)))
                pending = bytearray()
            out.append(Segment("special", data[pos:pos + m[0]], m[1]))
            pos += m[0]
            continue
        pending.append(data[pos])
        pos += 1
    if pending:
        out.append(Segment("literal", bytes(pending)))
    return out


# ---------------------------------------------------------------------------
# Packed batches


def pack_rows(rows: Sequence[Union[bytes, str]]) -> Tuple[np.ndarray, np.ndarray]:
    """List of rows -> (bytes u8[total], offsets u64[n+1])."""
    bs = [r.encode() if isinstance(r, str) else bytes(r) for r in rows]
    offsets = np.zeros(len(bs) + 1, dtype=np.uint64)
    if bs:
        np.cumsum(np.fromiter((len(b) for b in bs), dtype=np.uint64, count=len(bs)), out=offsets[1:])
    data = np.frombuffer(b"".join(bs), dtype=np.uint8) if bs else np.zeros(0, np.uint8)
    return data, offsets


ENGINES = {"pieces": 0, "block": 1}


GPT2_PATTERN = r"""'s|'t|'re|'ve|'m|'ll|'d| ?\p{L}+| ?\p{N}+| ?[^\s\p{L}\p{N}]+|\s+(?!\S)|\s+"""


def _pattern_code(pattern: Optional[str]) -> int:
    """None: byte-level (encode_batch); "gpt2" or the published gpt2 pattern
    (pretokenize.hpp:86-87): the device splitter."""
    if pattern is None:
        return 0
    if pattern in ("gpt2", GPT2_PATTERN):
        return 1
    raise UsageError(f'only the gpt2 split pattern runs on the device, got "{pattern}"')


class Encoder:
    """One encode context on one GPU (bbpe_ctx). Single-caller, like PhasePool."""

    def __init__(self, device: int = 0, config: Optional[BlockConfig] = None, engine: str = "pieces",
                 wave_bytes: int = 0, piece_memo: bool = True, dedup: bool = True, pattern: Optional[str] = None):
        self.device = device
        self.dedup = dedup
        self.pattern = pattern
        self.config = config or BlockConfig()
        self.engine = engine
        self.wave_bytes = wave_bytes
        self.piece_memo = piece_memo
        self._h = C.c_void_p()
        self._sp_key = ()
        _check(LIB.bbpe_ctx_create(device, C.byref(self._cfg()), C.byref(self._h)))

    def _cfg(self) -> Config:
        self.config.validate()
        if self.engine not in ENGINES:
            raise UsageError(f'unknown engine "{self.engine}"')
        return Config(self.config.block_size, self.config.max_passes or 0, ENGINES[self.engine], self.wave_bytes,
                      1 if self.piece_memo else 0, 0 if self.dedup else 1, _pattern_code(self.pattern))

    def set_config(self, config: BlockConfig = None, engine: str = None, wave_bytes: int = None,
                   piece_memo: bool = None, dedup: bool = None, pattern: Optional[str] = "unchanged"):
        if config is not None:
            self.config = config
        if engine is not None:
            self.engine = engine
        if wave_bytes is not None:
            self.wave_bytes = wave_bytes
        if piece_memo is not None:
            self.piece_memo = piece_memo
        if dedup is not None:
            self.dedup = dedup
        if pattern != "unchanged":
            self.pattern = pattern
        _check(LIB.bbpe_ctx_set_config(self._h, C.byref(self._cfg())))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            LIB.bbpe_ctx_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def prepare(self, table: MergeTable):
        _check(LIB.bbpe_ctx_prepare(self._h, table.handle))

    def kernel_launches(self) -> int:
        return LIB.bbpe_ctx_kernel_launches(self._h)

    KERNELS = ("k_tile_first", "k_pieces", "k_dedup", "k_merge", "k_refs", "k_long_pieces", "k_tile_scan",
               "k_gather")

    def kernel_times(self, reset: bool = True) -> Tuple[dict, int]:
        """Per-kernel device ms (CUDA events on the launching stream) summed
        over the encodes since the last reset, and the number of encodes."""
        ms = (C.c_double * len(self.KERNELS))()
        calls = C.c_uint64()
        _check(LIB.bbpe_ctx_kernel_times(self._h, ms, C.byref(calls), 1 if reset else 0))
        return dict(zip(self.KERNELS, list(ms))), calls.value

    PIECE_STATS = ("pieces", "memo_hits", "merge_pieces", "long_pieces", "long_bytes", "merged_after_dedupe",
                   "input_bytes")

    def piece_stats(self, reset: bool = True) -> dict:
        """What the piece decomposition did over the encodes since the last
        reset (bbpe_ctx_piece_stats), with memo hit rate and long-byte share."""
        v = np.zeros(len(self.PIECE_STATS), np.uint64)
        _check(LIB.bbpe_ctx_piece_stats(self._h, _p(v, C.c_uint64), 1 if reset else 0))
        d = {k: int(x) for k, x in zip(self.PIECE_STATS, v)}
        d["memo_hit_rate"] = d["memo_hits"] / d["pieces"] if d["pieces"] else None
        d["long_byte_fraction"] = d["long_bytes"] / d["input_bytes"] if d["input_bytes"] else None
        return d

    def encode_packed(self, table: MergeTable, data: np.ndarray, offsets: np.ndarray,
                      out_ids: Optional[np.ndarray] = None, out_offsets: Optional[np.ndarray] = None):
        """Host buffers -> CSR (ids u32, offsets u64[n+1]), stats dict."""
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        total = int(offsets[-1] - offsets[0]) if n >= 0 else 0
        if out_ids is None:
            out_ids = np.empty(max(total, 1), dtype=np.uint32)
        if out_offsets is None:
            out_offsets = np.empty(n + 1, dtype=np.uint64)
        st = Stats()
        dptr = _p(data, C.c_uint8) if data.size else None
        _check(LIB.bbpe_encode(self._h, table.handle, dptr, _p(offsets, C.c_uint64), n,
                               _p(out_ids, C.c_uint32), out_ids.size, _p(out_offsets, C.c_uint64), C.byref(st)))
        ntok = int(out_offsets[-1]) if n >= 0 else 0
        return out_ids[:ntok], out_offsets, st.as_dict()

    def encode_rows(self, table: MergeTable, rows: Sequence[Union[bytes, str]]) -> List[List[int]]:
        data, offsets = pack_rows(rows)
        ids, off, _ = self.encode_packed(table, data, offsets)
        return [ids[int(off[i]):int(off[i + 1])].tolist() for i in range(len(rows))]

    def encode_device(self, table: MergeTable, d_bytes, d_offsets, n: int, total: int, d_out_ids, d_out_offsets,
                      stream: int = 0, sync: bool = True) -> dict:
        """Device pointers (ints, e.g. torch tensor .data_ptr()) -> CSR on device."""
        st = Stats()
        _check(LIB.bbpe_encode_device(self._h, table.handle, C.c_void_p(d_bytes), C.c_void_p(d_offsets), n, total,
                                      C.c_void_p(d_out_ids), C.c_void_p(d_out_offsets),
                                      C.c_void_p(stream) if stream else None, 1 if sync else 0, C.byref(st)))
        return st.as_dict()

    def sync(self):
        _check(LIB.bbpe_ctx_sync(self._h))

    def pretokenize_device(self, d_bytes, d_offsets, n: int, total: int, d_chunk_bits):
        """The gpt2 splitter's chunk starts (row starts included) as a bitmap of
        (total + 31) // 32 u32 words (bbpe_pretokenize_device)."""
        _check(LIB.bbpe_pretokenize_device(self._h, C.c_void_p(d_bytes), C.c_void_p(d_offsets), n, total,
                                           C.c_void_p(d_chunk_bits)))

    def encode_tensors(self, table: MergeTable, data, offsets):
        """Zero-copy hand-off: device tensors in, device tensors
        out -- uint8 bytes and int64 row offsets on this encoder's GPU -> (ids
        int32, offsets int64), CSR, on the same GPU, ordered on torch's current
        stream. Export with torch.utils.dlpack.to_dlpack for other frameworks."""
        import torch
        dev = torch.device("cuda", self.device)
        if data.device != dev or offsets.device != dev:
            raise UsageError(f"encode_tensors needs tensors on {dev}")
        if data.dtype != torch.uint8 or offsets.dtype != torch.int64:
            raise UsageError("encode_tensors takes uint8 bytes and int64 offsets")
        data, offsets = data.contiguous(), offsets.contiguous()
        n = offsets.numel() - 1
        if n < 0:
            raise UsageError("offsets need n + 1 entries")
        first, total = (int(v) for v in offsets[[0, -1]].tolist())
        if first:
            data, offsets, total = data[first:], offsets - first, total - first
        ids = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        oo = torch.empty(n + 1, dtype=torch.int64, device=dev)
        self.encode_device(table, data.data_ptr(), offsets.data_ptr(), n, total, ids.data_ptr(), oo.data_ptr(),
                           stream=torch.cuda.current_stream(dev).cuda_stream)
        return ids[: int(oo[-1].item())], oo

    def set_specials(self, specials: Optional["SpecialTokenSet"]):
        """The device copy of a special-token set (bbpe_ctx_set_specials); None clears it."""
        ents = specials.entries() if specials is not None else []
        key = tuple(ents)
        if key == self._sp_key:
            return
        blob = np.frombuffer(b"".join(b for b, _ in ents) or b"\0", dtype=np.uint8)
        offs = np.zeros(len(ents) + 1, np.uint64)
        offs[1:] = np.cumsum([len(b) for b, _ in ents], dtype=np.uint64)
        ids = np.array([i for _, i in ents] or [0], np.uint32)
        _check(LIB.bbpe_ctx_set_specials(self._h, len(ents), _p(blob, C.c_uint8), _p(offs, C.c_uint64),
                                         _p(ids, C.c_uint32)))
        self._sp_key = key

    def encode_batch_packed(self, table: MergeTable, data: np.ndarray, offsets: np.ndarray,
                            bos_id: Optional[int] = None, eos_id: Optional[int] = None):
        """Host buffers through bbpe_encode_batch (what the C++ drop-in calls):
        encode_batch's rows as CSR (ids u32, offsets u64[n+1])."""
        data = np.ascontiguousarray(data, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        ids = np.empty(max(int(offsets[-1] - offsets[0]) + 2 * n + 1, 1), np.uint32)
        oo = np.empty(n + 1, np.uint64)
        k = C.c_uint64()
        none = 0xFFFFFFFF
        _check(LIB.bbpe_encode_batch(self._h, table.handle, _p(data, C.c_uint8) if data.size else None,
                                     _p(offsets, C.c_uint64), n, none if bos_id is None else bos_id,
                                     none if eos_id is None else eos_id, _p(ids, C.c_uint32), ids.size,
                                     _p(oo, C.c_uint64), C.byref(k)))
        return ids[: k.value], oo

    def encode_batch_device(self, table: MergeTable, d_bytes, d_offsets, n: int, total: int, d_out_ids, cap: int,
                            d_out_offsets, bos_id: Optional[int] = None, eos_id: Optional[int] = None) -> int:
        """encode_batch's rows as device CSR (bbpe_encode_batch_device): split at
        this encoder's special tokens (set_specials), literal segments encoded,
        special ids passed through, BOS/EOS added. Returns the id count."""
        nout = C.c_uint64()
        none = 0xFFFFFFFF
        _check(LIB.bbpe_encode_batch_device(self._h, table.handle, C.c_void_p(d_bytes), C.c_void_p(d_offsets), n,
                                            total, none if bos_id is None else bos_id,
                                            none if eos_id is None else eos_id, C.c_void_p(d_out_ids), cap,
                                            C.c_void_p(d_out_offsets), C.byref(nout)))
        return nout.value

    def decode_packed(self, table: MergeTable, ids: np.ndarray, offsets: np.ndarray,
                      out: Optional[np.ndarray] = None, out_offsets: Optional[np.ndarray] = None,
                      skip_specials: bool = False):
        """Device batch decode (decode / decode_batch, merge_table.hpp:565-579,
        batch.hpp:128-154): CSR ids -> (bytes u8, byte offsets u64[n+1]). Ids the
        table lacks decode through this encoder's special tokens (set_specials);
        skip_specials drops special ids."""
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        if out is None:
            # Upper bound: the longest token (or special) times the number of ids.
            widest = max([table.max_token_bytes()] + [len(b) for b, _ in self._sp_key])
            out = np.empty(max(int(offsets[-1] - offsets[0]) * widest, 1), dtype=np.uint8)
        if out_offsets is None:
            out_offsets = np.empty(n + 1, dtype=np.uint64)
        total = C.c_uint64()
        _check(LIB.bbpe_decode_batch_ex(self._h, table.handle, _p(ids, C.c_uint32) if ids.size else None,
                                        _p(offsets, C.c_uint64), n, int(skip_specials), _p(out, C.c_uint8), out.size,
                                        _p(out_offsets, C.c_uint64), C.byref(total)))
        if total.value > out.size:
            raise UsageError(f"decode output capacity {out.size} is smaller than the {total.value} bytes produced")
        return out[: total.value], out_offsets

    def jsonl_device(self, d_ids, d_offsets, n_rows: int, n_ids: int, d_out, cap: int) -> int:
        """JSON-lines text of a device CSR batch (write_batch_jsonl, batch.hpp:157-166)
        into d_out (at most cap bytes); returns the full text length."""
        total = C.c_uint64()
        _check(LIB.bbpe_jsonl_device(self._h, C.c_void_p(d_ids), C.c_void_p(d_offsets), n_rows, n_ids,
                                     C.c_void_p(d_out), cap, C.byref(total)))
        return total.value

    def decode_device(self, table: MergeTable, d_ids, d_offsets, n_rows: int, n_ids: int, d_out, cap: int,
                      d_out_offsets, skip_specials: bool = False) -> int:
        """Device pointers: CSR ids -> CSR bytes on device; returns the byte total."""
        total = C.c_uint64()
        _check(LIB.bbpe_decode_device_ex(self._h, table.handle, C.c_void_p(d_ids), C.c_void_p(d_offsets), n_rows,
                                         n_ids, int(skip_specials), C.c_void_p(d_out), cap,
                                         C.c_void_p(d_out_offsets), C.byref(total)))
        return total.value

    def block_bpe(self, table: MergeTable, tokens: Sequence[int], trace: bool = False):
        """block_engine.hpp:268-310 on explicit ids. Returns ids, or (ids, trace)
        with trace = [(pass_index, min_rank, merges_applied), ...]."""
        toks = np.ascontiguousarray(np.asarray(tokens, dtype=np.uint32))
        n = toks.size
        out = np.zeros(max(n, 1), np.uint32)
        out_n = C.c_size_t()
        npass = C.c_size_t()
        cap = n + 1 if trace else 0
        tr = np.zeros(max(cap, 1) * 3, np.uint64)
        rc = LIB.bbpe_block_bpe(self._h, table.handle, _p(toks, C.c_uint32) if n else None, n, _p(out, C.c_uint32),
                                C.byref(out_n), _p(tr, C.c_uint64) if trace else None, cap, C.byref(npass))
        res = out[: out_n.value].tolist()
        if rc == 6:
            raise MaxPassesError(LIB.bbpe_last_error().decode(), res, npass.value)
        _check(rc)
        if trace:
            k = min(npass.value, cap)
            return res, [tuple(int(v) for v in tr[3 * i:3 * i + 3]) for i in range(k)]
        return res


_DEFAULT_ENCODERS = {}


def default_encoder(device: int = 0) -> Encoder:
    if device not in _DEFAULT_ENCODERS:
        _DEFAULT_ENCODERS[device] = Encoder(device)
    return _DEFAULT_ENCODERS[device]


def partition(offsets: np.ndarray, parts: int) -> np.ndarray:
    """Cost-balanced contiguous row shards (bbpe_partition): parts+1 bounds."""
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    b = np.zeros(parts + 1, np.uint64)
    _check(LIB.bbpe_partition(_p(offsets, C.c_uint64), offsets.size - 1, parts, _p(b, C.c_uint64)))
    return b


def gather_csr(ids, offsets, dst: int = 0, group=None):
    """Per-rank CSR (ids int32 [k], offsets int64 [n+1] from 0) gathered to
    rank `dst` as one CSR in rank order, offsets rebased: the optional
    gather-to-one-GPU epilogue of a sharded encode. Sizes
    are all-gathered, then ids and offsets go point to point (NCCL send/recv
    over NVLink on GPUs, gloo on CPU). Returns (ids, offsets) on dst, None
    elsewhere. Not on the encode path: shards never exchange data to encode."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    k, n = ids.numel(), offsets.numel() - 1
    sz = torch.tensor([k, n], dtype=torch.int64, device=offsets.device)
    sizes = [torch.empty_like(sz) for _ in range(world)]
    dist.all_gather(sizes, sz, group=group)
    sizes = [tuple(int(v) for v in t.tolist()) for t in sizes]
    if rank != dst:
        if k:
            dist.send(ids.contiguous(), dst, group=group)
        dist.send(offsets.contiguous(), dst, group=group)
        return None
    out_ids = torch.empty(sum(x[0] for x in sizes), dtype=ids.dtype, device=ids.device)
    out_off = torch.empty(sum(x[1] for x in sizes) + 1, dtype=offsets.dtype, device=offsets.device)
    tb = rb = 0
    for r, (kr, nr) in enumerate(sizes):
        if r == dst:
            out_ids[tb:tb + kr] = ids
            o = offsets
        else:
            if kr:
                dist.recv(out_ids[tb:tb + kr], r, group=group)
            o = torch.empty(nr + 1, dtype=offsets.dtype, device=offsets.device)
            dist.recv(o, r, group=group)
        out_off[rb:rb + nr + 1] = o + tb
        tb += kr
        rb += nr
    return out_ids, out_off


def encode_sharded(encoders: Sequence[Encoder], table: MergeTable, data: np.ndarray, offsets: np.ndarray,
                   capacity: Optional[int] = None):
    """Rows split into cost-balanced contiguous shards (bbpe_partition), one
    per encoder/GPU, each on its own host thread near its GPU; CSR stitched.
    `capacity`: output ids to allocate (default: input bytes, the upper bound)."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = offsets.size - 1
    total = int(offsets[-1] - offsets[0]) if capacity is None else int(capacity)
    out = np.empty(max(total, 1), np.uint32)
    oo = np.empty(n + 1, np.uint64)
    hs = (C.c_void_p * len(encoders))(*[e.handle for e in encoders])
    st = Stats()
    _check(LIB.bbpe_encode_sharded(hs, len(encoders), table.handle, _p(data, C.c_uint8) if data.size else None,
                                   _p(offsets, C.c_uint64), n, _p(out, C.c_uint32), total, _p(oo, C.c_uint64),
                                   C.byref(st)))
    return out[: int(oo[-1])], oo, st.as_dict()


# ---------------------------------------------------------------------------
# Batch API (batch.hpp)


@dataclass
class BatchEncoding:
    batch_size: int = 0
    max_len: int = 0
    pad_id: int = 0
    ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    lengths: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    mask: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    truncated_rows: int = 0

    def at(self, row: int, col: int) -> int:
        return int(self.ids[row * self.max_len + col])

    def row(self, r: int) -> List[int]:
        b = r * self.max_len
        return self.ids[b:b + int(self.lengths[r])].tolist()


_ROW_RE = re.compile(r"^row (\d+): ")


def _remap_row_error(e: Error, seg_row: Sequence[int]):
    m = _ROW_RE.match(str(e))
    if not m:
        raise e
    r = seg_row[int(m.group(1))]
    raise type(e)(f"row {r}: {str(e)[m.end():]}") from None


def _encode_rows_device(rows: List[bytes], table: MergeTable, specials: SpecialTokenSet, add_bos: bool,
                        add_eos: bool, enc: "Encoder"):
    """Rows -> device CSR of encode_batch's rows (specials split on the device,
    bbpe_encode_batch_device). Returns (d_ids, d_offsets, n_ids) torch tensors."""
    import torch
    dev = torch.device("cuda", enc.device)
    data, offsets = pack_rows(rows)
    n, total = len(rows), int(offsets[-1])
    enc.set_specials(specials)
    d_data = torch.from_numpy(data if data.flags.writeable else data.copy()).to(dev)
    d_off = torch.from_numpy(offsets.view(np.int64)).to(dev)
    cap = max(total + 2 * n, 1)  # literal tokens + specials <= bytes, plus BOS/EOS
    d_ids = torch.empty(cap, dtype=torch.int32, device=dev)
    d_oo = torch.empty(n + 1, dtype=torch.int64, device=dev)
    nout = enc.encode_batch_device(table, d_data.data_ptr(), d_off.data_ptr(), n, total, d_ids.data_ptr(), cap,
                                   d_oo.data_ptr(), specials.bos_id() if add_bos else None,
                                   specials.eos_id() if add_eos else None)
    return d_ids, d_oo, nout


def encode_batch_csr(inputs: Sequence[Union[bytes, str]], table: MergeTable, specials: SpecialTokenSet,
                     config: BlockConfig, add_bos: bool = False, add_eos: bool = False,
                     encoder: Optional[Encoder] = None, device_split: bool = True) -> Tuple[np.ndarray, np.ndarray]:
    """encode_batch's per-row results as CSR (ids, offsets) -- no padding.
    Specials are split on the device (device_split, default) or, for A/B
    checks, on the host with the literal segments encoded on the device."""
    config.validate()
    if add_bos and specials.bos_id() is None:
        raise UsageError("add_bos requires a bos entry in the special token set")
    if add_eos and specials.eos_id() is None:
        raise UsageError("add_eos requires an eos entry in the special token set")
    enc = encoder or default_encoder()
    if enc.config.block_size != config.block_size or enc.config.max_passes != config.max_passes:
        enc.set_config(config=config)
    rows = [r.encode() if isinstance(r, str) else bytes(r) for r in inputs]
    if specials.empty() and not add_bos and not add_eos:
        data, offsets = pack_rows(rows)
        ids, off, _ = enc.encode_packed(table, data, offsets)
        return ids, off
    if device_split:
        d_ids, d_oo, nout = _encode_rows_device(rows, table, specials, add_bos, add_eos, enc)
        return d_ids[:nout].cpu().numpy().view(np.uint32).copy(), d_oo.cpu().numpy().view(np.uint64).copy()
    # Specials / BOS / EOS: literal segments become device rows, re-stitched here.
    seg_rows: List[bytes] = []
    seg_row: List[int] = []
    plan = []  # per input row: list of ("lit", seg index) | ("sp", id)
    for r, data in enumerate(rows):
        items = []
        for s in split_specials(data, specials):
            if s.kind == "special":
                items.append(("sp", s.special_id))
            else:
                items.append(("lit", len(seg_rows)))
                seg_rows.append(s.bytes)
                seg_row.append(r)
        plan.append(items)
    data, offsets = pack_rows(seg_rows)
    try:
        sids, soff, _ = enc.encode_packed(table, data, offsets)
    except Error as e:
        _remap_row_error(e, seg_row)
    out: List[np.ndarray] = []
    lens = np.zeros(len(rows) + 1, np.uint64)
    for r, items in enumerate(plan):
        parts = []
        if add_bos:
            parts.append(np.array([specials.bos_id()], np.uint32))
        for kind, v in items:
            if kind == "sp":
                parts.append(np.array([v], np.uint32))
            else:
                parts.append(sids[int(soff[v]):int(soff[v + 1])])
        if add_eos:
            parts.append(np.array([specials.eos_id()], np.uint32))
        row = np.concatenate(parts) if parts else np.zeros(0, np.uint32)
        out.append(row)
        lens[r + 1] = row.size
    return (np.concatenate(out) if out else np.zeros(0, np.uint32)), np.cumsum(lens).astype(np.uint64)


def _encode_batch_device(rows: List[bytes], table: MergeTable, specials: SpecialTokenSet, config: BlockConfig,
                         pad_id: int, add_bos: bool, add_eos: bool, enc: "Encoder",
                         limits: Optional[BatchLimits]) -> BatchEncoding:
    """Device epilogue: specials split, CSR encode, BOS/EOS,
    widest row and padding all on the GPU (bbpe_encode_batch_device,
    bbpe_batch_widest_device, bbpe_pad_device); one copy of the padded batch back."""
    import torch
    dev = torch.device("cuda", enc.device)
    n = len(rows)
    d_ids, d_oo, _ = _encode_rows_device(rows, table, specials, add_bos, add_eos, enc)
    widest = C.c_uint64()
    _check(LIB.bbpe_batch_widest_device(enc.handle, C.c_void_p(d_oo.data_ptr()), n, 0, 0, C.byref(widest)))
    out = BatchEncoding(batch_size=n, pad_id=pad_id)
    out.max_len = int(limits.max_len) if limits is not None and limits.max_len is not None else widest.value
    L = out.max_len
    t_ids = torch.empty(max(n * L, 1), dtype=torch.int32, device=dev)
    t_mask = torch.empty(max(n * L, 1), dtype=torch.uint8, device=dev)
    t_len = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    tr = C.c_uint64()
    nid = 0xFFFFFFFF
    _check(LIB.bbpe_pad_device(enc.handle, C.c_void_p(d_ids.data_ptr()), C.c_void_p(d_oo.data_ptr()), n, pad_id,
                               nid, nid, L,
                               C.c_void_p(t_ids.data_ptr()), C.c_void_p(t_len.data_ptr()),
                               C.c_void_p(t_mask.data_ptr()), C.byref(tr)))
    out.ids = t_ids[: n * L].cpu().numpy().view(np.uint32).copy()
    out.mask = t_mask[: n * L].cpu().numpy().copy()
    out.lengths = t_len[:n].cpu().numpy().view(np.uint32).copy()
    out.truncated_rows = int(tr.value)
    return out


def encode_batch(inputs: Sequence[Union[bytes, str]], table: MergeTable, specials: SpecialTokenSet,
                 config: BlockConfig, pad_id: int, add_bos: bool = False, add_eos: bool = False,
                 encoder: Optional[Encoder] = None, limits: Optional[BatchLimits] = None,
                 device_epilogue: Optional[bool] = None) -> BatchEncoding:
    """batch.hpp:64-126: rows encoded on the GPU, padded to max_len (or the fixed
    limits.max_len with right truncation), u8 mask. With an empty special-token
    set the padding runs on the device too (device_epilogue, default); with
    specials as well: the rows are split at special tokens on the device
    (device_epilogue=False: host split and padding, for A/B checks)."""
    config.validate()
    if add_bos and specials.bos_id() is None:
        raise UsageError("add_bos requires a bos entry in the special token set")
    if add_eos and specials.eos_id() is None:
        raise UsageError("add_eos requires an eos entry in the special token set")
    if device_epilogue is None:
        device_epilogue = True
    if device_epilogue:
        enc = encoder or default_encoder()
        if enc.config.block_size != config.block_size or enc.config.max_passes != config.max_passes:
            enc.set_config(config=config)
        rows = [r.encode() if isinstance(r, str) else bytes(r) for r in inputs]
        return _encode_batch_device(rows, table, specials, config, pad_id, add_bos, add_eos, enc, limits)
    ids, off = encode_batch_csr(inputs, table, specials, config, add_bos, add_eos, encoder, device_split=False)
    n = len(inputs)
    lengths = (off[1:] - off[:-1]).astype(np.int64)
    out = BatchEncoding(batch_size=n, pad_id=pad_id)
    widest = int(lengths.max()) if n else 0
    if limits is not None and limits.max_len is not None:
        out.max_len = int(limits.max_len)
        out.truncated_rows = int((lengths > out.max_len).sum())
        lengths = np.minimum(lengths, out.max_len)
    else:
        out.max_len = widest
    L = out.max_len
    out.ids = np.full(n * L, pad_id, dtype=np.uint32)
    out.mask = np.zeros(n * L, dtype=np.uint8)
    if n and L:
        col = np.arange(L)[None, :]
        m = col < lengths[:, None]
        src = (off[:-1].astype(np.int64)[:, None] + col)[m]
        out.ids.reshape(n, L)[m] = ids[src]
        out.mask.reshape(n, L)[m] = 1
    out.lengths = lengths.astype(np.uint32)
    return out


def encode_single(data: Union[bytes, str], table: MergeTable, specials: SpecialTokenSet, config: BlockConfig,
                  encoder: Optional[Encoder] = None) -> List[int]:
    """batch.hpp:46-59."""
    ids, off = encode_batch_csr([data], table, specials, config, False, False, encoder)
    return ids.tolist()


def bytes_to_initial_tokens(data: bytes, table: MergeTable) -> List[int]:
    """pretokenize.hpp:60-71 (host helper for building block_bpe inputs)."""
    out = []
    for b in data:
        t = table.byte_token(b)
        if t == INVALID_TOKEN:
            raise IntegrityError(f"vocabulary has no single-byte token for byte value {b}")
        out.append(t)
    return out


def block_bpe(tokens: Sequence[int], table: MergeTable, config: BlockConfig, encoder: Optional[Encoder] = None,
              trace: Optional[list] = None) -> List[int]:
    """block_engine.hpp:268-310 on the GPU; `trace` (a list) receives
    (pass_index, min_rank, merges_applied) records like PassTrace."""
    config.validate()
    enc = encoder or default_encoder()
    if enc.config.block_size != config.block_size or enc.config.max_passes != config.max_passes:
        enc.set_config(config=config)
    if trace is not None:
        res, tr = enc.block_bpe(table, tokens, trace=True)
        trace.extend(tr)
        return res
    return enc.block_bpe(table, tokens)


# ---- spec-level operations (block_engine.hpp:189-256), run on the device ----

def _u32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32).reshape(-1))


def pair_ranks(tokens: Sequence[int], table: MergeTable, encoder: Optional[Encoder] = None) -> List[Optional[int]]:
    """block_engine.hpp:189-199: rank of each adjacent pair, None if absent."""
    enc = encoder or default_encoder()
    t = _u32(tokens)
    if t.size < 2:
        return []
    out = np.zeros(t.size - 1, np.uint32)
    _check(LIB.bbpe_pair_ranks(enc.handle, table.handle, _p(t, C.c_uint32), t.size, _p(out, C.c_uint32)))
    return [None if int(r) == NO_RANK else int(r) for r in out]


def min_rank_reduce(ranks: Sequence[Optional[int]], encoder: Optional[Encoder] = None) -> Optional[int]:
    """block_engine.hpp:201-206."""
    enc = encoder or default_encoder()
    r = _u32([NO_RANK if x is None else x for x in ranks])
    out = C.c_uint32(0)
    _check(LIB.bbpe_min_rank_reduce(enc.handle, _p(r, C.c_uint32) if r.size else None, r.size, C.byref(out)))
    return None if out.value == NO_RANK else out.value


def mark_merges(tokens: Sequence[int], table: MergeTable, min_rank: int, encoder: Optional[Encoder] = None) -> List[int]:
    """block_engine.hpp:211-220: flags[i+1] = 1 for left-greedy rank-min pairs."""
    enc = encoder or default_encoder()
    t = _u32(tokens)
    f = np.zeros(max(t.size, 1), np.uint8)
    _check(LIB.bbpe_mark_merges(enc.handle, table.handle, _p(t, C.c_uint32) if t.size else None, t.size,
                                int(min_rank), _p(f, C.c_uint8)))
    return f[: t.size].tolist()


def exclusive_scan(flags: Sequence[int], encoder: Optional[Encoder] = None) -> List[int]:
    """block_engine.hpp:223-235 (ContractViolation on values > 1 or adjacent flags)."""
    enc = encoder or default_encoder()
    f = np.ascontiguousarray(np.asarray(flags, dtype=np.uint8).reshape(-1))
    out = np.zeros(max(f.size, 1), np.uint32)
    _check(LIB.bbpe_exclusive_scan(enc.handle, _p(f, C.c_uint8) if f.size else None, f.size, _p(out, C.c_uint32)))
    return out[: f.size].tolist()


def compact(tokens: Sequence[int], table: MergeTable, flags: Sequence[int], offsets: Sequence[int],
            encoder: Optional[Encoder] = None) -> List[int]:
    """block_engine.hpp:238-256 + compact_into 166-182 (ContractViolation on
    length/offset mismatch or a flagged pair that is not a merge)."""
    enc = encoder or default_encoder()
    t = _u32(tokens)
    f = np.ascontiguousarray(np.asarray(flags, dtype=np.uint8).reshape(-1))
    o = _u32(offsets)
    out = np.zeros(max(t.size, 1), np.uint32)
    n_out = C.c_size_t(0)
    _check(LIB.bbpe_compact(enc.handle, table.handle, _p(t, C.c_uint32) if t.size else None, t.size,
                            _p(f, C.c_uint8) if f.size else None, f.size, _p(o, C.c_uint32) if o.size else None,
                            o.size, _p(out, C.c_uint32), C.byref(n_out)))
    return out[: n_out.value].tolist()


def block_bpe_replay(tokens: Sequence[int], table: MergeTable, encoder: Optional[Encoder] = None,
                     trace: Optional[list] = None) -> List[int]:
    """block_bpe (block_engine.hpp:268-310) driven pass by pass through the
    device spec ops above: the per-phase debug replay of the engine."""
    t = [int(x) for x in tokens]
    npass = 0
    while len(t) >= 2:
        m = min_rank_reduce(pair_ranks(t, table, encoder), encoder)
        if m is None:
            break
        f = mark_merges(t, table, m, encoder)
        off = exclusive_scan(f, encoder)
        t = compact(t, table, f, off, encoder)
        npass += 1
        if trace is not None:
            trace.append((npass, m, int(sum(f))))
    return t


def decode(table: MergeTable, specials: SpecialTokenSet, ids: Sequence[int]) -> bytes:
    """merge_table.hpp:565-579."""
    out = bytearray()
    toks = table.token_bytes()
    for i, t in enumerate(ids):
        b = toks.get(int(t))
        if b is None:
            b = specials.bytes_of(int(t))
        if b is None:
            raise DecodeError(f"unknown token id {int(t)} at index {i}")
        out += b
    return bytes(out)


def decode_batch(encoding: BatchEncoding, table: MergeTable, specials: SpecialTokenSet,
                 skip_specials: bool, encoder: Optional[Encoder] = None) -> List[bytes]:
    """batch.hpp:128-154, on the GPU: the rows' ids as CSR, decoded through the
    table and the special tokens (bbpe_decode_batch_ex), "row r: " errors."""
    n = encoding.batch_size
    lens = np.asarray(encoding.lengths[:n], dtype=np.int64)
    offsets = np.zeros(n + 1, np.uint64)
    np.cumsum(lens, out=offsets[1:])
    L = int(encoding.max_len)
    if n and L:
        mask = np.arange(L)[None, :] < lens[:, None]
        ids = np.ascontiguousarray(np.asarray(encoding.ids, dtype=np.uint32).reshape(n, L)[mask])
    else:
        ids = np.zeros(0, np.uint32)
    enc = encoder or default_encoder()
    enc.set_specials(specials)
    data, boff = enc.decode_packed(table, ids, offsets, skip_specials=skip_specials)
    return [data[int(boff[r]):int(boff[r + 1])].tobytes() for r in range(n)]


def write_batch_jsonl(encoding: BatchEncoding) -> str:
    """batch.hpp:159-166: one {"ids":[...],"len":n} per row."""
    lines = []
    for r in range(encoding.batch_size):
        row = encoding.row(r)
        lines.append(json.dumps({"ids": row, "len": int(encoding.lengths[r])}, separators=(",", ":")))
    return "".join(l + "\n" for l in lines)


def read_jsonl_token_seqs(text: str, name: str) -> List[List[int]]:
    """batch.hpp:170-189."""
    out = []
    for no, line in enumerate(text.split("\n"), 1):
        if not line:
            continue
        try:
            row = json.loads(line)
        except json.JSONDecodeError as e:
            raise ParseError(f"{name}:{no}: {e}") from None
        if not isinstance(row, dict) or not isinstance(row.get("ids"), list):
            raise ParseError(f'{name}:{no}: expected an object with an "ids" array')
        out.append([int(x) for x in row["ids"]])
    return out


def write_batch_binary(encoding: BatchEncoding) -> bytes:
    """batch.hpp:211-218: "BBPE", u32 batch, u32 max_len, u32 pad_id, u32 ids."""
    hdr = np.array([encoding.batch_size, encoding.max_len, encoding.pad_id], dtype="<u4").tobytes()
    return b"BBPE" + hdr + np.asarray(encoding.ids, dtype="<u4").tobytes()


def read_batch_binary(blob: bytes, name: str) -> BatchEncoding:
    """batch.hpp:224-242 (lengths rebuilt by stripping trailing pad_id)."""
    if len(blob) < 4 or blob[:4] != b"BBPE":
        raise ParseError(f"{name}: bad magic, not a BBPE batch file")
    if len(blob) < 16:
        raise ParseError(f"{name}: truncated batch file")
    b, L, pad = np.frombuffer(blob[4:16], dtype="<u4").tolist()
    if len(blob) < 16 + 4 * b * L:
        raise ParseError(f"{name}: truncated batch file")
    ids = np.frombuffer(blob[16:16 + 4 * b * L], dtype="<u4").astype(np.uint32)
    out = BatchEncoding(batch_size=b, max_len=L, pad_id=pad, ids=ids)
    lengths = np.zeros(b, np.uint32)
    mask = np.zeros(b * L, np.uint8)
    for r in range(b):
        n = L
        while n > 0 and ids[r * L + n - 1] == pad:
            n -= 1
        lengths[r] = n
        mask[r * L:r * L + n] = 1
    out.lengths, out.mask = lengths, mask
    return out
