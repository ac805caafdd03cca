"""ctypes binding of the C-ABI in include/bbpe_b200.h (libbbpe_b200.so).

The library is built in-tree (``make -C paper_2507_11941_b200`` or
``__graft_entry__.build()``). There is no fallback: if the shared object is
missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BBPE_LIB_PATH selects an alternative in-tree build (A/B experiments).
LIB_PATH = os.environ.get("BBPE_LIB_PATH") or os.path.join(_HERE, "libbbpe_b200.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class Config(C.Structure):
    _fields_ = [
        ("block_size", C.c_uint32),
        ("max_passes", C.c_int64),
        ("engine", C.c_int32),
        ("wave_bytes", C.c_uint64),
        ("piece_memo", C.c_int32),
        ("no_dedup", C.c_int32),
        ("pattern", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("n_rows", C.c_uint64),
        ("input_bytes", C.c_uint64),
        ("tokens", C.c_uint64),
        ("long_pieces", C.c_uint64),
        ("waves", C.c_uint64),
        ("device_ms", C.c_double),
        ("h2d_ms", C.c_double),
        ("d2h_ms", C.c_double),
        ("total_ms", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class TableInfo(C.Structure):
    _fields_ = [
        ("token_count", C.c_uint64),
        ("merge_count", C.c_uint64),
        ("base_size", C.c_uint64),
        ("max_token_id", C.c_uint32),
        ("id_bits", C.c_uint32),
        ("rank_bits", C.c_uint32),
        ("remapped_ids", C.c_uint32),
        ("hash_slots", C.c_uint64),
        ("junction_bigrams", C.c_uint64),
        ("rank_consistent", C.c_uint32),
    ]


# name -> (restype, argtypes); every symbol declared in include/bbpe_b200.h.
SIGNATURES = {
    "bbpe_last_error": (C.c_char_p, []),
    "bbpe_abi_version": (C.c_int, []),
    "bbpe_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "bbpe_table_load_files": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "bbpe_table_create": (C.c_int, [C.c_size_t, u32p, u64p, u8p, C.c_size_t, u32p, C.POINTER(C.c_void_p)]),
    "bbpe_table_destroy": (C.c_int, [C.c_void_p]),
    "bbpe_table_get_info": (C.c_int, [C.c_void_p, C.POINTER(TableInfo)]),
    "bbpe_table_save_binary": (C.c_int, [C.c_void_p, C.c_char_p]),
    "bbpe_table_export": (C.c_int, [C.c_void_p, u32p, u64p, u8p, u64p, u64p, u32p, u64p]),
    "bbpe_table_byte_token": (C.c_uint32, [C.c_void_p, C.c_uint8]),
    "bbpe_table_rank_of": (C.c_uint32, [C.c_void_p, C.c_uint32, C.c_uint32, u32p]),
    "bbpe_decode": (C.c_int, [C.c_void_p, u32p, C.c_size_t, u8p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "bbpe_decode_batch": (C.c_int, [C.c_void_p, C.c_void_p, u32p, u64p, C.c_size_t, u8p, C.c_uint64, u64p, u64p]),
    "bbpe_decode_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64,
                                     C.c_void_p, C.c_uint64, C.c_void_p, u64p]),
    "bbpe_decode_batch_ex": (C.c_int, [C.c_void_p, C.c_void_p, u32p, u64p, C.c_size_t, C.c_int, u8p, C.c_uint64,
                                       u64p, u64p]),
    "bbpe_decode_device_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64,
                                        C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, u64p]),
    "bbpe_jsonl_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64, C.c_void_p,
                                    C.c_uint64, u64p]),
    "bbpe_batch_widest_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int, u64p]),
    "bbpe_pad_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint32, C.c_uint32,
                                  C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, u64p]),
    "bbpe_pretokenize_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64, C.c_void_p]),
    "bbpe_ctx_set_specials": (C.c_int, [C.c_void_p, C.c_size_t, u8p, u64p, u32p]),
    "bbpe_encode_batch_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64,
                                           C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64, C.c_void_p, u64p]),
    "bbpe_encode_batch": (C.c_int, [C.c_void_p, C.c_void_p, u8p, u64p, C.c_size_t, C.c_uint32, C.c_uint32, u32p,
                                    C.c_uint64, u64p, u64p]),
    "bbpe_ctx_create": (C.c_int, [C.c_int, C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "bbpe_ctx_destroy": (C.c_int, [C.c_void_p]),
    "bbpe_ctx_set_config": (C.c_int, [C.c_void_p, C.POINTER(Config)]),
    "bbpe_ctx_prepare": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bbpe_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "bbpe_host_free": (C.c_int, [C.c_void_p]),
    "bbpe_encode": (C.c_int, [C.c_void_p, C.c_void_p, u8p, u64p, C.c_size_t, u32p, C.c_uint64, u64p, C.POINTER(Stats)]),
    "bbpe_encode_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(Stats)]),
    "bbpe_ctx_sync": (C.c_int, [C.c_void_p]),
    "bbpe_ctx_kernel_launches": (C.c_uint64, [C.c_void_p]),
    "bbpe_ctx_kernel_times": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), u64p, C.c_int]),
    "bbpe_ctx_piece_stats": (C.c_int, [C.c_void_p, u64p, C.c_int]),
    "bbpe_block_bpe": (C.c_int, [C.c_void_p, C.c_void_p, u32p, C.c_size_t, u32p, C.POINTER(C.c_size_t),
                                 u64p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "bbpe_pair_ranks": (C.c_int, [C.c_void_p, C.c_void_p, u32p, C.c_size_t, u32p]),
    "bbpe_min_rank_reduce": (C.c_int, [C.c_void_p, u32p, C.c_size_t, u32p]),
    "bbpe_mark_merges": (C.c_int, [C.c_void_p, C.c_void_p, u32p, C.c_size_t, C.c_uint32, u8p]),
    "bbpe_exclusive_scan": (C.c_int, [C.c_void_p, u8p, C.c_size_t, u32p]),
    "bbpe_compact": (C.c_int, [C.c_void_p, C.c_void_p, u32p, C.c_size_t, u8p, C.c_size_t, u32p, C.c_size_t, u32p,
                               C.POINTER(C.c_size_t)]),
    "bbpe_partition": (C.c_int, [u64p, C.c_size_t, C.c_int, u64p]),
    "bbpe_encode_sharded": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, u8p, u64p, C.c_size_t,
                                      u32p, C.c_uint64, u64p, C.POINTER(Stats)]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make -C paper_2507_11941_b200` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = load()
