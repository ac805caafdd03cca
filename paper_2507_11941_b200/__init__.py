"""B200-native BlockBPE batch tokenizer (drop-in for the reference's encode path).

The merging runs in hand-written sm_100a kernels behind the C-ABI in
include/bbpe_b200.h; this package is the Python mirror of the reference's
`blockbpe` API over that ABI. Importing fails if libbbpe_b200.so is absent.
"""
from .api import (  # noqa: F401
    BatchEncoding, BatchLimits, BlockConfig, ContractViolation, DecodeError, Encoder, Error,
    IntegrityError, MaxPassesError, MergeTable, ParseError, Segment, SpecialTokenSet, UsageError,
    block_bpe, bytes_to_initial_tokens, coarsening_factor, decode, decode_batch, default_encoder,
    encode_batch, encode_batch_csr, encode_sharded, gather_csr, encode_single, load_merge_table_files, pack_rows,
    parse_vocab_format, partition, read_batch_binary, read_jsonl_token_seqs, split_specials,
    validate_specials, write_batch_binary, write_batch_jsonl,
    pair_ranks, min_rank_reduce, mark_merges, exclusive_scan, compact, block_bpe_replay,
)
from ._lib import LIB_PATH  # noqa: F401
