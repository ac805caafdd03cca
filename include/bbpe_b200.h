/* bbpe_b200.h -- C-ABI of the B200-native BlockBPE batch encoder.
 *
 * This is the drop-in boundary for the reference's batch-encode hot path
 * (reference = /root/reference/proj, header-only C++20 `namespace blockbpe`).
 * Plain pointers and sizes only; no C++ or torch types cross this line.
 * Each entry point names the reference interface it replaces:
 *
 *   bbpe_table_load_files   <- blockbpe::load_merge_table_files
 *                              (include/blockbpe/merge_table.hpp:513-522;
 *                               gpt2 loader 399-459, canonical JSON 473-497)
 *   bbpe_table_create       <- MergeTable::add_token / add_merge / finalize
 *                              (merge_table.hpp:257-297), i.e. the table that
 *                              MergeTable::merges().for_each exposes (180-184)
 *   bbpe_table_byte_token   <- MergeTable::byte_token (merge_table.hpp:246)
 *   bbpe_table_rank_of      <- MergeTable::rank_of / merged_of (225-235)
 *   bbpe_decode             <- blockbpe::decode (merge_table.hpp:565-579)
 *   bbpe_encode             <- blockbpe::encode_batch, block engine, CSR output
 *                              (include/blockbpe/batch.hpp:64-126; per row
 *                               encode_single 46-59 -> bytes_to_initial_tokens
 *                               pretokenize.hpp:60-71 -> block_bpe
 *                               block_engine.hpp:268-310)
 *   bbpe_encode_device      <- same, device-resident buffers (no host copies)
 *   bbpe_block_bpe          <- blockbpe::block_bpe on explicit token ids with
 *                              an optional PassTrace (block_engine.hpp:42-47,
 *                              268-310) and max_passes (MaxPassesError,
 *                              types.hpp:64-70)
 *   bbpe_encode_sharded     <- encode_batch's row fan-out (PhasePool::run_items,
 *                              thread_pool.hpp:95-101) re-targeted at several
 *                              GPUs: byte-balanced shards, no collective
 *   bbpe_partition          <- (new) the byte/cost-balanced row partitioner
 *
 * Error model: every call returns a bbpe_status that maps 1:1 onto the
 * reference exception taxonomy (types.hpp:32-70). bbpe_last_error() returns a
 * thread-local message; batch errors carry the reference's "row r: " prefix
 * (batch.hpp:84-90). Threading: a ctx is single-caller (like PhasePool,
 * thread_pool.hpp:141-142); a table is immutable and shareable.
 */
#ifndef BBPE_B200_H
#define BBPE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBPE_ABI_VERSION 2

typedef enum bbpe_status {
  BBPE_OK = 0,
  BBPE_USAGE = 1,       /* UsageError        */
  BBPE_PARSE = 2,       /* ParseError        */
  BBPE_INTEGRITY = 3,   /* IntegrityError    */
  BBPE_DECODE = 4,      /* DecodeError       */
  BBPE_CONTRACT = 5,    /* ContractViolation */
  BBPE_MAX_PASSES = 6,  /* MaxPassesError    */
  BBPE_ERROR = 7        /* Error (CUDA / runtime failure) */
} bbpe_status;

typedef enum bbpe_format {
  BBPE_FORMAT_GPT2 = 0,       /* vocab.json + merges.txt (VocabFormat::gpt2) */
  BBPE_FORMAT_CANONICAL = 1,  /* {tokens, merges, specials} JSON             */
  BBPE_FORMAT_BINARY = 2      /* this repo's .bbpt binary table              */
} bbpe_format;

/* Engine mode for bbpe_encode*: */
typedef enum bbpe_engine {
  /* Default. Each string is cut at "hard boundaries" -- byte positions whose
   * bigram is not the junction of any merge -- and the pieces are merged
   * independently: provably identical to block_bpe over the whole string
   * (DESIGN.md "Piece decomposition"). Short pieces: one lane each;
   * long pieces: one CTA each. */
  BBPE_ENGINE_PIECES = 0,
  /* One CTA per whole string, the paper's pass loop over the full string.
   * Required for max_passes (exact pass counting per string). */
  BBPE_ENGINE_BLOCK = 1
} bbpe_engine;

typedef struct bbpe_table bbpe_table;
typedef struct bbpe_ctx bbpe_ctx;

typedef struct bbpe_config {
  uint32_t block_size;     /* BlockConfig::block_size: 32..1024, pow2; results-neutral */
  int64_t max_passes;      /* <= 0: default (input length, never hit)        */
  int32_t engine;          /* bbpe_engine                                      */
  uint64_t wave_bytes;     /* host API: bytes per pipelined wave (0 = auto)     */
  int32_t piece_memo;      /* 1 (default): whole pieces equal to a vocabulary
                              token's bytes take that token's precomputed
                              encoding (exact; built from the table by this
                              engine on first use per device). 0: always run
                              the merge passes. Ignored by BBPE_ENGINE_BLOCK. */
  int32_t no_dedup;        /* 0 (default): within one call, the merge passes run
                              once per distinct merge piece of <= 15 bytes and
                              repeats copy that result (exact: a piece's
                              encoding depends on its bytes only). 1: every
                              piece runs its own passes.                      */
  int32_t pattern;         /* 0 (default): byte-level, merges across the whole row
                              (the block engine, encode_batch). 1: the gpt2 split
                              pattern (pattern_pretokenize, pretokenize.hpp:79-
                              258) on the device first, merges within each chunk
                              -- encode_reference's pattern mode (ref_engines.hpp
                              :119-146). Needs the pieces engine and a
                              rank-consistent table (heap == block there).    */
} bbpe_config;

typedef struct bbpe_stats {
  uint64_t n_rows;
  uint64_t input_bytes;
  uint64_t tokens;
  uint64_t long_pieces;    /* pieces that went to the CTA tier                 */
  uint64_t waves;
  double device_ms;        /* kernel time (CUDA events); 0 on the pipelined host path (untimed) */
  double h2d_ms;
  double d2h_ms;
  double total_ms;         /* wall time of the call                           */
} bbpe_stats;

typedef struct bbpe_table_info {
  uint64_t token_count;
  uint64_t merge_count;
  uint64_t base_size;      /* number of single-byte tokens                    */
  uint32_t max_token_id;
  uint32_t id_bits;        /* bits per token id in the device pair key        */
  uint32_t rank_bits;
  uint32_t remapped_ids;   /* 1 when ids were densified for the device        */
  uint64_t hash_slots;     /* device hash capacity (slots of 8 bytes)         */
  uint64_t junction_bigrams; /* |C|: bigrams that some merge can span         */
  uint32_t rank_consistent;  /* 1 when every merge's parts predate it         */
} bbpe_table_info;

/* ---- library ---- */
const char* bbpe_last_error(void);
int bbpe_abi_version(void);
int bbpe_device_count(int* count);

/* ---- tables ---- */
int bbpe_table_load_files(const char* vocab_path, const char* merges_path, int format,
                          bbpe_table** out);
/* ids[i] owns tok_bytes[tok_off[i] .. tok_off[i+1]); merges4 rows are
 * {rank, left, right, merged}. Same validation as MergeTable::finalize. */
int bbpe_table_create(size_t n_tokens, const uint32_t* ids, const uint64_t* tok_off,
                      const uint8_t* tok_bytes, size_t n_merges, const uint32_t* merges4,
                      bbpe_table** out);
int bbpe_table_destroy(bbpe_table* t);
int bbpe_table_get_info(const bbpe_table* t, bbpe_table_info* info);
int bbpe_table_save_binary(const bbpe_table* t, const char* path);
/* Exports tokens (sorted by id) and merges (sorted by rank). Pass null
 * buffers to query the sizes. */
int bbpe_table_export(const bbpe_table* t, uint32_t* ids, uint64_t* tok_off, uint8_t* tok_bytes,
                      uint64_t* n_tokens, uint64_t* n_bytes, uint32_t* merges4,
                      uint64_t* n_merges);
uint32_t bbpe_table_byte_token(const bbpe_table* t, uint8_t b); /* 0xFFFFFFFF = none */
/* rank (0xFFFFFFFF when absent); *merged receives the merged id when present. */
uint32_t bbpe_table_rank_of(const bbpe_table* t, uint32_t left, uint32_t right,
                            uint32_t* merged);
/* ids -> bytes; writes at most cap bytes and returns the full length in *len. */
int bbpe_decode(const bbpe_table* t, const uint32_t* ids, size_t n, uint8_t* out, size_t cap,
                size_t* len);

/* ---- device batch decode (decode merge_table.hpp:565-579,
 * decode_batch batch.hpp:128-154): CSR token ids -> CSR bytes.
 * ids[tok_offsets[r]..tok_offsets[r+1]) of row r decode to
 * out_bytes[out_byte_offsets[r]..out_byte_offsets[r+1]). At most cap bytes
 * are written; *total receives the full length (check it against cap).
 * Unknown id -> BBPE_DECODE, "row r: unknown token id X at index i".
 * Specials are not table tokens: decode rows containing them on the host. */
int bbpe_decode_batch(bbpe_ctx* ctx, const bbpe_table* t, const uint32_t* ids, const uint64_t* tok_offsets,
                      size_t n_rows, uint8_t* out_bytes, uint64_t cap, uint64_t* out_byte_offsets,
                      uint64_t* total);
/* The same on device buffers (n_ids = tok_offsets[n_rows] - tok_offsets[0]); synchronous. */
int bbpe_decode_device(bbpe_ctx* ctx, const bbpe_table* t, const uint32_t* d_ids, const uint64_t* d_tok_offsets,
                       size_t n_rows, uint64_t n_ids, uint8_t* d_out_bytes, uint64_t cap,
                       uint64_t* d_out_byte_offsets, uint64_t* total);

/* The same with the ctx's special-token set (bbpe_ctx_set_specials): ids the
 * table lacks decode to their special's bytes (decode, merge_table.hpp:565-579);
 * skip_specials != 0 drops special ids first (decode_batch, batch.hpp:128-154).
 * (The two calls above are these with skip_specials = 0.) */
int bbpe_decode_batch_ex(bbpe_ctx* ctx, const bbpe_table* t, const uint32_t* ids, const uint64_t* tok_offsets,
                         size_t n_rows, int skip_specials, uint8_t* out_bytes, uint64_t cap,
                         uint64_t* out_byte_offsets, uint64_t* total);
int bbpe_decode_device_ex(bbpe_ctx* ctx, const bbpe_table* t, const uint32_t* d_ids, const uint64_t* d_tok_offsets,
                          size_t n_rows, uint64_t n_ids, int skip_specials, uint8_t* d_out_bytes, uint64_t cap,
                          uint64_t* d_out_byte_offsets, uint64_t* total);

/* ---- JSON-lines text of a device CSR batch (
 * write_batch_jsonl, batch.hpp:157-166): {"ids":[...],"len":n}\n per row,
 * byte-identical to the compact nlohmann dump. Writes at most cap bytes;
 * *total receives the full text length. Synchronous. ---- */
int bbpe_jsonl_device(bbpe_ctx* ctx, const uint32_t* d_ids, const uint64_t* d_tok_offsets, size_t n_rows,
                      uint64_t n_ids, uint8_t* d_out, uint64_t cap, uint64_t* total);

/* ---- encode_batch's padded BatchEncoding on the device (
 * batch.hpp:64-126) from device CSR ids: row r = [bos] + ids + [eos],
 * right-truncated to max_len, pad_id elsewhere, u32 lengths, u8 mask.
 * bos_id / eos_id = 0xFFFFFFFF: not added. Both calls are synchronous. ---- */
/* Widest row (ids + add_bos + add_eos): the max_len encode_batch uses without limits. */
int bbpe_batch_widest_device(bbpe_ctx* ctx, const uint64_t* d_tok_offsets, size_t n_rows, int add_bos,
                             int add_eos, uint64_t* widest);
int bbpe_pad_device(bbpe_ctx* ctx, const uint32_t* d_ids, const uint64_t* d_tok_offsets, size_t n_rows,
                    uint32_t pad_id, uint32_t bos_id, uint32_t eos_id, uint64_t max_len, uint32_t* d_out_ids,
                    uint32_t* d_lengths, uint8_t* d_mask, uint64_t* truncated_rows);

/* The gpt2 split pattern's chunk starts (pattern_pretokenize, pretokenize.hpp:
 * 79-264, applied to every row; row starts included) as a bitmap of
 * (total_bytes + 31) / 32 u32 words at d_chunk_bits (bit p: a chunk starts at
 * byte p). The splitter that bbpe_config.pattern = 1 runs; device buffers,
 * synchronous. */
int bbpe_pretokenize_device(bbpe_ctx* ctx, const uint8_t* d_bytes, const uint64_t* d_offsets, size_t n_rows,
                            uint64_t total_bytes, uint32_t* d_chunk_bits);

/* ---- special tokens on the device ----
 * bbpe_ctx_set_specials replaces the ctx's special-token set (SpecialTokenSet,
 * merge_table.hpp:309-369): n byte strings blob[offsets[i], offsets[i+1]) with
 * ids[i]; empty or duplicate strings are BBPE_USAGE; n = 0 clears the set.
 * bbpe_encode_batch_device then produces encode_batch's rows (batch.hpp:64-126,
 * unpadded) as CSR: each row split at the specials (split_specials,
 * pretokenize.hpp:32-57: greedy, longest special first), literal segments
 * BPE-encoded, special ids passed through, bos_id / eos_id added unless
 * 0xFFFFFFFF. All buffers are device buffers; out_capacity ids are available
 * at d_out_ids (BBPE_USAGE if the rows need more); *n_out_ids receives the
 * total. Errors carry the input row ("row r: "). Synchronous. */
int bbpe_ctx_set_specials(bbpe_ctx* ctx, size_t n, const uint8_t* blob, const uint64_t* offsets,
                          const uint32_t* ids);
int bbpe_encode_batch_device(bbpe_ctx* ctx, const bbpe_table* t, const uint8_t* d_bytes,
                             const uint64_t* d_offsets, size_t n_rows, uint64_t total_bytes, uint32_t bos_id,
                             uint32_t eos_id, uint32_t* d_out_ids, uint64_t out_capacity,
                             uint64_t* d_out_offsets, uint64_t* n_out_ids);
/* The same on host buffers (offsets[0] may be non-zero; out_offsets start at 0). */
int bbpe_encode_batch(bbpe_ctx* ctx, const bbpe_table* t, const uint8_t* bytes, const uint64_t* offsets,
                      size_t n_rows, uint32_t bos_id, uint32_t eos_id, uint32_t* out_ids, uint64_t out_capacity,
                      uint64_t* out_offsets, uint64_t* n_out_ids);

/* ---- per-device encode contexts ---- */
int bbpe_ctx_create(int device, const bbpe_config* cfg, bbpe_ctx** out);
int bbpe_ctx_destroy(bbpe_ctx* ctx);
int bbpe_ctx_set_config(bbpe_ctx* ctx, const bbpe_config* cfg);
/* Upload (once) the table replica for this ctx's device. Implicit on first use. */
int bbpe_ctx_prepare(bbpe_ctx* ctx, const bbpe_table* t);
/* Page-locked host buffers for zero-copy staging (cudaHostAlloc). */
int bbpe_host_alloc(size_t bytes, void** out);
int bbpe_host_free(void* p);

/* Batch encode from HOST buffers. Row r is bytes[offsets[r] .. offsets[r+1]).
 * Output is CSR: ids of row r are out_ids[out_offsets[r] .. out_offsets[r+1]).
 * out_capacity must be >= the token total; offsets[n] (= total bytes) always
 * suffices since every token covers at least one byte. */
int bbpe_encode(bbpe_ctx* ctx, const bbpe_table* t, const uint8_t* bytes, const uint64_t* offsets,
                size_t n, uint32_t* out_ids, uint64_t out_capacity, uint64_t* out_offsets,
                bbpe_stats* stats);

/* Batch encode from DEVICE buffers on ctx's device, stream-ordered on `stream`
 * (a cudaStream_t, or NULL for the ctx's own stream). d_out_ids needs
 * total_bytes slots. total_bytes must equal d_offsets[n]. If sync is 0 the
 * call only enqueues work; errors raised on the device are then reported by
 * the next bbpe_ctx_sync. */
int bbpe_encode_device(bbpe_ctx* ctx, const bbpe_table* t, const uint8_t* d_bytes,
                       const uint64_t* d_offsets, size_t n, uint64_t total_bytes,
                       uint32_t* d_out_ids, uint64_t* d_out_offsets, void* stream, int sync,
                       bbpe_stats* stats);
int bbpe_ctx_sync(bbpe_ctx* ctx);
/* How many of this library's kernels the ctx has launched since creation. */
uint64_t bbpe_ctx_kernel_launches(const bbpe_ctx* ctx);
/* Per-kernel device time (CUDA events recorded between launches on the
 * launching stream) summed over the encodes since the last reset:
 * ms[0] k_tile_first (+ the gpt2 splitter in pattern mode), ms[1] k_pieces
 * (or k_block_rows), ms[2] k_dedup, ms[3] k_merge, ms[4] k_refs,
 * ms[5] k_long_pieces, ms[6] k_tile_scan, ms[7] k_gather (0 for a kernel
 * that did not run). Synchronises the streams used. *calls receives the
 * number of encodes. */
#define BBPE_N_KERNELS 8
int bbpe_ctx_kernel_times(bbpe_ctx* ctx, double* ms, uint64_t* calls, int reset);

/* Piece statistics of the encodes on this ctx since the last reset (what the
 * piece decomposition did with the input; diagnostics for the bench):
 * out[0] pieces, out[1] pieces resolved from the piece memo / byte LUT,
 * out[2] pieces sent to the lane-per-piece merge loop, out[3] long pieces
 * (> 32 bytes, or whole rows under BBPE_ENGINE_BLOCK), out[4] bytes in long
 * pieces, out[5] distinct merge pieces actually merged after the within-call
 * dedupe (0 when the dedupe did not run), out[6] input bytes. No reference
 * counterpart. Synchronises the device. */
#define BBPE_N_PIECE_STATS 7
int bbpe_ctx_piece_stats(bbpe_ctx* ctx, uint64_t* out, int reset);

/* block_bpe on explicit initial token ids (one sequence), always the
 * BBPE_ENGINE_BLOCK pass loop. trace (optional): per pass {pass_index (1-based),
 * min_rank, merges_applied} as 3 x u64, up to trace_cap passes; *n_passes gets
 * the full count. On BBPE_MAX_PASSES, out holds the partial state and *out_n
 * its length (MaxPassesError::partial_tokens / passes_run). */
int bbpe_block_bpe(bbpe_ctx* ctx, const bbpe_table* t, const uint32_t* tokens, size_t n,
                   uint32_t* out, size_t* out_n, uint64_t* trace, size_t trace_cap,
                   size_t* n_passes);

/* ---- spec-level operations (block_engine.hpp:189-256) on the device ----
 * A per-phase replay of one block_bpe pass, with the reference's contract
 * checks: BBPE_CONTRACT (ContractViolation) with the reference's messages.
 * Host buffers in and out; each call runs its kernels on the ctx's device.
 *   bbpe_pair_ranks      <- pair_ranks (189-199): ranks[i] = rank of
 *                           (tokens[i], tokens[i+1]) or 0xFFFFFFFF, n-1 entries
 *   bbpe_min_rank_reduce <- min_rank_reduce (201-206): 0xFFFFFFFF = none
 *   bbpe_mark_merges     <- mark_merges (211-220): n flags, left-greedy
 *   bbpe_exclusive_scan  <- exclusive_scan (223-235): flags must be 0/1 and
 *                           never adjacent
 *   bbpe_compact         <- compact (238-256) and compact_into (166-182):
 *                           lengths, offsets = exclusive scan of flags, and
 *                           every flagged pair a merge of the table */
int bbpe_pair_ranks(bbpe_ctx* ctx, const bbpe_table* t, const uint32_t* tokens, size_t n, uint32_t* ranks);
int bbpe_min_rank_reduce(bbpe_ctx* ctx, const uint32_t* ranks, size_t n, uint32_t* out);
int bbpe_mark_merges(bbpe_ctx* ctx, const bbpe_table* t, const uint32_t* tokens, size_t n, uint32_t min_rank,
                     uint8_t* flags);
int bbpe_exclusive_scan(bbpe_ctx* ctx, const uint8_t* flags, size_t n, uint32_t* offsets);
int bbpe_compact(bbpe_ctx* ctx, const bbpe_table* t, const uint32_t* tokens, size_t n, const uint8_t* flags,
                 size_t n_flags, const uint32_t* offsets, size_t n_offsets, uint32_t* out, size_t* out_n);

/* ---- multi-GPU ---- */
/* Splits rows [0, n) into `parts` contiguous shards with near-equal cost,
 * cost(row) = len + 64 (bytes plus a per-row overhead). bounds gets parts+1
 * row indices. */
int bbpe_partition(const uint64_t* offsets, size_t n, int parts, uint64_t* bounds);
/* Shards the batch across `n_devices` ctxs (one host thread each; tables are
 * replicated per device), stitches CSR output. No collective is involved. */
int bbpe_encode_sharded(bbpe_ctx* const* ctxs, int n_devices, const bbpe_table* t,
                        const uint8_t* bytes, const uint64_t* offsets, size_t n,
                        uint32_t* out_ids, uint64_t out_capacity, uint64_t* out_offsets,
                        bbpe_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* BBPE_B200_H */
