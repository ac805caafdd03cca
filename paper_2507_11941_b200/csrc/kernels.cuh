// kernels.cuh -- launch interface of the sm_100a BlockBPE kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bbpe_internal.h"

namespace bbpe {

#ifndef BBPE_TILE
#define BBPE_TILE 512
#endif
constexpr int kTile = BBPE_TILE;    // input bytes owned by one warp-tile
constexpr int kLmax = 32;           // longest piece merged by a single lane
constexpr int kWin = kTile + kLmax + 1;  // window positions [0, kWin) after b0
constexpr int kStage = kTile + kLmax;  // staging slots per tile (short-piece tokens)
constexpr int kScanTilesPerCta = 4096;  // k_tile_scan: 512 threads x 8 tiles
constexpr int kWarpsPerCta = 8;
#ifndef BBPE_TILES_PER_TICKET
#define BBPE_TILES_PER_TICKET 4
#endif
constexpr int kTilesPerTicket = BBPE_TILES_PER_TICKET;  // k_pieces: consecutive tiles per ticket
#ifndef BBPE_LP_WARPS
#define BBPE_LP_WARPS 4
#endif
#ifndef BBPE_LP_MINB
#define BBPE_LP_MINB 4
#endif
#ifndef BBPE_LP_SMEM
#define BBPE_LP_SMEM 8192
#endif
constexpr int kLpMinBlocks = BBPE_LP_MINB;  // k_long_sp (shared-memory instance): resident CTAs per SM (register cap)
constexpr int kLpWarps = BBPE_LP_WARPS;     // k_long_pieces: warps per CTA (one piece per warp)
constexpr int kLpSmemBytes = BBPE_LP_SMEM;  // long pieces: shared-memory bytes per warp (k_long_sp: 1024 positions)
constexpr int kWinVec = (kTile + 48) / 16;  // 16-byte chunks of a tile window: bytes [b0-16, b0+kTile+32)
constexpr int kRowWords = kTile / 32 + 4;   // row-start bit words copied per tile (whole 16-byte chunks)
constexpr int kMrecChunk = 256;     // merge records a warp reserves at a time
constexpr uint32_t kSentinel = 0xFFFFFFFFu;  // staging slot left empty by a merge piece
#ifndef BBPE_DEDUP_BYTES_PER_SLOT
#define BBPE_DEDUP_BYTES_PER_SLOT 128  // within-call dedupe table: one slot per this many input bytes
#endif
#ifndef BBPE_DEDUP_PROBES
#define BBPE_DEDUP_PROBES 4  // slots a piece probes before it gives up on the dedupe (mixed text: k_dedup 1.27 -> 0.94 ms at 16 -> 4)
#endif
constexpr int kDedupMax = 15;       // longest merge piece deduplicated within a call
constexpr uint64_t kDedupMinBytes = 64ull << 20;  // smaller batches: the dedupe pass costs more than it saves
constexpr uint64_t kRefFlag = 1ull << 62;  // merge-record header: a reference (k_dedup)
// DedupRes (32 bytes per dedupe slot): {staging index | count << 48, then up
// to kInlineRes result tokens (original ids, u32)}; references copy inline
// results without touching the owner's staging.
constexpr int kInlineRes = 6;

// Counter slots (u32).
enum { CNT_TILE_TICKET = 0, CNT_LONG = 1, CNT_LP_NEXT = 2, CNT_GROUP_TICKET = 3, CNT_LREC = 4,
       CNT_MERGE_TICKET = 5, CNT_MREC = 6, CNT_OWNERS = 7, CNT_PRETOK = 8, CNT_LCOPY = 9, CNT_LDONE = 10,
       CNT_LP_NEXT2 = 11, CNT_LONG2 = 12, CNT_N = 13 };
// k_gather leaves CNT_LREC / CNT_LCOPY / CNT_LDONE for k_long_copy, which resets them.
// Error slots (u64, initialised to ~0).
enum { ERR_BAD_BYTE_POS = 0, ERR_MAXPASS_ROW = 1, ERR_CONTRACT = 2, ERR_BAD_OFFSETS = 3, ERR_N = 4 };

// Deferred pieces, found by k_pieces (or k_block_rows) and merged later:
//  * long piece (> kLmax bytes, or a whole row under BBPE_ENGINE_BLOCK): a
//    LongRec, merged by k_long_pieces into lpo; takes no staging slots. The
//    long records of one tile are contiguous and in piece order (k_gather
//    interleaves their tokens with the tile's staging slots).
//  * merge piece (2..kLmax bytes, not in the piece memo): a 16-byte record
//    in `mrec`: {start << 16 | spref << 6 | len, the piece's first 8 bytes},
//    merged by k_merge into the `len` staging slots reserved at `spref`;
//    unused slots get kSentinel and the tile's token count drops by
//    len - count. A header of ~0 marks an unused record.
struct LongRec {
  uint64_t start;  // absolute byte position (token position for token input)
  uint64_t len;
  uint64_t row;    // row index (MaxPassesError reporting)
  uint32_t spref;  // staging slots of the tile before this piece
  uint32_t count;  // tokens out, written by the merging kernel
  uint64_t out;    // first output position (k_gather), for k_long_copy
};
__host__ __device__ inline uint64_t pack_mrec(uint64_t start, uint32_t spref, uint32_t len) {
  return (start << 16) | (uint64_t(spref) << 6) | len;
}

struct EncodeArgs {
  const uint8_t* bytes;
  const uint64_t* offsets;  // n_rows + 1, offsets[0] == 0
  const uint64_t* offsets_raw;  // optional: offsets + offsets_base, rebased by k_tile_first into offsets_w
  uint64_t* offsets_w;
  uint64_t offsets_base;
  uint64_t n_rows;
  uint64_t total;           // offsets[n_rows]
  uint64_t num_tiles;
  uint32_t* out_ids;
  uint64_t* out_offsets;
  // scratch
  uint64_t* tile_first;     // num_tiles + 1
  uint64_t* status;         // look-back words of k_tile_scan's CTAs
  uint64_t num_groups;      // k_tile_scan CTAs
  uint64_t* tile_base;      // num_tiles + 1: first output token of each tile
  uint32_t* staging;        // num_tiles * kStage: each tile's short-piece tokens, in order
  uint32_t* tile_count;     // num_tiles: tokens produced by the tile (final after k_merge/k_long_pieces)
  uint32_t* tile_slots;     // num_tiles: staging slots the tile used (incl. reserved)
  uint64_t* tile_lrec;      // num_tiles: (first LongRec << 24) | n long pieces, 0 when none
  uint32_t* rowbits;        // (num_tiles + 1) * (kTile/32) + kRowWords words: row-start bit per byte
  uint32_t* chunkbits;      // same layout, pattern mode only (else null): split-pattern chunk starts
  int bytes_aligned;        // bytes pointer is 16-byte aligned (cp.async window loads)
  ulonglong2* mrec;         // mrec_cap merge records (CNT_MREC allocated); k_merge
                            // leaves an owner's token count in .y
  uint64_t mrec_cap;
  // Within-call dedupe of merge pieces of <= kDedupMax bytes (dmask 0: off),
  // k_dedup: dkey[slot] = 16-byte key (15 zero-padded bytes, len in the top
  // byte), claimed by 128-bit CAS. The claimer owns the slot (downer[slot] =
  // its record, listed in `owners` for k_merge); a record whose bytes are
  // already owned becomes a reference {hdr | kRefFlag, slot} for k_refs.
  ulonglong2* dkey;
  uint64_t* dres;           // 4 u64 per slot, set by the owner in k_merge (DedupRes)
  uint64_t dmask;
  uint64_t* owners;         // mrec_cap: record index | (slot + 1) << 32 for k_merge (CNT_OWNERS used)
  LongRec* lrec;            // lp_cap records (CNT_LREC used)
  uint32_t* long_idx;       // indices of the long records (CNT_LONG used)
  uint32_t* long_idx2;      // the pieces > kPipeMin positions among them (CNT_LONG2 used; k_long_sp)
  uint64_t long_cap;
  uint32_t* counters;       // CNT_N
  uint64_t* err;            // ERR_N
  uint64_t lp_cap;
  uint32_t* lpo;            // total + 1: long-piece results {count, tokens...} at start
  uint64_t* lpx;            // total: long-piece working set {token | rank << 32}
  uint64_t* lpy;            // total: double buffer
  uint64_t* trace;          // optional per-pass trace (single piece), 3 x u64 per pass
  uint64_t trace_cap;
  uint64_t* trace_count;
  int engine;               // bbpe_engine
  int narrow;               // 1: 16-bit working arrays (ids < 0xFFFE, merges < 0xFFFE)
  int use_memo;             // 1: look whole pieces up in the table's piece memo first
  int tokens_input;         // 1: lpx already holds initial tokens (bbpe_block_bpe)
  int pattern;              // 1: gpt2 split pattern chunk starts are piece boundaries (pretok.cu)
  int64_t max_passes;       // <= 0: none
  uint64_t* pstats;         // PST_N piece statistics, accumulated across encodes (never reset by kernels)
};
// Piece statistics (bbpe_ctx_piece_stats): per-warp counts added once per warp.
enum { PST_PIECES = 0, PST_MEMO = 1, PST_MERGE = 2, PST_LONG = 3, PST_LONG_BYTES = 4, PST_OWNERS = 5,
       PST_BYTES = 6, PST_N = 8 };

struct LaunchPlan {
  int main_grid = 0;
  int main_grid_wide = 0;
  int merge_grid = 0;
  int merge_grid_wide = 0;
  int gather_grid = 0;
  int lp_grid = 0;
  int sm_count = 0;
};

LaunchPlan plan_launch(int device);
// Enqueues the full encode on `stream`; returns the number of kernels launched.
// ev (optional): BBPE_N_KERNELS + 1 events, before the first and after each kernel.
// Row starts + the gpt2 splitter only: chunk starts (row starts included) as a
// bitmap of (total + 31) / 32 words into d_out_bits. Returns the launch count.
int launch_pretok_only(const EncodeArgs& a, const LaunchPlan& p, uint32_t* d_out_bits, cudaStream_t stream);
int launch_encode(const EncodeArgs& a, const DevTable& t, const LaunchPlan& p, cudaStream_t stream,
                  cudaEvent_t* ev = nullptr);
// Copies one wave's results into the caller's device-mapped pinned buffers:
// row offsets (wave-relative + *run_base) and ids at *run_base (clamped to
// cap), then advances *run_base by the wave's token count.
// p[i] += v for i < n (chunked device encodes: a chunk's offsets onto the running base).
void launch_add_u64(uint64_t* d_p, uint64_t n, uint64_t v, int sm_count, cudaStream_t stream);
void launch_copy_out(const uint32_t* d_ids, uint32_t* mapped_out, const uint64_t* d_wave_offsets,
                     uint64_t* mapped_offsets, uint64_t nr, uint64_t* run_base, uint64_t cap, int sm_count,
                     cudaStream_t stream);
// k_long_pieces (longpieces.cu): the warp-per-piece block engine.
size_t long_pieces_smem(bool narrow);
int long_pieces_grid(int device, int sm_count);
int launch_long_pieces(const EncodeArgs& a, const DevTable& t, int grid, cudaStream_t stream);  // kernels launched
// Spec-level ops (specops.cu): per-phase replay of one block_bpe pass.
void launch_spec_ranks(const uint32_t* tok, uint64_t n, const DevTable& t, uint32_t* ranks, cudaStream_t s);
void launch_spec_min(const uint32_t* ranks, uint64_t n, uint32_t* out, cudaStream_t s);
void launch_spec_runs(const uint32_t* ranks, uint64_t n, uint32_t m, uint8_t* flags, cudaStream_t s);
void launch_spec_check(const uint8_t* flags, uint64_t n, unsigned long long* err, cudaStream_t s);
void launch_spec_scan(const uint8_t* flags, uint64_t n, uint32_t* offsets, uint32_t* total, cudaStream_t s);
void launch_spec_check_offsets(const uint32_t* offsets, const uint32_t* scan, uint64_t n, unsigned long long* err,
                               cudaStream_t s);
void launch_spec_compact(const uint32_t* dtok, const uint32_t* orig, const uint8_t* flags, const uint32_t* offsets,
                         uint64_t n, const DevTable& t, uint32_t* out, unsigned long long* err, cudaStream_t s);
// k_long_copy: long pieces' tokens into their CSR places (after k_gather).
void launch_long_copy(const EncodeArgs& a, const DevTable& t, int grid, cudaStream_t stream);
// Long-piece kernel only (token input, used by bbpe_block_bpe).
int launch_block_bpe(const EncodeArgs& a, const DevTable& t, const LaunchPlan& p,
                     cudaStream_t stream);

}  // namespace bbpe
