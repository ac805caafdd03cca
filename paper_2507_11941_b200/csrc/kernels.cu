// kernels.cu -- the sm_100a BlockBPE encode kernels.
//
// Semantics: bit-exact with the reference block engine, block_bpe
// (reference proj/include/blockbpe/block_engine.hpp:268-310): per pass, rank
// every adjacent pair (fill_pair_ranks 72-79), take the minimum (82-97), mark
// left-greedy non-overlapping occurrences (103-128), scan (133-162), compact
// (166-182); repeat until no pair is in the table.
//
// Decomposition: a byte position p of a row
// is a HARD BOUNDARY when the bigram (s[p-1], s[p]) is not the junction
// (last byte of left, first byte of right) of any merge. No merge can ever
// produce a token spanning a hard boundary, so the rows' pass loops factor into
// independent pass loops over the pieces between hard boundaries, and every
// piece evolves exactly as it does inside the whole-row pass loop (the global
// pass order only interleaves independent pieces). Pieces of <= kLmax bytes are
// merged by one lane each; longer pieces (and, with BBPE_ENGINE_BLOCK, whole
// rows) by one CTA each with the reference's phase structure.
//
// Kernels (one stream, no host sync in between):
//   k_tile_first  : row index of the first row starting at or after each tile
//   k_prepass     : invalid-byte check, long-piece discovery
//   k_long_pieces : CTA-per-piece pass loop (the paper's block engine)
//   k_encode      : warp-per-tile piece split + lane-per-piece pass loop +
//                   decoupled look-back -> CSR ids and row offsets, written once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace bbpe {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kProbe = 0xFFFFFFFEu;   // rank not yet looked up
constexpr uint32_t kMergeMark = 0xFFFFFFFDu;
constexpr uint32_t kUnchanged = 0x80000000u;  // lpo flag: piece merged nothing
constexpr int kWords = (kWin + 31) / 32;
constexpr int kTileWords = kTile / 32;
constexpr int kMaxLongPerTile = kTile / (kLmax + 1) + 2;
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t dmix64(uint64_t h) {
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdULL;
  h ^= h >> 33;
  return h;
}

// Pair -> dense rank (kNoRank when absent). One 32-byte bucket per step.
__device__ __forceinline__ uint32_t probe(const DevTable& T, uint32_t l, uint32_t r) {
  const uint64_t key = (uint64_t(l) << T.id_bits) | uint64_t(r);
  uint64_t b = dmix64(key) & T.bucket_mask;
  const uint64_t rmask = (1ull << T.rank_bits) - 1;
  for (;;) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.slots + b * kBucketSlots);
    ulonglong2 s01 = __ldg(p);
    ulonglong2 s23 = __ldg(p + 1);
    uint64_t s[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (s[j] == kEmptySlot) return kNoRank;
      if ((s[j] >> T.rank_bits) == key) return static_cast<uint32_t>(s[j] & rmask);
    }
    b = (b + 1) & T.bucket_mask;
  }
}

__device__ __forceinline__ bool is_junction(const uint32_t* junc, uint32_t a, uint32_t c) {
  uint32_t bit = (a << 8) | c;
  return (junc[bit >> 5] >> (bit & 31)) & 1u;
}

__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t warp_incl_sum(uint32_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t u = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += u;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  return v;
}
__device__ __forceinline__ unsigned lanemask_lt(int lane) { return (1u << lane) - 1u; }

// ---------------------------------------------------------------------------
// k_tile_first: F(t) = min{ s : offsets[s] >= t*kTile }, t in [0, num_tiles).
// Row s owns tiles t with offsets[s-1] < t*kTile <= offsets[s].
__global__ void k_tile_first(EncodeArgs a) {
  uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (s > a.n_rows) return;
  uint64_t hi = a.offsets[s] / kTile;
  uint64_t lo = (s == 0) ? 0 : a.offsets[s - 1] / kTile + 1;
  if (s == 0) hi = 0;  // offsets[0] == 0
  for (uint64_t t = lo; t <= hi && t < a.num_tiles; ++t) a.tile_first[t] = s;
  if (s == 0) a.tile_first[a.num_tiles] = a.n_rows + 1;
}

// ---------------------------------------------------------------------------
// Per-warp window over [b0-1, b0+kWin): bytes, row starts, hard boundaries.
struct Window {
  uint8_t wb[kWin + 8];    // wb[q+1] = byte at b0+q, wb[0] = byte at b0-1
  uint32_t sb[kWords];     // row-start bits
  uint32_t bd[kWords];     // piece-boundary bits
};

__device__ void load_window(Window& w, const EncodeArgs& a, const uint32_t* junc, uint64_t tile,
                            int lane, bool block_engine) {
  const uint64_t b0 = tile * kTile;
  // Bytes. Aligned 4-byte words covering [b0-4, b0+kWin+4).
  const uint64_t wbase = b0 >= 4 ? b0 - 4 : 0;
  for (int i = lane; i < (kWin + 12) / 4; i += 32) {
    uint64_t pos = wbase + 4ull * i;
    uint32_t v = 0;
    if (pos + 4 <= a.total) {
      v = __ldg(reinterpret_cast<const uint32_t*>(a.bytes + pos));
    } else {
      for (int k = 0; k < 4; ++k)
        if (pos + k < a.total) v |= uint32_t(a.bytes[pos + k]) << (8 * k);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int64_t q = int64_t(pos + k) - int64_t(b0);  // relative position
      if (q >= -1 && q < kWin) w.wb[q + 1] = uint8_t(v >> (8 * k));
    }
  }
  if (b0 == 0 && lane == 0) w.wb[0] = 0;
  for (int i = lane; i < kWords; i += 32) w.sb[i] = 0;
  __syncwarp();
  // Row starts inside the window.
  uint64_t s0 = a.tile_first[tile];
  for (uint64_t s = s0;; s += 32) {
    uint64_t my = s + lane;
    bool in = false;
    uint64_t o = 0;
    if (my <= a.n_rows) {
      o = a.offsets[my];
      in = o < b0 + kWin;
    }
    if (in) atomicOr(&w.sb[(o - b0) >> 5], 1u << ((o - b0) & 31));
    if (__ballot_sync(kFull, in) != kFull) break;
  }
  __syncwarp();
  // Boundaries.
  for (int wd = 0; wd < kWords; ++wd) {
    int q = wd * 32 + lane;
    uint64_t abs = b0 + q;
    bool b = true;
    if (q < kWin && abs < a.total) {
      b = (w.sb[wd] >> lane) & 1u;
      if (!b && !block_engine) b = !is_junction(junc, w.wb[q], w.wb[q + 1]);
    }
    unsigned m = __ballot_sync(kFull, b);
    if (lane == 0) w.bd[wd] = m;
  }
  __syncwarp();
}

// First boundary strictly after q, searching positions (q, q+limit]; returns
// q+limit+1 when there is none in range.
__device__ __forceinline__ int next_boundary(const uint32_t* bd, int q, int limit) {
  int p = q + 1;
  int last = q + limit;
  while (p <= last) {
    uint32_t bits = bd[p >> 5] >> (p & 31);
    if (bits) {
      int r = p + __ffs(bits) - 1;
      return r <= last ? r : last + 1;
    }
    p = (p | 31) + 1;
  }
  return last + 1;
}

// ---------------------------------------------------------------------------
// k_prepass: invalid bytes (IntegrityError, pretokenize.hpp:64-67) and long
// pieces (> kLmax bytes, or every row under BBPE_ENGINE_BLOCK).
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_prepass(EncodeArgs a, DevTable T) {
  __shared__ uint32_t s_lut[256];
  __shared__ uint32_t s_junc[2048];
  __shared__ Window s_win[kWarpsPerCta];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s_junc[i] = T.junction[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Window& w = s_win[wid];
  const bool block_engine = a.engine == BBPE_ENGINE_BLOCK;
  const uint64_t nwarps = uint64_t(gridDim.x) * kWarpsPerCta;
  for (uint64_t tile = blockIdx.x * uint64_t(kWarpsPerCta) + wid; tile < a.num_tiles;
       tile += nwarps) {
    const uint64_t b0 = tile * kTile;
    const int tlen = int(min((uint64_t)kTile, (uint64_t)(a.total - b0)));
    if (block_engine) {
      // Every non-empty row starting in this tile is one long piece.
      uint64_t s0 = a.tile_first[tile], s1 = a.tile_first[tile + 1];
      for (uint64_t s = s0 + lane; s < s1 && s < a.n_rows; s += 32) {
        uint64_t o = a.offsets[s], e = a.offsets[s + 1];
        if (e > o) {
          uint32_t slot = atomicAdd(&a.counters[CNT_LP_COUNT], 1u);
          if (slot < a.lp_cap) a.lp[slot] = LongPiece{o, e - o, s};
        }
      }
      // Invalid bytes still need checking.
      for (int q = lane; q < tlen; q += 32) {
        uint8_t byte = a.bytes[b0 + q];
        unsigned bad = __ballot_sync(__activemask(), s_lut[byte] == kInvalidToken);
        if (bad && lane == __ffs(bad) - 1) atomicMin(reinterpret_cast<unsigned long long*>(&a.err[ERR_BAD_BYTE_POS]), b0 + q);
      }
      continue;
    }
    load_window(w, a, s_junc, tile, lane, false);
    // Invalid bytes.
    for (int wd = 0; wd * 32 < tlen; ++wd) {
      int q = wd * 32 + lane;
      bool bad = q < tlen && s_lut[w.wb[q + 1]] == kInvalidToken;
      unsigned m = __ballot_sync(kFull, bad);
      if (m && lane == 0) {
        atomicMin(reinterpret_cast<unsigned long long*>(&a.err[ERR_BAD_BYTE_POS]),
                  (unsigned long long)(b0 + wd * 32 + __ffs(m) - 1));
      }
    }
    // Long pieces: starts in [0, tlen) with no boundary within kLmax bytes.
    for (int wd = 0; wd * 32 < tlen; ++wd) {
      int q = wd * 32 + lane;
      bool start = q < tlen && ((w.bd[wd] >> lane) & 1u);
      bool longp = start && next_boundary(w.bd, q, kLmax) > q + kLmax;
      unsigned lm = __ballot_sync(kFull, longp);
      while (lm) {
        int src = __ffs(lm) - 1;
        lm &= lm - 1;
        int lq = __shfl_sync(kFull, q, src);
        uint64_t abs = b0 + lq;
        // Row of the piece (rare path): binary search on offsets.
        uint64_t row = 0, row_end = 0;
        if (lane == 0) {
          uint64_t lo = 0, hi = a.n_rows;  // find max s with offsets[s] <= abs
          while (lo < hi) {
            uint64_t mid = (lo + hi + 1) >> 1;
            if (a.offsets[mid] <= abs) lo = mid; else hi = mid - 1;
          }
          row = lo;
          row_end = a.offsets[row + 1];
        }
        row = __shfl_sync(kFull, row, 0);
        row_end = __shfl_sync(kFull, row_end, 0);
        // Scan forward for the first hard boundary (pieces never cross rows).
        uint64_t end = row_end;
        for (uint64_t x = abs + kLmax + 1; x < row_end; x += 32) {
          uint64_t y = x + lane;
          bool b = y < row_end && !is_junction(s_junc, a.bytes[y - 1], a.bytes[y]);
          unsigned bm = __ballot_sync(kFull, b);
          if (bm) {
            end = x + __ffs(bm) - 1;
            break;
          }
        }
        if (lane == 0) {
          uint32_t slot = atomicAdd(&a.counters[CNT_LP_COUNT], 1u);
          if (slot < a.lp_cap) a.lp[slot] = LongPiece{abs, end - abs, row};
        }
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Block-level helpers for the CTA-per-piece kernel.
template <int NT>
struct BlockScratch {
  uint32_t red_u32[2][32];
  int32_t red_i32[2][32];
  uint32_t bcast_u32[4];
  int32_t bcast_i32[4];
};

template <int NT>
__device__ uint32_t block_min_u32(uint32_t v, BlockScratch<NT>& sc, int slot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = __reduce_min_sync(kFull, v);
  if (lane == 0) sc.red_u32[slot][wid] = v;
  __syncthreads();
  if (wid == 0) {
    uint32_t x = lane < NT / 32 ? sc.red_u32[slot][lane] : kNoRank;
    x = __reduce_min_sync(kFull, x);
    if (lane == 0) sc.bcast_u32[slot] = x;
  }
  __syncthreads();
  return sc.bcast_u32[slot];
}

// Exclusive scan (sum) of u32 over the block; *total receives the block sum.
template <int NT>
__device__ uint32_t block_excl_sum_u32(uint32_t v, BlockScratch<NT>& sc, int slot,
                                       uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t inc = warp_incl_sum(v, lane);
  if (lane == 31) sc.red_u32[slot][wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint32_t x = lane < NT / 32 ? sc.red_u32[slot][lane] : 0;
    uint32_t xi = warp_incl_sum(x, lane);
    if (lane < NT / 32) sc.red_u32[slot][lane] = xi - x;
    if (lane == 31) sc.bcast_u32[slot] = xi;
  }
  __syncthreads();
  *total = sc.bcast_u32[slot];
  return sc.red_u32[slot][wid] + inc - v;
}

// Exclusive max-scan of i32 (identity -1).
template <int NT>
__device__ int32_t block_excl_max_i32(int32_t v, BlockScratch<NT>& sc, int slot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int32_t u = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc = max(inc, u);
  }
  int32_t exc = __shfl_up_sync(kFull, inc, 1);
  if (lane == 0) exc = -1;
  if (lane == 31) sc.red_i32[slot][wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int32_t x = lane < NT / 32 ? sc.red_i32[slot][lane] : -1;
    int32_t xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int32_t u = __shfl_up_sync(kFull, xi, d);
      if (lane >= d) xi = max(xi, u);
    }
    int32_t xe = __shfl_up_sync(kFull, xi, 1);
    if (lane == 0) xe = -1;
    if (lane < NT / 32) sc.red_i32[slot][lane] = xe;
  }
  __syncthreads();
  return max(sc.red_i32[slot][wid], exc);
}

__device__ __forceinline__ uint32_t tok_of(uint64_t e) { return static_cast<uint32_t>(e); }
__device__ __forceinline__ uint32_t rank_of(uint64_t e) { return static_cast<uint32_t>(e >> 32); }
__device__ __forceinline__ uint64_t pack_tr(uint32_t t, uint32_t r) {
  return uint64_t(t) | (uint64_t(r) << 32);
}

// ---------------------------------------------------------------------------
// k_long_pieces: the block engine (block_engine.hpp:268-310) for one piece per
// CTA, persistent over the long-piece list. Working set {token, rank} pairs in
// global memory (L2-resident for pieces of a few MB), double-buffered like the
// reference (277-283, 306). Exactness-preserving deviations:
//   * ranks are cached and only pairs touching a merge are re-probed
//     (a pair whose two tokens are unchanged keeps its rank);
//   * the merged id of a pass is r2m[min_rank] (ranks are unique per pair,
//     merge_table.hpp:264-268), not a second probe per merge (173);
//   * left-greedy marking uses run parity: pair q merges iff rank(q) == m and
//     q - (start of its run of m's) is even, identical to flags[i+1] =
//     (ranks[i] == m && !flags[i]) (107-109).
template <int NT>
__global__ void __launch_bounds__(NT) k_long_pieces(EncodeArgs a, DevTable T) {
  __shared__ uint32_t s_lut[256];
  __shared__ BlockScratch<NT> sc;
  __shared__ uint32_t s_idx;
  for (int i = threadIdx.x; i < 256; i += NT) s_lut[i] = T.lut[i];
  const int tid = threadIdx.x;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_idx = atomicAdd(&a.counters[CNT_LP_NEXT], 1u);
    __syncthreads();
    const uint32_t idx = s_idx;
    const uint32_t count = min((uint64_t)a.counters[CNT_LP_COUNT], (uint64_t)a.lp_cap);
    if (idx >= count) return;
    const LongPiece P = a.lp[idx];
    const int32_t len = static_cast<int32_t>(P.len);
    uint64_t* X = a.lpx + P.start;
    uint64_t* Y = a.lpy + P.start;
    if (!a.tokens_input) {
      for (int32_t i = tid; i < len; i += NT) X[i] = pack_tr(s_lut[a.bytes[P.start + i]], kProbe);
    }
    __syncthreads();
    int32_t n = len;
    uint64_t pass = 0;
    bool maxpass_hit = false;
    while (n >= 2) {
      const int32_t chunk = (n + NT - 1) / NT;
      const int32_t c0 = min(n, tid * chunk), c1 = min(n, c0 + chunk);
      // (1) ranks for unresolved pairs + local min.
      uint32_t lmin = kNoRank;
      for (int32_t i = c0; i < c1 && i < n - 1; ++i) {
        uint64_t e = X[i];
        uint32_t r = rank_of(e);
        if (r == kProbe) {
          r = probe(T, tok_of(e), tok_of(X[i + 1]));
          X[i] = pack_tr(tok_of(e), r);
        }
        lmin = min(lmin, r);
      }
      const uint32_t m = block_min_u32<NT>(lmin, sc, 0);
      if (m == kNoRank) break;
      if (a.max_passes > 0 && pass >= uint64_t(a.max_passes)) {
        maxpass_hit = true;
        break;
      }
      // (2) start of the run of m's active at my chunk start.
      int32_t agg = -1;
      bool prev_is_m = (c0 > 0 && c0 < n) ? rank_of(X[c0 - 1]) == m : false;
      {
        bool pm = prev_is_m;
        for (int32_t i = c0; i < c1 && i < n - 1; ++i) {
          bool im = rank_of(X[i]) == m;
          if (im && !pm) agg = i;
          pm = im;
        }
      }
      const int32_t carry = block_excl_max_i32<NT>(agg, sc, 0);
      // (3) mark merges (run parity) and count them.
      uint32_t my_merges = 0;
      {
        int32_t s = carry;
        bool pm = prev_is_m;
        for (int32_t i = c0; i < c1 && i < n - 1; ++i) {
          uint64_t e = X[i];
          bool im = rank_of(e) == m;
          if (im) {
            if (!pm) s = i;
            if (((i - s) & 1) == 0) {
              X[i] = pack_tr(tok_of(e), kMergeMark);
              ++my_merges;
            }
          }
          pm = im;
        }
      }
      uint32_t total_merges;
      const uint32_t before = block_excl_sum_u32<NT>(my_merges, sc, 1, &total_merges);
      // (4) compaction into Y (block_engine.hpp:166-182) with cached ranks.
      const uint32_t M = T.r2m[m];
      {
        uint32_t run = before;  // merges at pair positions q < i
        for (int32_t i = c0; i < c1; ++i) {
          if (i > c0 && rank_of(X[i - 1]) == kMergeMark) ++run;
          bool removed = i > 0 && rank_of(X[i - 1]) == kMergeMark;
          if (removed) continue;
          uint64_t e = X[i];
          bool mi = (i < n - 1) && rank_of(e) == kMergeMark;
          bool mnext = (i + 1 < n - 1) && rank_of(X[i + 1]) == kMergeMark;
          uint32_t t = mi ? M : tok_of(e);
          uint32_t r = (mi || mnext) ? kProbe : rank_of(e);
          Y[i - run] = pack_tr(t, r);
        }
      }
      if (a.trace && tid == 0) {
        if (pass < a.trace_cap) {
          a.trace[3 * pass] = pass + 1;
          a.trace[3 * pass + 1] = T.rank_orig[m];
          a.trace[3 * pass + 2] = total_merges;
        }
      }
      ++pass;
      n -= static_cast<int32_t>(total_merges);
      uint64_t* tmp = X;
      X = Y;
      Y = tmp;
      __syncthreads();
    }
    __syncthreads();
    if (maxpass_hit && tid == 0)
      atomicMin(reinterpret_cast<unsigned long long*>(&a.err[ERR_MAXPASS_ROW]),
                (unsigned long long)P.row);
    if (a.trace && tid == 0 && a.trace_count) *a.trace_count = pass;
    // Result: lpo[start] = count, tokens follow when anything merged (or on token input).
    uint32_t* O = a.lpo + P.start;
    if (tid == 0) O[0] = static_cast<uint32_t>(n) | ((n == len && !a.tokens_input) ? kUnchanged : 0u);
    if (n < len || a.tokens_input)
      for (int32_t i = tid; i < n; i += NT) O[1 + i] = tok_of(X[i]);
  }
}

// ---------------------------------------------------------------------------
// k_encode: warp-per-tile. Per tile: window -> pieces -> lane-per-piece pass
// loops -> tile token count -> decoupled look-back -> CSR writes.
struct WarpSmem {
  Window w;
  uint16_t plist[kTile];
  uint32_t pref[kTile + 1];
  uint32_t tok[kWin + 1];
  uint32_t rnk[kWin + 1];
  uint32_t nlong;
  uint32_t longk[kMaxLongPerTile];
  uint64_t tile;
};

// One lane: the reference pass loop over a piece of n <= kLmax tokens held at
// tok[0..n) / rnk[0..n-1) (shared memory). Returns when no pair remains.
// Per pass: min over cached ranks, sweep-compact in place (left-greedy:
// a pair at the current minimum merges unless its left token was just
// consumed -- exactly flags[i+1] = (ranks[i] == m && !flags[i])), then
// re-probe only the pairs touching a merged token.
__device__ __forceinline__ int lane_pass(const DevTable& T, uint32_t* tok, uint32_t* rnk, int n) {
  uint32_t m = kNoRank;
  for (int i = 0; i < n - 1; ++i) m = min(m, rnk[i]);
  if (m == kNoRank) return -1;
  const uint32_t M = __ldg(T.r2m + m);
  int j = 0, i = 0;
  while (i < n) {
    uint32_t ri = (i < n - 1) ? rnk[i] : kNoRank;
    if (ri == m) {
      tok[j] = M;
      rnk[j] = kProbe;
      if (j > 0) rnk[j - 1] = kProbe;
      i += 2;
    } else {
      tok[j] = tok[i];
      rnk[j] = ri;
      i += 1;
    }
    ++j;
  }
  for (int k = 0; k < j - 1; ++k)
    if (rnk[k] == kProbe) rnk[k] = probe(T, tok[k], tok[k + 1]);
  return j;
}

__global__ void __launch_bounds__(kWarpsPerCta * 32) k_encode(EncodeArgs a, DevTable T) {
  __shared__ uint32_t s_lut[256];
  __shared__ uint32_t s_junc[2048];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s_junc[i] = T.junction[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem& S = reinterpret_cast<WarpSmem*>(s_dyn)[wid];
  const bool block_engine = a.engine == BBPE_ENGINE_BLOCK;

  for (;;) {
    uint64_t tile = 0;
    if (lane == 0) tile = atomicAdd(&a.counters[CNT_TILE_TICKET], 1u);
    tile = __shfl_sync(kFull, tile, 0);
    if (tile >= a.num_tiles) return;
    const uint64_t b0 = tile * kTile;
    const int tlen = int(min((uint64_t)kTile, (uint64_t)(a.total - b0)));
    load_window(S.w, a, s_junc, tile, lane, block_engine);

    // Piece list (ordered).
    int npieces = 0;
    for (int wd = 0; wd < kTileWords; ++wd) {
      int q = wd * 32 + lane;
      bool st = q < tlen && ((S.w.bd[wd] >> lane) & 1u);
      unsigned m = __ballot_sync(kFull, st);
      if (st) S.plist[npieces + __popc(m & lanemask_lt(lane))] = static_cast<uint16_t>(q);
      npieces += __popc(m);
    }
    if (lane == 0) S.nlong = 0;
    __syncwarp();

    // Lane-per-piece pass loops with dynamic piece assignment.
    int my_k = -1, my_n = 0, my_q = 0;
    int next_k = 0;
    for (;;) {
      const bool idle = my_n == 0;
      const unsigned im = __ballot_sync(kFull, idle);
      if (idle) {
        const int k = next_k + __popc(im & lanemask_lt(lane));
        my_k = -1;
        if (k < npieces) {
          my_k = k;
          my_q = S.plist[k];
          int len = block_engine ? kLmax + 2 : next_boundary(S.w.bd, my_q, kLmax) - my_q;
          if (len > kLmax) {
            // Long piece: merged by k_long_pieces; its count is in lpo[start].
            S.pref[k] = __ldcg(a.lpo + b0 + my_q) & ~kUnchanged;
            uint32_t slot = atomicAdd(&S.nlong, 1u);
            if (slot < kMaxLongPerTile) S.longk[slot] = k;
            my_n = 0;
          } else {
            uint32_t* tk = S.tok + my_q;
            uint32_t* rk = S.rnk + my_q;
            for (int i = 0; i < len; ++i) tk[i] = s_lut[S.w.wb[my_q + 1 + i]];
            for (int i = 0; i < len - 1; ++i) rk[i] = probe(T, tk[i], tk[i + 1]);
            if (len < 2) {
              S.pref[k] = len;
              my_n = 0;
            } else {
              my_n = len;
            }
          }
        }
      }
      next_k += __popc(im);
      const bool active = my_n >= 2;
      if (!__any_sync(kFull, active) && next_k >= npieces) break;
      if (active) {
        int r = lane_pass(T, S.tok + my_q, S.rnk + my_q, my_n);
        if (r < 0) {
          S.pref[my_k] = my_n;
          my_n = 0;
        } else {
          my_n = r;
          if (my_n < 2) {
            S.pref[my_k] = my_n;
            my_n = 0;
          }
        }
      }
    }
    __syncwarp();

    // Exclusive scan of piece counts -> pref (in place), tile total.
    uint32_t run = 0;
    for (int k0 = 0; k0 < npieces; k0 += 32) {
      int k = k0 + lane;
      uint32_t c = k < npieces ? S.pref[k] : 0;
      uint32_t inc = warp_incl_sum(c, lane);
      if (k < npieces) S.pref[k] = run + inc - c;
      run += __shfl_sync(kFull, inc, 31);
    }
    if (lane == 0) S.pref[npieces] = run;
    __syncwarp();
    const uint64_t agg = run;

    // Decoupled look-back over tiles (tickets are handed out in order, so every
    // predecessor is owned by a running warp).
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_release(&a.status[0], kFlagPrefix | agg);
    } else {
      if (lane == 0) st_release(&a.status[tile], kFlagAgg | agg);
      int64_t look = int64_t(tile) - 1;
      for (;;) {
        const int64_t idx = look - lane;
        uint64_t v = kFlagPrefix;
        for (;;) {
          if (idx >= 0) v = ld_acquire(&a.status[idx]);
          if (__all_sync(kFull, (v >> 62) != 0)) break;
          __nanosleep(64);
        }
        const unsigned pm = __ballot_sync(kFull, (v >> 62) == 2);
        const int first_p = pm ? __ffs(pm) - 1 : 31;
        uint64_t contrib = lane <= first_p ? (v & kValMask) : 0;
        excl += warp_sum64(contrib);
        if (pm) break;
        look -= 32;
      }
      if (lane == 0) st_release(&a.status[tile], kFlagPrefix | (excl + agg));
    }
    const uint64_t base = excl;

    // Token writes (short pieces by their lane; long pieces cooperatively).
    const uint32_t* d2id = T.d2id;
    for (int k0 = 0; k0 < npieces; k0 += 32) {
      int k = k0 + lane;
      if (k < npieces) {
        const uint32_t c = S.pref[k + 1] - S.pref[k];
        const int q = S.plist[k];
        const int len = block_engine ? kLmax + 2 : next_boundary(S.w.bd, q, kLmax) - q;
        if (len <= kLmax) {
          uint32_t* dst = a.out_ids + base + S.pref[k];
          for (uint32_t i = 0; i < c; ++i) {
            uint32_t v = S.tok[q + i];
            dst[i] = d2id ? __ldg(d2id + v) : v;
          }
        }
      }
    }
    __syncwarp();
    const uint32_t nlong = min((uint32_t)S.nlong, (uint32_t)kMaxLongPerTile);
    for (uint32_t li = 0; li < nlong; ++li) {
      const int k = S.longk[li];
      const uint64_t start = b0 + S.plist[k];
      const uint32_t c = S.pref[k + 1] - S.pref[k];
      uint32_t* dst = a.out_ids + base + S.pref[k];
      // k_long_pieces flags a piece that merged nothing (tokens = byte LUT).
      const bool unchanged = (__ldcg(a.lpo + start) & kUnchanged) != 0;
      const uint32_t* src = a.lpo + start + 1;
      for (uint32_t i = lane; i < c; i += 32) {
        uint32_t v = unchanged ? s_lut[a.bytes[start + i]] : __ldcg(src + i);
        dst[i] = d2id ? __ldg(d2id + v) : v;
      }
    }

    // Row offsets for rows starting in this tile (the last tile also owns rows
    // starting exactly at the end of the input, including offsets[n_rows]).
    const uint64_t s0 = a.tile_first[tile], s1 = a.tile_first[tile + 1];
    for (uint64_t s = s0 + lane; s < s1 && s <= a.n_rows; s += 32) {
      const int o = static_cast<int>(a.offsets[s] - b0);
      int lo = 0, hi = npieces;  // first piece with plist >= o
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (S.plist[mid] < o) lo = mid + 1; else hi = mid;
      }
      a.out_offsets[s] = base + S.pref[lo];
    }
    __syncwarp();
  }
}

}  // namespace

LaunchPlan plan_launch(int device) {
  LaunchPlan p;
  cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, device);
  const size_t dyn = sizeof(WarpSmem) * kWarpsPerCta;
  cudaFuncSetAttribute(k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, int(dyn));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_encode, kWarpsPerCta * 32, dyn);
  p.main_grid = p.sm_count * (per_sm > 0 ? per_sm : 1);
  int pre_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pre_sm, k_prepass, kWarpsPerCta * 32, 0);
  p.prepass_grid = p.sm_count * (pre_sm > 0 ? pre_sm : 1);
  int lp_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&lp_sm, k_long_pieces<kLpThreads>, kLpThreads, 0);
  p.lp_grid = p.sm_count * (lp_sm > 0 ? lp_sm : 1);
  return p;
}

int launch_encode(const EncodeArgs& a, const DevTable& t, const LaunchPlan& p, cudaStream_t stream,
                  cudaEvent_t* ev) {
  int launched = 0;
  if (ev) cudaEventRecord(ev[0], stream);
  {
    unsigned threads = 256;
    unsigned blocks = unsigned((a.n_rows + 1 + threads - 1) / threads);
    k_tile_first<<<blocks, threads, 0, stream>>>(a);
    ++launched;
  }
  if (ev) cudaEventRecord(ev[1], stream);
  k_prepass<<<p.prepass_grid, kWarpsPerCta * 32, 0, stream>>>(a, t);
  ++launched;
  if (ev) cudaEventRecord(ev[2], stream);
  k_long_pieces<kLpThreads><<<p.lp_grid, kLpThreads, 0, stream>>>(a, t);
  ++launched;
  if (ev) cudaEventRecord(ev[3], stream);
  const size_t dyn = sizeof(WarpSmem) * kWarpsPerCta;
  k_encode<<<p.main_grid, kWarpsPerCta * 32, dyn, stream>>>(a, t);
  ++launched;
  if (ev) cudaEventRecord(ev[4], stream);
  return launched;
}

int launch_block_bpe(const EncodeArgs& a, const DevTable& t, const LaunchPlan& p,
                     cudaStream_t stream) {
  (void)p;
  k_long_pieces<kLpThreads><<<1, kLpThreads, 0, stream>>>(a, t);
  return 1;
}

}  // namespace bbpe
