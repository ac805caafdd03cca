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
//   k_pieces      : warp-per-tile piece split + lane-per-piece pass loops ->
//                   tokens staged per tile (no ordering wait)
//   k_long_pieces : CTA-per-piece pass loop over the long pieces k_pieces found
//                   (the paper's block engine; every row under BBPE_ENGINE_BLOCK)
//   k_gather      : decoupled look-back over tile groups -> CSR ids + row offsets
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
__device__ __forceinline__ uint32_t probe32(const DevTable& T, uint32_t l, uint32_t r) {
  const uint32_t key = (l << 16) | r;
  uint64_t b = mix32(key) & T.bucket_mask;
  for (;;) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.slots + b * kBucketSlots);
    const ulonglong2 s01 = __ldg(p), s23 = __ldg(p + 1);
    const uint64_t s[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (s[j] == kEmptySlot) return kNoRank;
      if (uint32_t(s[j] >> 32) == key) return uint32_t(s[j]);
    }
    b = (b + 1) & T.bucket_mask;
  }
}

__device__ __forceinline__ uint32_t probe(const DevTable& T, uint32_t l, uint32_t r) {
  if (T.key32) return probe32(T, l, r);
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
// Per-warp window over [b0-4, b0+kWin+4): bytes, row starts, hard boundaries.
// Bytes are copied as aligned words: wb[q + 4] is the byte at b0 + q.
constexpr int kWinWordsB = (kWin + 8 + 15) / 16 * 4;  // u32 words of bytes
struct Window {
  uint32_t wbw[kWinWordsB];  // window bytes (as words)
  uint32_t sb[kWords];       // row-start bits
  uint32_t bd[kWords];       // piece-boundary bits
  __device__ __forceinline__ uint32_t byte(int q) const {  // byte at b0 + q, q >= -4
    return reinterpret_cast<const uint8_t*>(wbw)[q + 4];
  }
  __device__ __forceinline__ const uint8_t* bytes() const {
    return reinterpret_cast<const uint8_t*>(wbw);
  }
};

// Loads the window and computes boundaries; returns (lane 0's view of) the
// first invalid byte position found in [b0, b0 + tlen), or ~0.
__device__ void load_window(Window& w, const EncodeArgs& a, const uint32_t* junc, const uint32_t* lut,
                            uint64_t tile, int lane, int tlen) {
  const uint64_t b0 = tile * kTile;
  const uint64_t wbase = b0 >= 4 ? b0 - 4 : 0;
  const int wofs = b0 >= 4 ? 0 : 1;  // tile 0: word 0 of the window is before the input
#pragma unroll 1
  for (int i = lane; i < kWinWordsB; i += 32) {
    const int gi = i - wofs;
    uint32_t v = 0;
    if (gi >= 0) {
      const uint64_t pos = wbase + 4ull * gi;
      if (pos + 4 <= a.total) {
        v = __ldg(reinterpret_cast<const uint32_t*>(a.bytes + pos));
      } else {
        for (int k = 0; k < 4; ++k)
          if (pos + k < a.total) v |= uint32_t(a.bytes[pos + k]) << (8 * k);
      }
    }
    w.wbw[i] = v;
  }
  for (int i = lane; i < kWords; i += 32) w.sb[i] = 0;
  __syncwarp();
  // Row starts inside the window.
  const uint64_t s0 = a.tile_first[tile];
  for (uint64_t s = s0;; s += 32) {
    const uint64_t my = s + lane;
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
  // Boundaries, and the invalid-byte check (pretokenize.hpp:64-67).
  uint32_t badw = 0xFFFFFFFFu;
#pragma unroll 1
  for (int wd = 0; wd < kWords; ++wd) {
    const int q = wd * 32 + lane;
    const uint64_t abs = b0 + q;
    bool b = true;
    if (q < kWin && abs < a.total) {
      const uint32_t cur = w.byte(q);
      b = (w.sb[wd] >> lane) & 1u;
      if (!b) b = !is_junction(junc, w.byte(q - 1), cur);
      if (q < tlen && lut[cur] == kInvalidToken && badw == 0xFFFFFFFFu) badw = uint32_t(q);
    }
    const unsigned m = __ballot_sync(kFull, b);
    if (lane == 0) w.bd[wd] = m;
  }
  const uint32_t bad = __reduce_min_sync(kFull, badw);
  if (bad != 0xFFFFFFFFu && lane == 0)
    atomicMin(reinterpret_cast<unsigned long long*>(&a.err[ERR_BAD_BYTE_POS]),
              (unsigned long long)(b0 + bad));
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
    const uint32_t count = min((uint64_t)a.counters[CNT_LREC], (uint64_t)a.lp_cap);
    if (idx >= count) return;
    const LongRec P = a.lrec[idx];
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
    if (tid == 0) {
      O[0] = static_cast<uint32_t>(n) | ((n == len && !a.tokens_input) ? kUnchanged : 0u);
      a.lrec[idx].count = static_cast<uint32_t>(n);
    }
    if (n < len || a.tokens_input)
      for (int32_t i = tid; i < n; i += NT) O[1 + i] = tok_of(X[i]);
  }
}

// ---------------------------------------------------------------------------
// k_pieces: warp-per-tile merge of all short pieces starting in the tile.
// Per tile: window -> piece list -> initial tokens -> warp-parallel, batched
// initial pair probes -> sub-warp "blocks" run the reference pass loop, one
// piece per group of W lanes (one token per lane) -> tokens staged per tile
// (no ordering wait; k_gather assembles the CSR afterwards).
//
// This is the paper's one-block-per-string engine scaled to the piece: a
// pass is a W-lane shuffle min-reduction, a ballot of the pairs at the
// minimum (left-greedy over runs), a ballot/popc compaction, and re-probes
// of only the pairs that touch a merged token.
template <typename Tk>
struct Marks {
  static constexpr uint32_t kNone = Tk(~Tk(0));  // no rank / uncovered position
};

constexpr int kMemoDone = 0x40;  // plen flag: piece resolved by the memo

template <typename Tk>
struct PieceSmem {
  Window w;
  uint16_t plist[kTile];      // piece starts (window-relative), in order
  uint8_t plen[kTile];        // piece length, 0xFF = long (> kLmax)
  uint16_t clist[kTile];      // pieces that need merge passes
  uint16_t cnt[kTile + 1];    // short tokens per piece -> exclusive prefix
  Tk tok[kWin + 1];
  Tk rnk[kWin + 1];
  uint64_t llen[kTile / (kLmax + 1) + 2];    // byte length of each long piece, in order
  uint16_t lk[kTile / (kLmax + 1) + 2];      // their piece indices
};

// Batched probe: issue the bucket loads, resolve later. K32: narrow tables
// (ids < 2^16) with 32-bit keys, slot = key32 << 32 | rank.
struct ProbeReq {
  uint64_t key, b;
  ulonglong2 s01, s23;
};
template <bool K32>
__device__ __forceinline__ void probe_issue(ProbeReq& q, const DevTable& T, uint32_t l, uint32_t r) {
  if (K32) {
    const uint32_t k32 = (l << 16) | r;
    q.key = k32;
    q.b = mix32(k32) & T.bucket_mask;
  } else {
    q.key = (uint64_t(l) << T.id_bits) | uint64_t(r);
    q.b = dmix64(q.key) & T.bucket_mask;
  }
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.slots + q.b * kBucketSlots);
  q.s01 = __ldg(p);
  q.s23 = __ldg(p + 1);
}

// Bucket full without a hit: keep probing linearly (rare at load <= 0.5).
template <bool K32>
__device__ __noinline__ uint32_t probe_overflow(const DevTable& T, uint64_t key, uint64_t b) {
  const uint64_t rmask = (1ull << T.rank_bits) - 1;
  for (;;) {
    b = (b + 1) & T.bucket_mask;
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.slots + b * kBucketSlots);
    const ulonglong2 x = __ldg(p), y = __ldg(p + 1);
    const uint64_t t[4] = {x.x, x.y, y.x, y.y};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (t[j] == kEmptySlot) return kNoRank;
      if (K32 ? (uint32_t(t[j] >> 32) == uint32_t(key)) : ((t[j] >> T.rank_bits) == key))
        return K32 ? uint32_t(t[j]) : static_cast<uint32_t>(t[j] & rmask);
    }
  }
}

template <bool K32>
__device__ __forceinline__ uint32_t probe_resolve(const ProbeReq& q, const DevTable& T) {
  const uint64_t s[4] = {q.s01.x, q.s01.y, q.s23.x, q.s23.y};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (s[j] == kEmptySlot) return kNoRank;
    if (K32) {
      if (uint32_t(s[j] >> 32) == uint32_t(q.key)) return uint32_t(s[j]);
    } else {
      if ((s[j] >> T.rank_bits) == q.key) return static_cast<uint32_t>(s[j] & ((1ull << T.rank_bits) - 1));
    }
  }
  return probe_overflow<K32>(T, q.key, q.b);
}

template <typename Tk>
__device__ __forceinline__ uint32_t tk_rank(uint32_t r) {
  return r == kNoRank ? Marks<Tk>::kNone : r;
}

// One lane, one pass of the reference loop over a piece of n <= kLmax tokens
// at tok[0..n) / rnk[0..n-1) (block_engine.hpp:286-307): min over cached
// ranks, sweep-compact in place (a pair at the minimum merges unless its left
// token was just consumed -- exactly flags[i+1] = (ranks[i] == m && !flags[i])),
// then re-probe only the pairs touching a merged token, two in flight.
// Returns the new length, or -1 when no pair is mergeable.
template <typename Tk>
__device__ __forceinline__ int lane_pass(const DevTable& T, Tk* tok, Tk* rnk, int n) {
  constexpr bool K32 = sizeof(Tk) == 2;  // narrow tables use 32-bit pair keys
  constexpr uint32_t NONE = Marks<Tk>::kNone, PROBE = Marks<Tk>::kNone - 1;
  uint32_t m = NONE;
  for (int i = 0; i < n - 1; ++i) m = min(m, uint32_t(rnk[i]));
  if (m == NONE) return -1;
  const Tk M = Tk(__ldg(T.r2m + m));
  int j = 0, i = 0;
  while (i < n) {
    const uint32_t ri = (i < n - 1) ? uint32_t(rnk[i]) : NONE;
    if (ri == m) {
      tok[j] = M;
      rnk[j] = Tk(PROBE);
      if (j > 0) rnk[j - 1] = Tk(PROBE);
      i += 2;
    } else {
      tok[j] = tok[i];
      rnk[j] = Tk(ri);
      i += 1;
    }
    ++j;
  }
  int k = 0;
  for (;;) {
    while (k < j - 1 && uint32_t(rnk[k]) != PROBE) ++k;
    if (k >= j - 1) break;
    int k2 = k + 1;
    while (k2 < j - 1 && uint32_t(rnk[k2]) != PROBE) ++k2;
    ProbeReq pa, pb;
    probe_issue<K32>(pa, T, tok[k], tok[k + 1]);
    const bool two = k2 < j - 1;
    if (two) probe_issue<K32>(pb, T, tok[k2], tok[k2 + 1]);
    rnk[k] = Tk(tk_rank<Tk>(probe_resolve<K32>(pa, T)));
    if (two) rnk[k2] = Tk(tk_rank<Tk>(probe_resolve<K32>(pb, T)));
    k = two ? k2 + 1 : j;
  }
  return j;
}

// Whole-piece memo lookup (exact: the entry holds this engine's own encoding
// of the same bytes, computed from the table alone at upload time).
__device__ __forceinline__ int memo_match(const ulonglong2 lo, const ulonglong2 hi, const uint32_t* w,
                                          int len, uint32_t& r0, uint32_t& r1, uint32_t& nres) {
  const uint32_t meta = uint32_t(hi.x >> 32), elen = meta & 0xFF;
  if (elen == 0) return 0;  // empty slot: miss
  if (elen == uint32_t(len) && uint32_t(lo.x) == w[0] && uint32_t(lo.x >> 32) == w[1] &&
      uint32_t(lo.y) == w[2] && uint32_t(lo.y >> 32) == w[3] && uint32_t(hi.x) == w[4]) {
    nres = (meta >> 8) & 0xFF;
    r0 = uint32_t(hi.y);
    r1 = uint32_t(hi.y >> 32);
    return 1;  // hit
  }
  return -1;  // occupied by another piece: keep probing
}

__device__ __noinline__ bool memo_overflow(const DevTable& T, const uint32_t* w, int len, uint64_t b,
                                           uint32_t& r0, uint32_t& r1, uint32_t& nres) {
  for (;;) {
    b = (b + 1) & T.memo_mask;
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.memo + b);
    const int m = memo_match(__ldg(p), __ldg(p + 1), w, len, r0, r1, nres);
    if (m >= 0) return m == 1;
  }
}

__device__ __forceinline__ bool memo_lookup(const DevTable& T, const uint32_t* ww, int q, int len,
                                            uint32_t& r0, uint32_t& r1, uint32_t& nres) {
  const int start = q + 4, a = start >> 2, sh = (start & 3) * 8;
  uint32_t x[6], w[5];
#pragma unroll
  for (int i = 0; i < 6; ++i) x[i] = ww[a + i];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    uint32_t v = __funnelshift_r(x[i], x[i + 1], sh);
    const int nb = len - 4 * i;
    v &= nb >= 4 ? 0xFFFFFFFFu : (nb <= 0 ? 0u : ((1u << (8 * nb)) - 1u));
    w[i] = v;
  }
  const uint64_t b = memo_hash(w, uint32_t(len)) & T.memo_mask;
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.memo + b);
  const int m = memo_match(__ldg(p), __ldg(p + 1), w, len, r0, r1, nres);
  if (m >= 0) return m == 1;
  return memo_overflow(T, w, len, b, r0, r1, nres);
}

// Length of a long piece starting at abs (warp-cooperative, rare path).
__device__ __noinline__ uint64_t long_piece_length(const EncodeArgs& a, const uint32_t* junc,
                                                   uint64_t abs, int lane) {
  uint64_t row_end = 0;
  if (lane == 0) {
    uint64_t lo = 0, hi = a.n_rows;  // max s with offsets[s] <= abs
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) >> 1;
      if (a.offsets[mid] <= abs) lo = mid; else hi = mid - 1;
    }
    row_end = a.offsets[lo + 1];
  }
  row_end = __shfl_sync(kFull, row_end, 0);
  for (uint64_t x = abs + kLmax + 1; x < row_end; x += 32) {
    const uint64_t y = x + lane;
    const bool bnd = y < row_end && !is_junction(junc, a.bytes[y - 1], a.bytes[y]);
    const unsigned bm = __ballot_sync(kFull, bnd);
    if (bm) return x + __ffs(bm) - 1 - abs;
  }
  return row_end - abs;
}

#ifndef BBPE_PIECES_MINB
#define BBPE_PIECES_MINB 3
#endif
template <typename Tk>
__global__ void __launch_bounds__(kWarpsPerCta * 32, BBPE_PIECES_MINB) k_pieces(EncodeArgs a, DevTable T) {
  constexpr bool K32 = sizeof(Tk) == 2;
  __shared__ uint32_t s_lut[256];
  __shared__ uint32_t s_junc[2048];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s_junc[i] = T.junction[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  PieceSmem<Tk>& S = reinterpret_cast<PieceSmem<Tk>*>(s_dyn)[wid];
  const uint32_t* d2id = T.d2id;

  for (;;) {
    uint64_t tile = 0;
    if (lane == 0) tile = atomicAdd(&a.counters[CNT_TILE_TICKET], 1u);
    tile = __shfl_sync(kFull, tile, 0);
    if (tile >= a.num_tiles) return;
    const uint64_t b0 = tile * kTile;
    const uint64_t s0 = a.tile_first[tile], s1 = a.tile_first[tile + 1];

    const int tlen = int(min((uint64_t)kTile, (uint64_t)(a.total - b0)));
    load_window(S.w, a, s_junc, s_lut, tile, lane, tlen);

    // (1) Piece list with lengths (distance to the next piece start; the
    // last piece of the tile searches the boundary bits past the tile).
    int npieces = 0;
#pragma unroll 1
    for (int wd = 0; wd * 32 < tlen; ++wd) {
      const int q = wd * 32 + lane;
      const bool st = q < tlen && ((S.w.bd[wd] >> lane) & 1u);
      const unsigned m = __ballot_sync(kFull, st);
      if (st) S.plist[npieces + __popc(m & lanemask_lt(lane))] = static_cast<uint16_t>(q);
      npieces += __popc(m);
    }
    __syncwarp();
    for (int k = lane; k < npieces; k += 32) {
      const int q = S.plist[k];
      const int len = (k + 1 < npieces) ? S.plist[k + 1] - q : next_boundary(S.w.bd, q, kLmax) - q;
      S.plen[k] = len > kLmax ? 0xFF : static_cast<uint8_t>(len);
    }
    __syncwarp();

    // (2) Piece memo: a piece equal to a vocabulary token's bytes takes its
    // precomputed encoding (1-2 tokens, parked in rnk[q..] until staging).
    // Everything else of 2..kLmax bytes goes on the merge list.
    int nmerge = 0;
    for (int k0 = 0; k0 < npieces; k0 += 32) {
      const int k = k0 + lane;
      int len = k < npieces ? S.plen[k] : 0;
      bool merge = false;
      if (k < npieces) {
        if (len == 0xFF) {
          S.cnt[k] = 0;
        } else if (len < 2) {
          S.cnt[k] = static_cast<uint16_t>(len);
          S.tok[S.plist[k]] = Tk(s_lut[S.w.byte(S.plist[k])]);
        } else {
          merge = true;
          const int q = S.plist[k];
          uint32_t r0, r1, nres;
          if (a.use_memo && len <= kMemoMaxLen && memo_lookup(T, S.w.wbw, q, len, r0, r1, nres)) {
            S.plen[k] = static_cast<uint8_t>(len | kMemoDone);
            S.cnt[k] = static_cast<uint16_t>(nres);
            S.rnk[q] = Tk(r0);
            S.rnk[q + 1] = Tk(r1);
            merge = false;
          }
        }
      }
      const unsigned mm = __ballot_sync(kFull, merge);
      if (merge) S.clist[nmerge + __popc(mm & lanemask_lt(lane))] = static_cast<uint16_t>(k);
      nmerge += __popc(mm);
    }
    __syncwarp();

    if (nmerge) {
      // (3) Lane-per-piece pass loops over the merge list (pieces refill
      // lanes as they finish). A new piece gets its initial tokens and pair
      // ranks (two probes in flight), then one pass per loop iteration.
      int my_n = 0, my_q = 0, my_k = 0, next = 0;
      for (;;) {
        const bool idle = my_n == 0;
        const unsigned im = __ballot_sync(kFull, idle);
        if (idle) {
          const int i = next + __popc(im & lanemask_lt(lane));
          if (i < nmerge) {
            my_k = S.clist[i];
            my_q = S.plist[my_k];
            my_n = S.plen[my_k];
            Tk* tk = S.tok + my_q;
            Tk* rk = S.rnk + my_q;
            for (int j = 0; j < my_n; ++j) tk[j] = Tk(s_lut[S.w.byte(my_q + j)]);
            for (int j = 0; j < my_n - 1; j += 2) {
              ProbeReq p0, p1;
              probe_issue<K32>(p0, T, tk[j], tk[j + 1]);
              const bool two = j + 2 < my_n;
              if (two) probe_issue<K32>(p1, T, tk[j + 1], tk[j + 2]);
              rk[j] = Tk(tk_rank<Tk>(probe_resolve<K32>(p0, T)));
              if (two) rk[j + 1] = Tk(tk_rank<Tk>(probe_resolve<K32>(p1, T)));
            }
          }
        }
        next += __popc(im);
        const bool active = my_n >= 2;
        if (!__any_sync(kFull, active) && next >= nmerge) break;
        if (active) {
          const int r = lane_pass<Tk>(T, S.tok + my_q, S.rnk + my_q, my_n);
          if (r < 2) {
            S.cnt[my_k] = static_cast<uint16_t>(r < 0 ? my_n : r);
            my_n = 0;
          } else {
            my_n = r;
          }
        }
      }
      __syncwarp();
    }

    // (5) Exclusive scan of short counts; long pieces listed in order.
    uint32_t run = 0, nlong = 0;
    for (int k0 = 0; k0 < npieces; k0 += 32) {
      const int k = k0 + lane;
      const uint32_t c = k < npieces ? S.cnt[k] : 0;
      const uint32_t inc = warp_incl_sum(c, lane);
      const bool lg = k < npieces && S.plen[k] == 0xFF;
      const unsigned lm = __ballot_sync(kFull, lg);
      if (lg) S.lk[nlong + __popc(lm & lanemask_lt(lane))] = static_cast<uint16_t>(k);
      nlong += __popc(lm);
      __syncwarp();
      if (k < npieces) S.cnt[k] = static_cast<uint16_t>(run + inc - c);
      run += __shfl_sync(kFull, inc, 31);
    }
    if (lane == 0) S.cnt[npieces] = static_cast<uint16_t>(run);
    __syncwarp();
    // Long pieces (rare): full length = distance to the next hard boundary or
    // the end of the row; k_long_pieces merges them after this kernel.
    for (uint32_t li = 0; li < nlong; ++li) {
      const uint64_t len = long_piece_length(a, s_junc, b0 + S.plist[S.lk[li]], lane);
      if (lane == 0) S.llen[li] = len;
    }
    __syncwarp();

    // (6) Stage short tokens in piece order (final ids).
    uint32_t* stage = a.staging + tile * kStage;
    for (int k = lane; k < npieces; k += 32) {
      const int pl = S.plen[k];
      if (pl == 0xFF) continue;
      const int q = S.plist[k];
      const uint32_t c = S.cnt[k + 1] - S.cnt[k];
      uint32_t* dst = stage + S.cnt[k];
      const Tk* src = (pl != 0xFF && (pl & kMemoDone)) ? S.rnk + q : S.tok + q;
      for (uint32_t i = 0; i < c; ++i) {
        const uint32_t v = src[i];
        dst[i] = d2id ? __ldg(d2id + v) : v;
      }
    }
    // (7) Long-piece records, tile short total.
    if (lane == 0) {
      uint64_t rec = 0;
      if (nlong) {
        const uint32_t first = atomicAdd(&a.counters[CNT_LREC], nlong);
        for (uint32_t li = 0; li < nlong && first + li < a.lp_cap; ++li) {
          const int k = S.lk[li];
          a.lrec[first + li] = LongRec{b0 + S.plist[k], S.llen[li], 0, S.cnt[k], 0u};
        }
        rec = (uint64_t(first) << 24) | nlong;
      }
      a.tile_lrec[tile] = rec;
      a.tile_count[tile] = run;
    }
    // (8) Row offsets relative to the tile: short tokens before the row in
    // the low 40 bits, long pieces before it above; k_gather resolves them.
    for (uint64_t s = s0 + lane; s < s1 && s <= a.n_rows; s += 32) {
      const int o = static_cast<int>(a.offsets[s] - b0);
      int lo = 0, hi = npieces;  // first piece with plist >= o
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (S.plist[mid] < o) lo = mid + 1; else hi = mid;
      }
      uint64_t lb = 0;
      while (lb < nlong && S.lk[lb] < lo) ++lb;
      a.out_offsets[s] = uint64_t(S.cnt[lo]) | (lb << 40);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// k_block_rows (BBPE_ENGINE_BLOCK): every non-empty row is one long piece for
// k_long_pieces -- the paper's one-block-per-string engine. Warp per tile:
// invalid-byte check, records in row order, row offsets relative to the tile.
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_block_rows(EncodeArgs a, DevTable T) {
  __shared__ uint32_t s_lut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = uint64_t(gridDim.x) * kWarpsPerCta;
  for (uint64_t tile = blockIdx.x * uint64_t(kWarpsPerCta) + (threadIdx.x >> 5); tile < a.num_tiles;
       tile += nwarps) {
    const uint64_t b0 = tile * kTile;
    const uint64_t s0 = a.tile_first[tile], s1 = a.tile_first[tile + 1];
      // Every non-empty row is one long piece for k_long_pieces; the tile's
      // output is its rows' results in order.
      const int tl = int(min((uint64_t)kTile, (uint64_t)(a.total - b0)));
      for (int q0 = 0; q0 < tl; q0 += 32) {  // invalid bytes (pretokenize.hpp:64-67)
        const int q = q0 + lane;
        const bool bad = q < tl && s_lut[a.bytes[b0 + q]] == kInvalidToken;
        const unsigned bm = __ballot_sync(kFull, bad);
        if (bm && lane == 0)
          atomicMin(reinterpret_cast<unsigned long long*>(&a.err[ERR_BAD_BYTE_POS]),
                    (unsigned long long)(b0 + q0 + __ffs(bm) - 1));
      }
      uint32_t ne = 0;
      for (uint64_t s = s0 + lane; s < s1 && s < a.n_rows; s += 32)
        ne += a.offsets[s + 1] > a.offsets[s] ? 1u : 0u;
      ne = __reduce_add_sync(kFull, ne);
      uint64_t first = 0;
      if (lane == 0 && ne) first = atomicAdd(&a.counters[CNT_LREC], ne);
      first = __shfl_sync(kFull, first, 0);
      uint32_t ri = 0;
      for (uint64_t sb = s0; sb < s1 && sb <= a.n_rows; sb += 32) {
        const uint64_t s = sb + lane;
        bool ne_row = false;
        uint64_t o = 0, e = 0;
        if (s < s1 && s < a.n_rows) {
          o = a.offsets[s];
          e = a.offsets[s + 1];
          ne_row = e > o;
        }
        const unsigned nm = __ballot_sync(kFull, ne_row);
        const uint32_t before = ri + __popc(nm & lanemask_lt(lane));
        if (s < s1 && s <= a.n_rows) a.out_offsets[s] = uint64_t(before) << 40;
        if (ne_row && first + before < a.lp_cap)
          a.lrec[first + before] = LongRec{o, e - o, s, 0u, 0u};
        ri += __popc(nm);
      }
      if (lane == 0) {
        a.tile_lrec[tile] = ne ? ((first << 24) | ne) : 0;
        a.tile_count[tile] = 0;
      }
        }
}

// ---------------------------------------------------------------------------
// k_tile_scan: exclusive scan of tile token totals (short + long pieces) into
// tile_base[0..num_tiles]. One CTA per kScanTiles tiles, CTAs chained by a
// decoupled look-back (a few hundred CTAs even for GB inputs).
constexpr int kScanThreads = 512;
constexpr int kScanPer = 8;
constexpr int kScanTiles = kScanThreads * kScanPer;
static_assert(kScanTiles == kScanTilesPerCta, "scan geometry");

__global__ void __launch_bounds__(kScanThreads) k_tile_scan(EncodeArgs a) {
  __shared__ uint64_t s_warp[kScanThreads / 32];
  __shared__ uint64_t s_base;
  __shared__ uint32_t s_cta;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_cta = atomicAdd(&a.counters[CNT_GROUP_TICKET], 1u);
  __syncthreads();
  const uint64_t cta = s_cta;
  const uint64_t t0 = cta * kScanTiles + uint64_t(tid) * kScanPer;
  uint64_t v[kScanPer];
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    const uint64_t t = t0 + i;
    uint64_t c = 0;
    if (t < a.num_tiles) {
      c = __ldcg(a.tile_count + t);
      const uint64_t rec = __ldcg(a.tile_lrec + t);
      if (rec) {
        const uint64_t first = rec >> 24;
        const uint32_t nl = uint32_t(rec & 0xFFFFFF);
        for (uint32_t li = 0; li < nl; ++li) c += __ldcg(&a.lrec[first + li].count);
      }
    }
    v[i] = c;
    sum += c;
  }
  // Block exclusive scan of per-thread sums.
  uint64_t inc = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t u = __shfl_up_sync(kFull, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint64_t x = lane < kScanThreads / 32 ? s_warp[lane] : 0;
    uint64_t xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t u = __shfl_up_sync(kFull, xi, d);
      if (lane >= d) xi += u;
    }
    if (lane < kScanThreads / 32) s_warp[lane] = xi - x;
    const uint64_t agg = __shfl_sync(kFull, xi, 31);
    // Look-back across CTAs (warp 0).
    uint64_t excl = 0;
    if (cta == 0) {
      if (lane == 0) st_release(&a.status[0], kFlagPrefix | agg);
    } else {
      if (lane == 0) st_release(&a.status[cta], kFlagAgg | agg);
      int64_t look = int64_t(cta) - 1;
      for (;;) {
        const int64_t idx = look - lane;
        uint64_t sv = kFlagPrefix;
        unsigned pm, xm;
        for (;;) {
          if (idx >= 0) sv = ld_acquire(&a.status[idx]);
          pm = __ballot_sync(kFull, (sv >> 62) == 2);
          xm = __ballot_sync(kFull, (sv >> 62) == 0);
          const unsigned first_p = pm ? __ffs(pm) : 33, first_x = xm ? __ffs(xm) : 33;
          if (first_x > first_p) break;
          __nanosleep(64);
        }
        const int first_p = pm ? __ffs(pm) - 1 : 31;
        excl += warp_sum64(lane <= first_p ? (sv & kValMask) : 0);
        if (pm) break;
        look -= 32;
      }
      if (lane == 0) st_release(&a.status[cta], kFlagPrefix | (excl + agg));
    }
    if (lane == 0) s_base = excl;
  }
  __syncthreads();
  uint64_t run = s_base + s_warp[wid] + inc - sum;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    const uint64_t t = t0 + i;
    if (t < a.num_tiles) a.tile_base[t] = run;
    if (t == a.num_tiles - 1) a.tile_base[a.num_tiles] = run + v[i];
    run += v[i];
  }
}

// ---------------------------------------------------------------------------
// k_gather: warp per tile, fully parallel. Copies the tile's staged short
// tokens and its long pieces (in piece order) to their final CSR place and
// resolves the row offsets written by k_pieces.
__device__ __forceinline__ void copy_tokens(uint32_t* dst, const uint32_t* src, uint32_t n, int lane) {
  for (uint32_t i = lane; i < n; i += 32) dst[i] = __ldcg(src + i);
}

__global__ void __launch_bounds__(kWarpsPerCta * 32) k_gather(EncodeArgs a, DevTable T) {
  __shared__ uint32_t s_lut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t* d2id = T.d2id;
  const uint64_t nwarps = uint64_t(gridDim.x) * kWarpsPerCta;
  for (uint64_t t = blockIdx.x * uint64_t(kWarpsPerCta) + (threadIdx.x >> 5); t < a.num_tiles; t += nwarps) {
    const uint64_t tbase = __ldcg(a.tile_base + t);
    const uint64_t rec = __ldcg(a.tile_lrec + t);
    const uint32_t nshort = __ldcg(a.tile_count + t);
    const uint32_t* stage = a.staging + t * kStage;
    uint32_t* out = a.out_ids + tbase;
    if (rec == 0) {
      copy_tokens(out, stage, nshort, lane);
    } else {
      const uint64_t first = rec >> 24;
      const uint32_t nl = uint32_t(rec & 0xFFFFFF);
      uint64_t pos = 0;
      uint32_t sp = 0;
      for (uint32_t li = 0; li < nl; ++li) {
        const LongRec lr = a.lrec[first + li];
        copy_tokens(out + pos, stage + sp, lr.spref - sp, lane);
        pos += lr.spref - sp;
        sp = lr.spref;
        const bool unchanged = (__ldcg(a.lpo + lr.start) & kUnchanged) != 0;
        for (uint32_t i = lane; i < lr.count; i += 32) {
          const uint32_t v = unchanged ? s_lut[a.bytes[lr.start + i]] : __ldcg(a.lpo + lr.start + 1 + i);
          out[pos + i] = d2id ? __ldg(d2id + v) : v;
        }
        pos += lr.count;
      }
      copy_tokens(out + pos, stage + sp, nshort - sp, lane);
    }
    // Row offsets: short tokens before the row (low 40 bits) plus the first
    // (v >> 40) long pieces of the tile.
    const uint64_t s0 = a.tile_first[t], s1 = a.tile_first[t + 1];
    const uint64_t rb = a.run_base ? *a.run_base : 0;
    for (uint64_t s = s0 + lane; s < s1 && s <= a.n_rows; s += 32) {
      const uint64_t v = __ldcg(a.out_offsets + s);
      const uint32_t lb = uint32_t(v >> 40);
      uint64_t lsum = 0;
      for (uint32_t li = 0; li < lb; ++li) lsum += __ldcg(&a.lrec[(rec >> 24) + li].count);
      a.out_offsets[s] = rb + tbase + (v & ((1ull << 40) - 1)) + lsum;
    }
  }
}

__global__ void k_rebase_input(uint64_t* off, uint64_t n, uint64_t base) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) off[i] -= base;
}
__global__ void k_advance_base(uint64_t* run_base, const uint64_t* wave_total) {
  *run_base += *wave_total;
}
__global__ void k_fill_offsets(uint64_t* out, uint64_t n, const uint64_t* run_base) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = run_base ? *run_base : 0;
}

}  // namespace

void launch_rebase_input(uint64_t* d_off, uint64_t n, uint64_t base, cudaStream_t stream) {
  if (base == 0 || n == 0) return;
  k_rebase_input<<<unsigned((n + 255) / 256), 256, 0, stream>>>(d_off, n, base);
}
void launch_advance_base(uint64_t* run_base, const uint64_t* wave_total, cudaStream_t stream) {
  k_advance_base<<<1, 1, 0, stream>>>(run_base, wave_total);
}
void launch_fill_offsets(uint64_t* d_out_off, uint64_t n, const uint64_t* run_base, cudaStream_t stream) {
  if (n == 0) return;
  k_fill_offsets<<<unsigned((n + 255) / 256), 256, 0, stream>>>(d_out_off, n, run_base);
}

template <typename Tk>
size_t pieces_smem() {
  return sizeof(PieceSmem<Tk>) * kWarpsPerCta;
}

LaunchPlan plan_launch(int device) {
  LaunchPlan p;
  cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, device);
  int per_sm = 0;
  cudaFuncSetAttribute(k_pieces<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(pieces_smem<uint16_t>()));
  cudaFuncSetAttribute(k_pieces<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(pieces_smem<uint32_t>()));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pieces<uint16_t>, kWarpsPerCta * 32,
                                                pieces_smem<uint16_t>());
  p.main_grid = p.sm_count * (per_sm > 0 ? per_sm : 1);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pieces<uint32_t>, kWarpsPerCta * 32,
                                                pieces_smem<uint32_t>());
  p.main_grid_wide = p.sm_count * (per_sm > 0 ? per_sm : 1);
  int lp_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&lp_sm, k_long_pieces<kLpThreads>, kLpThreads, 0);
  p.lp_grid = p.sm_count * (lp_sm > 0 ? lp_sm : 1);
  int g_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_sm, k_gather, kWarpsPerCta * 32, 0);
  p.gather_grid = p.sm_count * (g_sm > 0 ? g_sm : 1);
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
  if (a.engine == BBPE_ENGINE_BLOCK)
    k_block_rows<<<p.gather_grid, kWarpsPerCta * 32, 0, stream>>>(a, t);
  else if (a.narrow)
    k_pieces<uint16_t><<<p.main_grid, kWarpsPerCta * 32, pieces_smem<uint16_t>(), stream>>>(a, t);
  else
    k_pieces<uint32_t><<<p.main_grid_wide, kWarpsPerCta * 32, pieces_smem<uint32_t>(), stream>>>(a, t);
  ++launched;
  if (ev) cudaEventRecord(ev[2], stream);
  k_long_pieces<kLpThreads><<<p.lp_grid, kLpThreads, 0, stream>>>(a, t);
  ++launched;
  if (ev) cudaEventRecord(ev[3], stream);
  k_tile_scan<<<unsigned((a.num_tiles + kScanTiles - 1) / kScanTiles), kScanThreads, 0, stream>>>(a);
  ++launched;
  if (ev) cudaEventRecord(ev[4], stream);
  k_gather<<<p.gather_grid, kWarpsPerCta * 32, 0, stream>>>(a, t);
  ++launched;
  if (ev) cudaEventRecord(ev[5], stream);
  return launched;
}

int launch_block_bpe(const EncodeArgs& a, const DevTable& t, const LaunchPlan& p,
                     cudaStream_t stream) {
  (void)p;
  k_long_pieces<kLpThreads><<<1, kLpThreads, 0, stream>>>(a, t);
  return 1;
}

}  // namespace bbpe
