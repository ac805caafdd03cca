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
constexpr int kWords = (kWin + 127) / 128 * 4;  // boundary words, whole 128-position chunks
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
constexpr int kWinWordsB = kWords * 8 + 4;  // u32 words of bytes (all boundary positions + 4)
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
                            uint64_t tile, int lane, int tlen, bool full_lut) {
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
  // Boundaries: lane handles 4 consecutive positions per 128-position chunk
  // (one word of bytes + the byte before), 8 lanes OR their nibbles into a
  // boundary word. Plus the invalid-byte check (pretokenize.hpp:64-67) when
  // the table lacks a token for some byte value.
  const int64_t limit = min((int64_t)kWin, (int64_t)(a.total - b0));  // positions past this are boundaries
  uint32_t badw = 0xFFFFFFFFu;
#pragma unroll 1
  for (int c = 0; c < kWords / 4; ++c) {
    const int q0 = 128 * c + 4 * lane;
    const uint32_t cur = w.wbw[32 * c + lane + 1];
    const uint32_t prv = w.wbw[32 * c + lane] >> 24;
    uint32_t nib = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t pb = j == 0 ? prv : (cur >> (8 * (j - 1))) & 0xFFu;
      const uint32_t cb = (cur >> (8 * j)) & 0xFFu;
      if (!is_junction(junc, pb, cb)) nib |= 1u << j;
      if (!full_lut && q0 + j < tlen && lut[cb] == kInvalidToken && badw == 0xFFFFFFFFu) badw = uint32_t(q0 + j);
    }
    nib |= (w.sb[4 * c + (lane >> 3)] >> (4 * (lane & 7))) & 0xFu;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (q0 + j >= limit) nib |= 1u << j;
    uint32_t v = nib << (4 * (lane & 7));
    v |= __shfl_xor_sync(kFull, v, 1);
    v |= __shfl_xor_sync(kFull, v, 2);
    v |= __shfl_xor_sync(kFull, v, 4);
    if ((lane & 7) == 0) w.bd[4 * c + (lane >> 3)] = v;
  }
  if (!full_lut) {
    const uint32_t bad = __reduce_min_sync(kFull, badw);
    if (bad != 0xFFFFFFFFu && lane == 0)
      atomicMin(reinterpret_cast<unsigned long long*>(&a.err[ERR_BAD_BYTE_POS]),
                (unsigned long long)(b0 + bad));
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
    const uint32_t count = min((uint64_t)a.counters[CNT_LONG], (uint64_t)a.long_cap);
    if (idx >= count) return;
    const uint32_t ridx = a.long_idx[idx];
    const LongRec P = a.lrec[ridx];
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
      a.lrec[ridx].count = static_cast<uint32_t>(n);
    }
    if (n < len || a.tokens_input)
      for (int32_t i = tid; i < n; i += NT) O[1 + i] = tok_of(X[i]);
  }
}

// ---------------------------------------------------------------------------
// Marks in the per-lane working arrays of k_merge (16- or 32-bit).
template <typename Tk>
struct Marks {
  static constexpr uint32_t kNone = Tk(~Tk(0));  // no rank / uncovered position
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

struct PieceSmem {
  Window w;
  uint16_t plist[kTile];      // piece starts (window-relative), in order
  uint8_t plen[kTile];        // piece length, 0xFF = long (> kLmax)
  uint16_t cnt[kTile + 1];    // staging slot of each piece (exclusive prefix)
  uint16_t dk[kTile];         // deferred pieces (merge or long), in order
  uint64_t llen[kTile / (kLmax + 1) + 2];
};

#ifndef BBPE_PIECES_MINB
#define BBPE_PIECES_MINB 4
#endif
// k_pieces: warp per tile. Window -> hard boundaries -> piece list; each piece
// is resolved in place when it is a single byte or a piece-memo hit, and its
// tokens go to the tile's staging slots right away; other pieces are deferred
// (records, in piece order): 2..kLmax-byte pieces to k_merge (slots reserved),
// longer ones to k_long_pieces.
__global__ void __launch_bounds__(kWarpsPerCta * 32, BBPE_PIECES_MINB) k_pieces(EncodeArgs a, DevTable T) {
  __shared__ uint32_t s_lut[256];
  __shared__ uint32_t s_junc[2048];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s_junc[i] = T.junction[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  PieceSmem& S = reinterpret_cast<PieceSmem*>(s_dyn)[wid];
  const uint32_t* d2id = T.d2id;

  for (;;) {
    uint64_t tile = 0;
    if (lane == 0) tile = atomicAdd(&a.counters[CNT_TILE_TICKET], 1u);
    tile = __shfl_sync(kFull, tile, 0);
    if (tile >= a.num_tiles) return;
    const uint64_t b0 = tile * kTile;
    const uint64_t s0 = a.tile_first[tile], s1 = a.tile_first[tile + 1];
    const int tlen = int(min((uint64_t)kTile, (uint64_t)(a.total - b0)));
    load_window(S.w, a, s_junc, s_lut, tile, lane, tlen, T.full_lut != 0);

    // (1) Piece list: lane w expands boundary word w.
    int npieces = 0;
    {
      const int nw = (tlen + 31) / 32;
      uint32_t m = 0;
      if (lane < nw) {
        m = S.w.bd[lane];
        const int rem = tlen - 32 * lane;
        if (rem < 32) m &= (1u << rem) - 1u;
      }
      const uint32_t c = __popc(m);
      const uint32_t inc = warp_incl_sum(c, lane);
      int pos = int(inc - c);
      while (m) {
        S.plist[pos++] = static_cast<uint16_t>(32 * lane + __ffs(m) - 1);
        m &= m - 1;
      }
      npieces = int(__shfl_sync(kFull, inc, 31));
    }
    __syncwarp();

    // (2) Resolve or defer every piece, 32 at a time, staging as we go.
    uint32_t* stage = a.staging + tile * kStage;
    uint32_t run = 0, ndef = 0, nlong = 0;
    for (int k0 = 0; k0 < npieces; k0 += 32) {
      const int k = k0 + lane;
      int len = 0, q = 0;
      uint32_t c = 0, r0 = 0, r1 = 0;
      bool deferred = false, lg = false;
      if (k < npieces) {
        q = S.plist[k];
        len = (k + 1 < npieces) ? S.plist[k + 1] - q : next_boundary(S.w.bd, q, kLmax) - q;
        if (len > kLmax) {
          lg = deferred = true;  // long: k_long_pieces, no staging slots
        } else if (len == 1) {
          c = 1;
          r0 = s_lut[S.w.byte(q)];
        } else {
          uint32_t nres;
          if (a.use_memo && len <= kMemoMaxLen && memo_lookup(T, S.w.wbw, q, len, r0, r1, nres)) {
            c = nres;
          } else {
            deferred = true;  // merge piece: k_merge fills `len` reserved slots
            c = uint32_t(len);
          }
        }
        S.plen[k] = lg ? 0xFF : static_cast<uint8_t>(len);
      }
      const uint32_t inc = warp_incl_sum(c, lane);
      const uint32_t slot = run + inc - c;
      if (k < npieces) S.cnt[k] = static_cast<uint16_t>(slot);
      if (!deferred && c) {
        stage[slot] = d2id ? __ldg(d2id + r0) : r0;
        if (c > 1) stage[slot + 1] = d2id ? __ldg(d2id + r1) : r1;
      }
      const unsigned dm = __ballot_sync(kFull, deferred);
      if (deferred) S.dk[ndef + __popc(dm & lanemask_lt(lane))] = static_cast<uint16_t>(k);
      ndef += __popc(dm);
      nlong += __popc(__ballot_sync(kFull, lg));
      run += __shfl_sync(kFull, inc, 31);
    }
    if (lane == 0) S.cnt[npieces] = static_cast<uint16_t>(run);
    __syncwarp();

    // (3) Deferred-piece records (contiguous per tile, in piece order).
    uint64_t first = 0, lfirst = 0;
    if (lane == 0 && ndef) first = atomicAdd(&a.counters[CNT_LREC], ndef);
    if (lane == 0 && nlong) lfirst = atomicAdd(&a.counters[CNT_LONG], nlong);
    first = __shfl_sync(kFull, first, 0);
    lfirst = __shfl_sync(kFull, lfirst, 0);
    if (nlong) {
      // Long pieces (rare): full length to the next hard boundary or row end.
      uint32_t li = 0;
      for (uint32_t i = 0; i < ndef; ++i) {
        const int k = S.dk[i];
        if (S.plen[k] != 0xFF) continue;
        const uint64_t abs = b0 + S.plist[k];
        const uint64_t len = long_piece_length(a, s_junc, abs, lane);
        if (lane == 0) {
          if (first + i < a.lp_cap) a.lrec[first + i] = LongRec{abs, len, 0, S.cnt[k], 0u};
          if (lfirst + li < a.long_cap) a.long_idx[lfirst + li] = uint32_t(first + i);
        }
        ++li;
      }
    }
    for (uint32_t i = lane; i < ndef; i += 32) {
      const int k = S.dk[i];
      if (S.plen[k] == 0xFF) continue;
      if (first + i < a.lp_cap)
        a.lrec[first + i] = LongRec{b0 + S.plist[k], S.plen[k], kMergeKind, S.cnt[k], 0u};
    }
    if (lane == 0) {
      a.tile_lrec[tile] = ndef ? ((first << 24) | ndef) : 0;
      a.tile_count[tile] = run;
    }
    // (4) Row offsets relative to the tile: staging slots before the row (low
    // 40 bits) and deferred pieces before it (above); k_gather resolves them.
    for (uint64_t s = s0 + lane; s < s1 && s <= a.n_rows; s += 32) {
      const int o = static_cast<int>(a.offsets[s] - b0);
      int lo = 0, hi = npieces;  // first piece with plist >= o
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (S.plist[mid] < o) lo = mid + 1; else hi = mid;
      }
      uint64_t lb = 0;
      while (lb < ndef && S.dk[lb] < lo) ++lb;
      a.out_offsets[s] = uint64_t(S.cnt[lo]) | (lb << 40);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// k_merge: the deferred 2..kLmax-byte pieces of every tile, lane per piece,
// lanes refilled as pieces finish. Working arrays live in shared memory in a
// [slot][lane] layout (bank = lane: conflict-free for any per-lane index).
// Tokens go to the slots k_pieces reserved in the piece's tile staging.
template <typename Tk>
struct MergeSmem {
  Tk tok[kLmax][32];
  Tk rnk[kLmax][32];
};

// One lane, one pass (block_engine.hpp:286-307) over a piece held in a
// column of the [slot][lane] arrays: min over cached ranks, sweep-compact in
// place (a pair at the minimum merges unless its left token was just
// consumed -- flags[i+1] = (ranks[i] == m && !flags[i])), re-probe only the
// pairs touching a merged token, two in flight. Returns the new length, or -1.
template <typename Tk>
__device__ __forceinline__ int lane_pass_col(const DevTable& T, Tk (*tok)[32], Tk (*rnk)[32], int lane,
                                             int n) {
  constexpr bool K32 = sizeof(Tk) == 2;
  constexpr uint32_t NONE = Marks<Tk>::kNone, PROBE = Marks<Tk>::kNone - 1;
  uint32_t m = NONE;
  for (int i = 0; i < n - 1; ++i) m = min(m, uint32_t(rnk[i][lane]));
  if (m == NONE) return -1;
  const Tk M = Tk(__ldg(T.r2m + m));
  int j = 0, i = 0;
  while (i < n) {
    const uint32_t ri = (i < n - 1) ? uint32_t(rnk[i][lane]) : NONE;
    if (ri == m) {
      tok[j][lane] = M;
      rnk[j][lane] = Tk(PROBE);
      if (j > 0) rnk[j - 1][lane] = Tk(PROBE);
      i += 2;
    } else {
      tok[j][lane] = tok[i][lane];
      rnk[j][lane] = Tk(ri);
      i += 1;
    }
    ++j;
  }
  int k = 0;
  for (;;) {
    while (k < j - 1 && uint32_t(rnk[k][lane]) != PROBE) ++k;
    if (k >= j - 1) break;
    int k2 = k + 1;
    while (k2 < j - 1 && uint32_t(rnk[k2][lane]) != PROBE) ++k2;
    ProbeReq pa, pb;
    probe_issue<K32>(pa, T, tok[k][lane], tok[k + 1][lane]);
    const bool two = k2 < j - 1;
    if (two) probe_issue<K32>(pb, T, tok[k2][lane], tok[k2 + 1][lane]);
    rnk[k][lane] = Tk(tk_rank<Tk>(probe_resolve<K32>(pa, T)));
    if (two) rnk[k2][lane] = Tk(tk_rank<Tk>(probe_resolve<K32>(pb, T)));
    k = two ? k2 + 1 : j;
  }
  return j;
}

template <typename Tk>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_merge(EncodeArgs a, DevTable T) {
  constexpr bool K32 = sizeof(Tk) == 2;
  __shared__ uint32_t s_lut[256];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  MergeSmem<Tk>* s_m = reinterpret_cast<MergeSmem<Tk>*>(s_dyn);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Tk(*tok)[32] = s_m[wid].tok;
  Tk(*rnk)[32] = s_m[wid].rnk;
  const uint32_t nrec = min((uint64_t)a.counters[CNT_LREC], (uint64_t)a.lp_cap);
  const uint32_t* d2id = T.d2id;
  uint32_t base = 0, next = 0, avail = 0;  // warp-uniform slice of record indices
  bool exhausted = false;
  int n = 0;  // my piece's current length (0 = idle)
  uint32_t ridx = 0;
  for (;;) {
    const bool idle = n == 0;
    const unsigned im = __ballot_sync(kFull, idle);
    if (im && next >= avail && !exhausted) {
      uint32_t c0 = 0;
      if (lane == 0) c0 = atomicAdd(&a.counters[CNT_MERGE_TICKET], 32u);
      base = __shfl_sync(kFull, c0, 0);
      next = 0;
      avail = base < nrec ? min(32u, nrec - base) : 0u;
      exhausted = avail == 0;
    }
    const uint32_t take = min(uint32_t(__popc(im)), avail - next);
    const uint32_t rank = __popc(im & lanemask_lt(lane));
    if (idle && rank < take) {
      ridx = base + next + rank;
      const LongRec r = a.lrec[ridx];
      if (r.row & kMergeKind) {
        n = int(r.len);
        const uint8_t* src = a.bytes + r.start;
        for (int i = 0; i < n; ++i) tok[i][lane] = Tk(s_lut[src[i]]);
        for (int i = 0; i < n - 1; i += 2) {
          ProbeReq p0, p1;
          probe_issue<K32>(p0, T, tok[i][lane], tok[i + 1][lane]);
          const bool two = i + 2 < n;
          if (two) probe_issue<K32>(p1, T, tok[i + 1][lane], tok[i + 2][lane]);
          rnk[i][lane] = Tk(tk_rank<Tk>(probe_resolve<K32>(p0, T)));
          if (two) rnk[i + 1][lane] = Tk(tk_rank<Tk>(probe_resolve<K32>(p1, T)));
        }
      }
    }
    next += take;
    const bool busy = n > 0;
    if (!__any_sync(kFull, busy)) {
      if (exhausted) break;
      continue;
    }
    if (busy) {
      const int r = lane_pass_col<Tk>(T, tok, rnk, lane, n);
      if (r < 2) {
        const int cnt = r < 0 ? n : r;
        const LongRec& rec = a.lrec[ridx];
        uint32_t* dst = a.staging + (rec.start / kTile) * kStage + rec.spref;
        for (int i = 0; i < cnt; ++i) {
          const uint32_t v = tok[i][lane];
          dst[i] = d2id ? __ldg(d2id + v) : v;
        }
        a.lrec[ridx].count = uint32_t(cnt);
        n = 0;
      } else {
        n = r;
      }
    }
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
      uint64_t first = 0, lfirst = 0;
      if (lane == 0 && ne) {
        first = atomicAdd(&a.counters[CNT_LREC], ne);
        lfirst = atomicAdd(&a.counters[CNT_LONG], ne);
      }
      first = __shfl_sync(kFull, first, 0);
      lfirst = __shfl_sync(kFull, lfirst, 0);
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
        if (ne_row && first + before < a.lp_cap) {
          a.lrec[first + before] = LongRec{o, e - o, s, 0u, 0u};
          if (lfirst + before < a.long_cap) a.long_idx[lfirst + before] = uint32_t(first + before);
        }
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
      if (rec) {  // deferred pieces: long ones add their tokens, merge ones
                  // replace their reserved slots by their tokens
        const uint64_t first = rec >> 24;
        const uint32_t nl = uint32_t(rec & 0xFFFFFF);
        for (uint32_t li = 0; li < nl; ++li) {
          const LongRec& r = a.lrec[first + li];
          c += __ldcg(&r.count);
          if (__ldcg(&r.row) & kMergeKind) c -= __ldcg(&r.len);
        }
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
      // Staged slots in order; at each deferred piece: a merge piece's tokens
      // sit in its reserved slots (copy `count`, skip `len`), a long piece's
      // tokens come from lpo (no slots).
      const uint64_t first = rec >> 24;
      const uint32_t nl = uint32_t(rec & 0xFFFFFF);
      uint64_t pos = 0;
      uint32_t sp = 0;
      for (uint32_t li = 0; li < nl; ++li) {
        const LongRec lr = a.lrec[first + li];
        copy_tokens(out + pos, stage + sp, lr.spref - sp, lane);
        pos += lr.spref - sp;
        sp = lr.spref;
        if (lr.row & kMergeKind) {
          copy_tokens(out + pos, stage + sp, lr.count, lane);
          sp += uint32_t(lr.len);
        } else {
          const bool unchanged = (__ldcg(a.lpo + lr.start) & kUnchanged) != 0;
          for (uint32_t i = lane; i < lr.count; i += 32) {
            const uint32_t v = unchanged ? s_lut[a.bytes[lr.start + i]] : __ldcg(a.lpo + lr.start + 1 + i);
            out[pos + i] = d2id ? __ldg(d2id + v) : v;
          }
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
      for (uint32_t li = 0; li < lb; ++li) {
        const LongRec& r = a.lrec[(rec >> 24) + li];
        lsum += __ldcg(&r.count);
        if (__ldcg(&r.row) & kMergeKind) lsum -= __ldcg(&r.len);
      }
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

size_t pieces_smem() { return sizeof(PieceSmem) * kWarpsPerCta; }

LaunchPlan plan_launch(int device) {
  LaunchPlan p;
  cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, device);
  auto grid = [&](auto kern, int threads, size_t smem) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    return p.sm_count * (per_sm > 0 ? per_sm : 1);
  };
  cudaFuncSetAttribute(k_pieces, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pieces_smem()));
  p.main_grid = grid(k_pieces, kWarpsPerCta * 32, pieces_smem());
  p.main_grid_wide = p.main_grid;
  cudaFuncSetAttribute(k_merge<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(MergeSmem<uint16_t>) * kWarpsPerCta));
  cudaFuncSetAttribute(k_merge<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(sizeof(MergeSmem<uint32_t>) * kWarpsPerCta));
  p.merge_grid = grid(k_merge<uint16_t>, kWarpsPerCta * 32, sizeof(MergeSmem<uint16_t>) * kWarpsPerCta);
  p.merge_grid_wide = grid(k_merge<uint32_t>, kWarpsPerCta * 32, sizeof(MergeSmem<uint32_t>) * kWarpsPerCta);
  p.lp_grid = grid(k_long_pieces<kLpThreads>, kLpThreads, 0);
  p.gather_grid = grid(k_gather, kWarpsPerCta * 32, 0);
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
  if (a.engine == BBPE_ENGINE_BLOCK) {
    k_block_rows<<<p.gather_grid, kWarpsPerCta * 32, 0, stream>>>(a, t);
    ++launched;
    if (ev) cudaEventRecord(ev[2], stream);
  } else {
    k_pieces<<<p.main_grid, kWarpsPerCta * 32, pieces_smem(), stream>>>(a, t);
    ++launched;
    if (ev) cudaEventRecord(ev[2], stream);
    if (a.narrow)
      k_merge<uint16_t><<<p.merge_grid, kWarpsPerCta * 32, sizeof(MergeSmem<uint16_t>) * kWarpsPerCta,
                          stream>>>(a, t);
    else
      k_merge<uint32_t><<<p.merge_grid_wide, kWarpsPerCta * 32, sizeof(MergeSmem<uint32_t>) * kWarpsPerCta,
                          stream>>>(a, t);
    ++launched;
  }
  if (ev) cudaEventRecord(ev[3], stream);
  k_long_pieces<kLpThreads><<<p.lp_grid, kLpThreads, 0, stream>>>(a, t);
  ++launched;
  if (ev) cudaEventRecord(ev[4], stream);
  k_tile_scan<<<unsigned((a.num_tiles + kScanTiles - 1) / kScanTiles), kScanThreads, 0, stream>>>(a);
  ++launched;
  if (ev) cudaEventRecord(ev[5], stream);
  k_gather<<<p.gather_grid, kWarpsPerCta * 32, 0, stream>>>(a, t);
  ++launched;
  if (ev) cudaEventRecord(ev[6], stream);
  return launched;
}

int launch_block_bpe(const EncodeArgs& a, const DevTable& t, const LaunchPlan& p,
                     cudaStream_t stream) {
  (void)p;
  k_long_pieces<kLpThreads><<<1, kLpThreads, 0, stream>>>(a, t);
  return 1;
}

}  // namespace bbpe
