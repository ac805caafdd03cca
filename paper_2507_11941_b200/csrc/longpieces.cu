// longpieces.cu -- the block engine for long pieces: one WARP per piece.
//
// Semantics: block_bpe (reference proj/include/blockbpe/block_engine.hpp:268-310)
// on one piece: per pass, m = min rank over all adjacent pairs (fill_pair_ranks
// 72-79, reduce_min_rank 82-97), stop when no pair is in the table (288-289);
// mark left-greedy, non-overlapping occurrences of the rank-m pair
// (fill_merge_flags 103-128: f[i+1] = r[i] == m && !f[i]); replace each
// marked pair by its merged token (compact_into 166-182). Used for pieces of
// more than kLmax bytes that k_pieces found, every row under
// BBPE_ENGINE_BLOCK (the paper's one-block-per-string engine), max_passes,
// and bbpe_block_bpe.
//
// The pass loop costs O(work that changes), not O(piece length) per pass
// (exactness-preserving restatements):
//   * tombstones: positions never move; a merged-away token is cleared from
//     its segment's live mask. "Adjacent" means adjacent LIVE tokens.
//   * cached ranks: a pair's rank depends on its two tokens only, so only
//     pairs touching a merged token are probed again (PEND).
//   * cached minima: segment = 32 consecutive positions (one per lane, bank =
//     lane); smin[s] = min rank of the segment's live pairs, gmin[g] = min of
//     32 segments. The global minimum is a REDUX over gmin; a pass visits only
//     the segments whose minimum is m ("dirty") and re-minimises only the
//     segments it touched.
//   * left-greedy marking walks the rank-m pairs of a dirty segment in order;
//     the token a merge consumes is cleared at once, also when it lies in a
//     later segment, so a run of m-pairs continues correctly across segments.
//   * the merged id of a pass is r2m[m] (ranks are unique per pair,
//     merge_table.hpp:264-268), not a probe per merge (compact_into 173).
// Working set: a piece of <= kLpSmemBytes / record size tokens lives in the
// warp's slice of shared memory; for longer ones (64 KiB byte runs, long
// rows under the block engine) the positions move to the global scratch
// (L2-resident) and, beyond ~64K positions, the metadata too: same code
// through generic pointers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"
#include "probe.cuh"

namespace bbpe {
namespace {

constexpr unsigned kFullMask = 0xFFFFFFFFu;
constexpr uint32_t kUnchangedFlag = 0x80000000u;  // lpo flag: piece merged nothing (k_gather reads bytes)

// Position record: token + rank of the pair (this, next live). Narrow tables
// (ids, ranks < 2^16): u32 = rank << 16 | token; wide: u64 = rank << 32 | token.
template <bool NARROW>
struct Pos;
template <>
struct Pos<true> {
  using T = uint32_t;
  static constexpr uint32_t NONE = 0xFFFFu, PEND = 0xFFFEu;
  __device__ static uint32_t tok(T e) { return e & 0xFFFFu; }
  __device__ static uint32_t rank(T e) { return e >> 16; }
  __device__ static T make(uint32_t t, uint32_t r) { return (r << 16) | t; }
  __device__ static uint32_t from_rk(uint32_t rk) { return rk >> 16; }  // probe32: rank << 16 | merged
};
template <>
struct Pos<false> {
  using T = uint64_t;
  static constexpr uint32_t NONE = 0xFFFFFFFFu, PEND = 0xFFFFFFFEu;
  __device__ static uint32_t tok(T e) { return static_cast<uint32_t>(e); }
  __device__ static uint32_t rank(T e) { return static_cast<uint32_t>(e >> 32); }
  __device__ static T make(uint32_t t, uint32_t r) { return (uint64_t(r) << 32) | t; }
  __device__ static uint32_t from_rk(uint32_t rk) { return rk; }  // dense rank, kNoRank on a miss
};

// Bits strictly above `b` (b in [0, 31]).
__device__ __forceinline__ uint32_t above(uint32_t b) { return b >= 31 ? 0u : (~0u << (b + 1)); }

// The warp's view of one piece: n positions, nseg = ceil(n / 32) segments,
// ngrp = ceil(nseg / 32) groups (one aff word and one gmin per group).
template <bool NARROW>
struct Piece {
  typename Pos<NARROW>::T* P;
  uint32_t* live;  // nseg: live-token mask per segment
  uint32_t* smin;  // nseg: min rank of the segment's live pairs
  uint32_t* gmin;  // ngrp
  uint32_t* aff;   // ngrp: segments touched in this pass (bit s & 31 of word s >> 5)
  uint32_t n, nseg, ngrp;
};

// Per-warp metadata words in shared memory for a piece of `cap` positions.
__host__ __device__ constexpr uint32_t lp_meta_words(uint32_t cap) {
  return 2 * ((cap + 31) / 32) + 2 * ((cap + 1023) / 1024);
}
template <bool NARROW>
__host__ __device__ constexpr uint32_t lp_cap() {
  return NARROW ? kLpSmemBytes / 4 : kLpSmemBytes / 8;
}
template <bool NARROW>
__host__ __device__ constexpr uint32_t lp_warp_bytes() {
  return kLpSmemBytes + 4 * lp_meta_words(lp_cap<NARROW>());
}

// First live position in segments >= s, or -1 (warp-uniform loop).
template <bool NARROW>
__device__ __forceinline__ int64_t first_live_from(const Piece<NARROW>& V, uint32_t s) {
  for (; s < V.nseg; ++s) {
    const uint32_t L = V.live[s];
    if (L) return int64_t(32) * s + __ffs(L) - 1;
  }
  return -1;
}
// Last live position in segments < s, or -1.
template <bool NARROW>
__device__ __forceinline__ int64_t last_live_before(const Piece<NARROW>& V, uint32_t s) {
  while (s > 0) {
    --s;
    const uint32_t L = V.live[s];
    if (L) return int64_t(32) * s + 31 - __clz(L);
  }
  return -1;
}

__device__ __forceinline__ void mark_aff(uint32_t* aff, uint32_t s) { aff[s >> 5] |= 1u << (s & 31); }

// Re-ranks the PEND pairs of every touched segment (probes in flight across
// up to 4 segments per batch), then their segment and group minima.
template <bool NARROW>
__device__ void resolve_touched(const Piece<NARROW>& V, const DevTable& T, int lane) {
  using PT = Pos<NARROW>;
  constexpr int B = 4;
  for (uint32_t g0 = 0; g0 < V.ngrp; g0 += 32) {
    const uint32_t gl = g0 + lane;
    const uint32_t aw = gl < V.ngrp ? V.aff[gl] : 0u;
    for (unsigned gm = __ballot_sync(kFullMask, aw != 0); gm; gm &= gm - 1) {
      const uint32_t g = g0 + __ffs(gm) - 1;
      uint32_t w = __shfl_sync(kFullMask, aw, __ffs(gm) - 1);
      while (w) {
        uint32_t segs[B];
        int k = 0;
#pragma unroll
        for (int u = 0; u < B; ++u) {
          segs[u] = w ? 32 * g + __ffs(w) - 1 : ~0u;
          if (w) {
            w &= w - 1;
            ++k;
          }
        }
        typename PT::T e[B];
        uint32_t L[B];
        bool pend[B], has_r[B];
        ProbeReq q[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          pend[u] = false;
          has_r[u] = false;
          e[u] = 0;
          L[u] = 0;
          if (u < k) {
            if (32 * segs[u] + lane < V.n) e[u] = V.P[32 * segs[u] + lane];
            L[u] = V.live[segs[u]];
          }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
          if (u >= k) continue;
          const bool lv = (L[u] >> lane) & 1u;
          pend[u] = lv && PT::rank(e[u]) == PT::PEND;
          const uint32_t nb = L[u] & above(lane);
          const uint32_t rt_in = __shfl_sync(kFullMask, PT::tok(e[u]), nb ? __ffs(nb) - 1 : lane);
          uint32_t rt = rt_in;
          has_r[u] = nb != 0;
          if (pend[u] && !nb) {  // the right neighbour lies in a later segment (or there is none)
            const int64_t q2 = first_live_from(V, segs[u] + 1);
            has_r[u] = q2 >= 0;
            if (has_r[u]) rt = PT::tok(V.P[q2]);
          }
          if (pend[u] && has_r[u]) probe_issue<NARROW>(q[u], T, PT::tok(e[u]), rt);
        }
        __syncwarp();  // reads of right neighbours in later segments before this batch's writes
#pragma unroll
        for (int u = 0; u < B; ++u) {
          if (u >= k) continue;
          const bool lv = (L[u] >> lane) & 1u;
          if (pend[u]) {
            const uint32_t r = has_r[u] ? PT::from_rk(probe_resolve<NARROW>(q[u], T)) : PT::NONE;
            e[u] = PT::make(PT::tok(e[u]), r);
            V.P[32 * segs[u] + lane] = e[u];
          }
          const uint32_t sm = __reduce_min_sync(kFullMask, lv ? PT::rank(e[u]) : PT::NONE);
          if (lane == 0) V.smin[segs[u]] = sm;
        }
      }
      __syncwarp();
      const uint32_t sl = 32 * g + lane;
      const uint32_t gmv = __reduce_min_sync(kFullMask, sl < V.nseg ? V.smin[sl] : PT::NONE);
      if (lane == 0) {
        V.gmin[g] = gmv;
        V.aff[g] = 0;
      }
      __syncwarp();
    }
  }
}

// One pass at rank m over the dirty segments: left-greedy marks, merges,
// tombstones, PEND for every pair whose tokens changed. Returns the number
// of merges.
template <bool NARROW>
__device__ uint32_t merge_pass(const Piece<NARROW>& V, uint32_t m, uint32_t M, int lane) {
  using PT = Pos<NARROW>;
  uint32_t merges = 0;
  for (uint32_t g0 = 0; g0 < V.ngrp; g0 += 32) {
    const uint32_t gl = g0 + lane;
    const bool gd = gl < V.ngrp && V.gmin[gl] == m;
    for (unsigned gm = __ballot_sync(kFullMask, gd); gm; gm &= gm - 1) {
      const uint32_t g = g0 + __ffs(gm) - 1;
      const uint32_t sl = 32 * g + lane;
      unsigned dm = __ballot_sync(kFullMask, sl < V.nseg && V.smin[sl] == m);
      for (; dm; dm &= dm - 1) {
        const uint32_t s = 32 * g + __ffs(dm) - 1;
        const uint32_t p = 32 * s + lane;
        typename PT::T e = p < V.n ? V.P[p] : typename PT::T(0);
        const uint32_t L = V.live[s];
        const bool lv = (L >> lane) & 1u;
        const bool isM = lv && PT::rank(e) == m;
        const unsigned Mb = __ballot_sync(kFullMask, isM);
        // Left-greedy in live order (fill_merge_flags 103-128) by run parity:
        // a run is a stretch of consecutive live lanes whose pairs have rank m;
        // its lanes at even live offsets from the run start are marked, each
        // consuming the next live token. A run never continues from an earlier
        // segment: if that segment's last pair was marked, this segment's first
        // live token is already cleared (out_kill below), otherwise the first
        // m-pair here is at an even offset anyway.
        const uint32_t below = L & ((1u << lane) - 1u);
        const bool prev_m = below && ((Mb >> (31 - __clz(below))) & 1u);
        const unsigned S = __ballot_sync(kFullMask, isM && !prev_m);  // run starts
        const uint32_t sb = S & (lane == 31 ? ~0u : ((2u << lane) - 1u));
        const uint32_t st = sb ? 31 - __clz(sb) : 0;
        const bool mk = isM && !(__popc(below & ~((1u << st) - 1u)) & 1u);
        const uint32_t merged = __ballot_sync(kFullMask, mk);
        if (!merged) continue;
        // consumed tokens: the live successor of every marked lane
        const uint32_t kill = __ballot_sync(kFullMask, lv && below && ((merged >> (31 - __clz(below))) & 1u));
        const bool last_marked = (merged >> (31 - __clz(L))) & 1u;  // its right token is in a later segment
        const int64_t out_kill = last_marked ? first_live_from(V, s + 1) : -1;
        merges += __popc(merged);
        const uint32_t Ln = L & ~kill;
        const bool me = (merged >> lane) & 1u;
        // The left neighbour of a merged token: its pair changed.
        const uint32_t nbx = Ln & above(lane);
        const bool left_of_merge = ((Ln >> lane) & 1u) && !me && nbx && ((merged >> (__ffs(nbx) - 1)) & 1u);
        __syncwarp();  // every lane has read live[s] and its neighbours before they change
        if (me) V.P[p] = PT::make(M, PT::PEND);
        else if (left_of_merge) V.P[p] = PT::make(PT::tok(e), PT::PEND);
        if (lane == 0) {
          V.live[s] = Ln;
          mark_aff(V.aff, s);
          // First merged token without a live predecessor in the segment: the
          // predecessor's pair (in an earlier segment) changed.
          if (__ffs(merged) == __ffs(Ln)) {
            const int64_t pv = last_live_before(V, s);
            if (pv >= 0) {
              V.P[pv] = PT::make(PT::tok(V.P[pv]), PT::PEND);
              mark_aff(V.aff, uint32_t(pv >> 5));
            }
          }
          if (out_kill >= 0) {  // a token of a later segment consumed
            const uint32_t s2 = uint32_t(out_kill >> 5);
            V.live[s2] &= ~(1u << (out_kill & 31));
            mark_aff(V.aff, s2);
          }
        }
        __syncwarp();
      }
    }
  }
  return merges;
}

template <bool NARROW>
__device__ uint32_t global_min(const Piece<NARROW>& V, int lane) {
  uint32_t x = Pos<NARROW>::NONE;
  for (uint32_t g = lane; g < V.ngrp; g += 32) x = min(x, V.gmin[g]);
  return __reduce_min_sync(kFullMask, x);
}

// The whole pass loop for piece `ridx` of the long list, by one warp.
template <bool NARROW>
__device__ void run_piece(const EncodeArgs& a, const DevTable& T, const uint32_t* s_lut, uint32_t ridx,
                          unsigned char* smem, int lane) {
  using PT = Pos<NARROW>;
  const LongRec R = a.lrec[ridx];
  const uint32_t n = static_cast<uint32_t>(R.len);
  Piece<NARROW> V;
  V.n = n;
  V.nseg = (n + 31) / 32;
  V.ngrp = (V.nseg + 31) / 32;
  // Working set: positions and metadata in the warp's shared memory (n <=
  // cap); positions in the global scratch lpy and metadata in shared memory
  // (up to ~64K positions); both in global scratch (lpy, lpx) beyond.
  const uint32_t meta_words = 2 * V.nseg + 2 * V.ngrp;
  uint32_t* meta;
  if (n <= lp_cap<NARROW>()) {
    V.P = reinterpret_cast<typename PT::T*>(smem);
    meta = reinterpret_cast<uint32_t*>(smem + kLpSmemBytes);
  } else {
    V.P = reinterpret_cast<typename PT::T*>(a.lpy + R.start);
    meta = meta_words * 4 <= uint32_t(kLpSmemBytes) ? reinterpret_cast<uint32_t*>(smem)
                                                    : reinterpret_cast<uint32_t*>(a.lpx + R.start);
  }
  V.live = meta;
  V.smin = meta + V.nseg;
  V.gmin = meta + 2 * V.nseg;
  V.aff = V.gmin + V.ngrp;
  // Initial tokens (bytes_to_initial_tokens, pretokenize.hpp:60-71) or the
  // caller's tokens (bbpe_block_bpe: lpx holds them, read before lpx is
  // reused for metadata), every pair pending except the last.
  for (uint32_t s = 0; s < V.nseg; ++s) {
    const uint32_t i = 32 * s + lane;
    if (i < n) {
      const uint32_t t = a.tokens_input ? static_cast<uint32_t>(a.lpx[R.start + i]) : s_lut[a.bytes[R.start + i]];
      V.P[i] = PT::make(t, i + 1 < n ? PT::PEND : PT::NONE);
    }
  }
  __syncwarp();
  for (uint32_t s = lane; s < V.nseg; s += 32) {
    const uint32_t rem = n - 32 * s;
    V.live[s] = rem >= 32 ? ~0u : ((1u << rem) - 1u);
  }
  for (uint32_t g = lane; g < V.ngrp; g += 32) {
    const uint32_t rem = V.nseg - 32 * g;
    V.aff[g] = rem >= 32 ? ~0u : ((1u << rem) - 1u);
  }
  __syncwarp();
  resolve_touched<NARROW>(V, T, lane);

  uint64_t pass = 0;
  bool maxpass_hit = false;
  uint32_t count = n;
  for (;;) {
    const uint32_t m = global_min<NARROW>(V, lane);
    if (m == PT::NONE) break;  // no pair in the table (block_engine.hpp:288-289)
    if (a.max_passes > 0 && pass >= uint64_t(a.max_passes)) {  // (291-295)
      maxpass_hit = true;
      break;
    }
    const uint32_t M = __ldg(T.r2m + m);
    const uint32_t merges = merge_pass<NARROW>(V, m, M, lane);
    if (a.trace && lane == 0 && pass < a.trace_cap) {  // PassTrace (42-47, 303-304)
      a.trace[3 * pass] = pass + 1;
      a.trace[3 * pass + 1] = T.rank_orig[m];
      a.trace[3 * pass + 2] = merges;
    }
    count -= merges;
    ++pass;
    resolve_touched<NARROW>(V, T, lane);
  }
  if (maxpass_hit && lane == 0)
    atomicMin(reinterpret_cast<unsigned long long*>(&a.err[ERR_MAXPASS_ROW]), (unsigned long long)R.row);
  if (a.trace && lane == 0 && a.trace_count) *a.trace_count = pass;
  // Result: lpo[start] = count (| unchanged), then the live tokens in order.
  uint32_t* O = a.lpo + R.start;
  const bool unchanged = count == n && !a.tokens_input;
  if (lane == 0) {
    O[0] = count | (unchanged ? kUnchangedFlag : 0u);
    a.lrec[ridx].count = count;
    if (!a.tokens_input) atomicAdd(&a.tile_count[R.start / kTile], count);
  }
  if (!unchanged) {
    uint32_t base = 0;
    for (uint32_t s = 0; s < V.nseg; ++s) {
      const uint32_t L = V.live[s];
      if ((L >> lane) & 1u) O[1 + base + __popc(L & ((1u << lane) - 1u))] = PT::tok(V.P[32 * s + lane]);
      base += __popc(L);
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Super-pass engine: many consecutive passes of block_bpe per sweep, exactly.
//
// Let the current pairs have ranks r_i (kNoRank = none). Run the passes of
// block_bpe (block_engine.hpp:286-307) from here, and call a token FRESH if
// one of these passes created it. As long as no pass merges a pair with a
// fresh token, the passes only merge current pairs, each in its own rank's
// pass, so which current pairs merge is decided by rank order alone:
//   * pair i merges iff it is not consumed first by a lower-ranked neighbour
//     pair that merges, nor (equal ranks = a run of one repeated pair) by a
//     left neighbour of the run that merges (left-greedy, fill_merge_flags
//     103-128). Closed form: with a_i = the number of consecutive
//     non-decreasing steps r_{i-1} <= r_i ending at i and b_i = the number of
//     consecutive strictly decreasing steps r_{i+1} < r_i starting at i,
//     pair i merges iff r_i != none, a_i is even and b_i is even (chains of
//     decreasing rank alternate from their minimum; a peak merges iff both
//     lower neighbours do not).
// The first pass that merges a fresh token: a merge of pair i (at rank
// tau = r_i, merged token M) creates the pairs (left token at tau, M) and
// (M, right token at tau), whose ranks x are processed no earlier than
// max(x, tau + 1). With C = the minimum of that over all merges, every pass
// below C merges current pairs only, so applying all merges with r_i < C in
// one sweep is exactly those passes (C > the global minimum rank, so every
// super-pass makes progress). Conservative in one respect only (a fresh pair
// that a later merge of the same sweep destroys still bounds C), which costs
// sweeps, never exactness. Checked against block_bpe on the compiled
// reference (tests) and on random consistent and inconsistent tables
// (oracle/bpe_oracle.c restatement, tests/test_superpass.py).
//
// Layout: positions in a warp's slice of shared memory (or, for pieces
// longer than kLpSmemBytes / 8, in the piece's global scratch): X[i] token,
// R[i] = rk of (X[i], X[i+1]); per 32-position segment a b-parity mask and a
// merge mask. Every super-pass is four coalesced sweeps (b parity right to
// left, merge mask left to right, cut, in-place compaction with re-probes of
// the pairs that changed); positions shrink to the live tokens each time.
// Used unless a pass cap or a trace asks for pass-by-pass execution.

template <bool NARROW>
__device__ __forceinline__ uint32_t sp_merged(const DevTable& T, uint32_t rk) {
  return NARROW ? (rk & 0xFFFFu) : __ldg(T.r2m + rk);
}

// Value of lane + k of a segment (k = 1, 2), continuing into the next segment.
__device__ __forceinline__ uint32_t lane_ahead(uint32_t cur, uint32_t nxt, int lane, int k) {
  const uint32_t a = __shfl_down_sync(kFullMask, cur, k);
  const uint32_t b = __shfl_sync(kFullMask, nxt, (lane + k) & 31);
  return lane + k < 32 ? a : b;
}
// Value of lane - k (k = 1, 2), continuing into the previous segment.
__device__ __forceinline__ uint32_t lane_behind(uint32_t cur, uint32_t prv, int lane, int k) {
  const uint32_t a = __shfl_up_sync(kFullMask, cur, k);
  const uint32_t b = __shfl_sync(kFullMask, prv, (lane - k) & 31);
  return lane >= k ? a : b;
}
__device__ __forceinline__ uint32_t bit_ahead(uint32_t cur, uint32_t nxt, int lane, int k) {
  return lane + k < 32 ? (cur >> (lane + k)) & 1u : (nxt >> (lane + k - 32)) & 1u;
}
__device__ __forceinline__ uint32_t bit_behind(uint32_t cur, uint32_t prv, int lane, int k) {
  return lane >= k ? (cur >> (lane - k)) & 1u : (prv >> (lane + 32 - k)) & 1u;
}

constexpr uint32_t kEvenLanes = 0x55555555u, kOddLanes = 0xAAAAAAAAu;
// Segments per batch of the sweeps (b parity, merge masks + cut, apply) of
// the shared-memory instance; the pipelined instance uses 8 / 4 / 4.
#ifndef BBPE_SP_UA
#define BBPE_SP_UA 8
#endif
#ifndef BBPE_SP_UB
#define BBPE_SP_UB 2
#endif
#ifndef BBPE_PIPE_UA
#define BBPE_PIPE_UA 8
#endif
#ifndef BBPE_PIPE_UB
#define BBPE_PIPE_UB 2
#endif
#ifndef BBPE_PIPE_UC
#define BBPE_PIPE_UC 2
#endif
#ifndef BBPE_SP_UC
#define BBPE_SP_UC 2
#endif

template <bool NARROW, bool PIPE>
__device__ void run_piece_sp(const EncodeArgs& a, const DevTable& T, const uint32_t* s_lut, uint32_t ridx,
                             unsigned char* smem, int lane) {
  const LongRec Rec = a.lrec[ridx];
  const uint32_t n0 = static_cast<uint32_t>(Rec.len);
  const uint32_t nseg0 = (n0 + 31) / 32;
  constexpr uint32_t cap = kLpSmemBytes / 8;
  uint32_t *X, *R, *bm, *mm;
  if (n0 <= cap) {
    X = reinterpret_cast<uint32_t*>(smem);
    R = X + cap;
    bm = R + cap;
    mm = bm + cap / 32;
  } else {
    X = reinterpret_cast<uint32_t*>(a.lpx + Rec.start);
    R = X + n0;
    bm = reinterpret_cast<uint32_t*>(a.lpy + Rec.start);
    mm = bm + nseg0;
  }
  const uint8_t* bytes = a.bytes + Rec.start;
  const uint32_t lt_mask = (1u << lane) - 1u;
  // Initial tokens (bytes_to_initial_tokens, pretokenize.hpp:60-71) and ranks
  // (fill_pair_ranks, block_engine.hpp:72-79).
  {
    constexpr int U = 4;
    for (uint32_t s0 = 0; s0 < nseg0; s0 += U) {
      uint32_t t[U], nx[U];
      ProbeReq q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = 32 * (s0 + u) + lane;
        t[u] = i < n0 ? s_lut[bytes[i]] : 0u;
        nx[u] = (lane == 31 && i + 1 < n0) ? s_lut[bytes[i + 1]] : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = 32 * (s0 + u) + lane;
        const uint32_t d = __shfl_down_sync(kFullMask, t[u], 1);
        if (i + 1 < n0) probe_issue<NARROW>(q[u], T, t[u], lane == 31 ? nx[u] : d);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = 32 * (s0 + u) + lane;
        if (i < n0) {
          X[i] = t[u];
          R[i] = i + 1 < n0 ? probe_resolve<NARROW>(q[u], T) : kNoRank;
        }
      }
    }
  }
  __syncwarp();
  uint32_t n = n0;
  for (;;) {
    const uint32_t nseg = (n + 31) / 32;
    // Phase A, right to left: bm[s] bit = b_i even (b_i = strictly decreasing
    // steps from i). The carry between segments is one parity bit; the ballots
    // do not depend on it, so consecutive segments overlap.
    {
      constexpr int U = PIPE ? BBPE_PIPE_UA : BBPE_SP_UA;
      uint32_t r_next0 = kNoRank, c = 0;
      // Software-pipelined: the next batch's loads are in flight while this
      // one is processed (the L2 path's latency).
      uint32_t rq[U];
#pragma unroll
      for (int u = 0; u < U && PIPE; ++u) {
        const int s = int(nseg) - 1 - u;
        const uint32_t i = 32 * uint32_t(s) + lane;
        rq[u] = (s >= 0 && i < n) ? R[i] : kNoRank;
      }
      for (int s0 = int(nseg) - 1; s0 >= 0; s0 -= U) {
        uint32_t r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (PIPE) {
            r[u] = rq[u];
            const int s = s0 - U - u;
            const uint32_t i = 32 * uint32_t(s) + lane;
            rq[u] = (s >= 0 && i < n) ? R[i] : kNoRank;
          } else {
            const int s = s0 - u;
            const uint32_t i = 32 * uint32_t(s) + lane;
            r[u] = (s >= 0 && i < n) ? R[i] : kNoRank;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int s = s0 - u;
          if (s < 0) break;
          const uint32_t nx0 = u == 0 ? r_next0 : __shfl_sync(kFullMask, r[u > 0 ? u - 1 : 0], 0);
          const uint32_t rd = __shfl_down_sync(kFullMask, r[u], 1);
          const uint32_t rn = lane == 31 ? nx0 : rd;
          const unsigned D = __ballot_sync(kFullMask, rn < r[u]);
          const uint32_t Z = ~D & (~0u << lane);  // non-descending steps at or above lane
          const unsigned Eb = __ballot_sync(kFullMask, Z && !((__ffs(Z) - 1 - lane) & 1u));
          const unsigned Zt = __ballot_sync(kFullMask, Z == 0);  // lanes whose run reaches the next segment
          const unsigned E = Eb | (Zt & (c ? kOddLanes : kEvenLanes));
          if (lane == 0) bm[s] = E;
          c = (E & 1u) ^ 1u;  // parity of b at lane 0
        }
        r_next0 = __shfl_sync(kFullMask, r[U - 1], 0);
      }
    }
    __syncwarp();
    // Phase B, left to right: a parity and the merge masks, and (one segment
    // behind, once the next segment's mask is known) the cut C.
    bool any = false;
    uint32_t C = kNoRank;
    {
      constexpr int U = PIPE ? BBPE_PIPE_UB : BBPE_SP_UB;
      // window: [0] = segment s0-2, [1] = s0-1, [2 + u] = s0 + u
      uint32_t wx[U + 2], wr[U + 2], wm[U + 2];
      wx[0] = wx[1] = 0u;
      wr[0] = wr[1] = kNoRank;
      wm[0] = wm[1] = 0u;
      uint32_t c = 0;  // parity of a at lane 31 of the previous segment
      uint32_t qx[U], qr[U], qb[U];  // the next batch, in flight (software pipelining)
#pragma unroll
      for (int u = 0; u < U && PIPE; ++u) {
        const uint32_t s = u, i = 32 * s + lane;
        qx[u] = i < n ? X[i] : 0u;
        qr[u] = i < n ? R[i] : kNoRank;
        qb[u] = s < nseg ? bm[s] : 0u;
      }
      for (uint32_t s0 = 0; s0 <= nseg; s0 += U) {
        uint32_t bv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (PIPE) {
            wx[2 + u] = qx[u];
            wr[2 + u] = qr[u];
            bv[u] = qb[u];
            const uint32_t s = s0 + U + u, i = 32 * s + lane;
            qx[u] = i < n ? X[i] : 0u;
            qr[u] = i < n ? R[i] : kNoRank;
            qb[u] = s < nseg ? bm[s] : 0u;
          } else {
            const uint32_t s = s0 + u, i = 32 * s + lane;
            wx[2 + u] = i < n ? X[i] : 0u;
            wr[2 + u] = i < n ? R[i] : kNoRank;
            bv[u] = s < nseg ? bm[s] : 0u;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t s = s0 + u;
          if (s >= nseg) {
            wm[2 + u] = 0u;
            continue;
          }
          const uint32_t p31 = __shfl_sync(kFullMask, wr[1 + u], 31);
          const uint32_t ru = __shfl_up_sync(kFullMask, wr[2 + u], 1);
          const uint32_t rp = lane == 0 ? p31 : ru;
          const unsigned Up = __ballot_sync(kFullMask, rp <= wr[2 + u]);
          const uint32_t Z = ~Up & (lane == 31 ? ~0u : ((2u << lane) - 1u));  // breaks at or below lane
          const unsigned Ab = __ballot_sync(kFullMask, Z && !((lane - (31 - __clz(Z))) & 1u));
          const unsigned Zb = __ballot_sync(kFullMask, Z == 0);  // runs from the previous segment
          const unsigned A = Ab | (Zb & (c ? kEvenLanes : kOddLanes));
          const unsigned Nn = __ballot_sync(kFullMask, wr[2 + u] != kNoRank);
          const uint32_t Mm = A & bv[u] & Nn;
          wm[2 + u] = Mm;
          if (lane == 0) mm[s] = Mm;
          any |= Mm != 0;
          c = ((A >> 31) & 1u) ^ 1u;  // parity of a at lane 31
        }
        // The cut for window segments [1, U] (s0-1 .. s0+U-2).
        uint32_t cmin = kNoRank;
#pragma unroll
        for (int j = 1; j <= U; ++j) {
          const int64_t s = int64_t(s0) + j - 2;
          if (s < 0 || s >= int64_t(nseg) || !wm[j]) continue;
          const uint32_t i = 32 * uint32_t(s) + lane;
          const uint32_t tau = wr[j];
          const bool act = ((wm[j] >> lane) & 1u) && tau < C;
          // left token when pair i merges: M of pair i-2 if it merged first, else X[i-1]
          const uint32_t xm1 = lane_behind(wx[j], wx[j - 1], lane, 1);
          const uint32_t rm2 = lane_behind(wr[j], wr[j - 1], lane, 2);
          const uint32_t mm2 = bit_behind(wm[j], wm[j - 1], lane, 2);
          // right token: M of pair i+2 if it merged first, else X[i+2]
          const uint32_t xp2 = lane_ahead(wx[j], wx[j + 1], lane, 2);
          const uint32_t rp2 = lane_ahead(wr[j], wr[j + 1], lane, 2);
          const uint32_t mp2 = bit_ahead(wm[j], wm[j + 1], lane, 2);
          ProbeReq ql, qr;
          const bool hl = act && i >= 1, hr = act && i + 2 < n;
          if (act) {
            const uint32_t M = sp_merged<NARROW>(T, tau);
            if (hl) probe_issue<NARROW>(ql, T, (i >= 2 && mm2 && rm2 <= tau) ? sp_merged<NARROW>(T, rm2) : xm1, M);
            if (hr) probe_issue<NARROW>(qr, T, M, (mp2 && rp2 <= tau) ? sp_merged<NARROW>(T, rp2) : xp2);
          }
          if (hl) {
            const uint32_t x = probe_resolve<NARROW>(ql, T);
            if (x != kNoRank) cmin = min(cmin, max(x, tau + 1));
          }
          if (hr) {
            const uint32_t x = probe_resolve<NARROW>(qr, T);
            if (x != kNoRank) cmin = min(cmin, max(x, tau + 1));
          }
        }
        C = __reduce_min_sync(kFullMask, min(C, cmin));
        wx[0] = wx[U];
        wx[1] = wx[U + 1];
        wr[0] = wr[U];
        wr[1] = wr[U + 1];
        wm[0] = wm[U];
        wm[1] = wm[U + 1];
      }
    }
    if (!any) break;  // no pair in the table (block_engine.hpp:288-289)
    __syncwarp();
    // Phase C, left to right: apply the merges below C, compact in place
    // (destinations never pass the position being read), re-rank the pairs
    // whose tokens changed.
    {
      constexpr int U = PIPE ? BBPE_PIPE_UC : BBPE_SP_UC;
      uint32_t q0 = 0, ap_prev = 0;
      // Segments s0..s0+U (one of lookahead); segments s0+U+1.. of the next
      // batch are loaded before this batch's writes, which only reach
      // positions below 32 (s0 + U) (in-place compaction never passes its reads).
      uint32_t px[U + 1], pr[U + 1], pm[U + 1];
#pragma unroll
      for (int u = 0; u <= U && PIPE; ++u) {
        const uint32_t s = u, i = 32 * s + lane;
        px[u] = i < n ? X[i] : 0u;
        pr[u] = i < n ? R[i] : kNoRank;
        pm[u] = s < nseg ? mm[s] : 0u;
      }
      for (uint32_t s0 = 0; s0 < nseg; s0 += U) {
        uint32_t wx[U + 1], wr[U + 1], Aa[U + 1];
        if (!PIPE) {
#pragma unroll
          for (int u = 0; u <= U; ++u) {
            const uint32_t s = s0 + u, i = 32 * s + lane;
            px[u] = i < n ? X[i] : 0u;
            pr[u] = i < n ? R[i] : kNoRank;
            pm[u] = s < nseg ? mm[s] : 0u;
          }
        }
#pragma unroll
        for (int u = 0; u <= U; ++u) {
          wx[u] = px[u];
          wr[u] = pr[u];
          Aa[u] = __ballot_sync(kFullMask, ((pm[u] >> lane) & 1u) && wr[u] < C);
        }
        if (PIPE) {
          px[0] = px[U];
          pr[0] = pr[U];
          pm[0] = pm[U];
#pragma unroll
          for (int u = 1; u <= U; ++u) {
            const uint32_t s = s0 + U + u, i = 32 * s + lane;
            px[u] = i < n ? X[i] : 0u;
            pr[u] = i < n ? R[i] : kNoRank;
            pm[u] = s < nseg ? mm[s] : 0u;
          }
        }
        uint32_t outv[U], nr[U], dst[U];
        bool emit[U], prb[U];
        ProbeReq q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t s = s0 + u, i = 32 * s + lane;
          emit[u] = prb[u] = false;
          if (s >= nseg) continue;
          const bool ap = (Aa[u] >> lane) & 1u;
          const bool consumed = lane == 0 ? ap_prev != 0 : ((Aa[u] >> (lane - 1)) & 1u);
          const bool em = i < n && !consumed;
          const unsigned Em = __ballot_sync(kFullMask, em);
          dst[u] = q0 + __popc(Em & lt_mask);
          q0 += __popc(Em);
          ap_prev = Aa[u] >> 31;
          const uint32_t x1 = lane_ahead(wx[u], wx[u + 1], lane, 1), r1 = lane_ahead(wr[u], wr[u + 1], lane, 1);
          const uint32_t x2 = lane_ahead(wx[u], wx[u + 1], lane, 2), r2 = lane_ahead(wr[u], wr[u + 1], lane, 2);
          const bool ap1 = bit_ahead(Aa[u], Aa[u + 1], lane, 1), ap2 = bit_ahead(Aa[u], Aa[u + 1], lane, 2);
          emit[u] = em;
          outv[u] = ap ? sp_merged<NARROW>(T, wr[u]) : wx[u];
          nr[u] = (ap || ap1) ? kNoRank : wr[u];  // unchanged pair: its rank stays
          if (!em || !(ap || ap1)) continue;
          uint32_t nt = 0;
          if (ap) {  // the next live token is at i + 2
            prb[u] = i + 2 < n;
            nt = ap2 ? sp_merged<NARROW>(T, r2) : x2;
          } else {  // pair i+1 merged: the next token is its merged token
            prb[u] = true;
            nt = sp_merged<NARROW>(T, r1);
          }
          (void)x1;
          if (prb[u]) probe_issue<NARROW>(q[u], T, outv[u], nt);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (!emit[u]) continue;
          X[dst[u]] = outv[u];
          R[dst[u]] = prb[u] ? probe_resolve<NARROW>(q[u], T) : nr[u];
        }
        __syncwarp();
      }
      n = q0;
    }
    __syncwarp();
  }
  // Result: lpo[start] = count (| unchanged), then the tokens in order.
  uint32_t* O = a.lpo + Rec.start;
  const bool unchanged = n == n0;
  if (lane == 0) {
    O[0] = n | (unchanged ? kUnchangedFlag : 0u);
    a.lrec[ridx].count = n;
    atomicAdd(&a.tile_count[Rec.start / kTile], n);
  }
  if (!unchanged)
    for (uint32_t i = lane; i < n; i += 32) O[1 + i] = X[i];
  __syncwarp();
}

// Persistent: each warp takes long pieces from the list by ticket.
template <bool NARROW>
__global__ void __launch_bounds__(kLpWarps * 32, 3) k_long_pieces(EncodeArgs a, DevTable T) {
  __shared__ uint32_t s_lut[256];
  extern __shared__ __align__(16) unsigned char s_lp[];
  const uint32_t count = static_cast<uint32_t>(min((uint64_t)a.counters[CNT_LONG], (uint64_t)a.long_cap));
  if (count == 0) return;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* smem = s_lp + size_t(wid) * lp_warp_bytes<NARROW>();
  for (;;) {
    uint32_t idx = 0;
    if (lane == 0) idx = atomicAdd(&a.counters[CNT_LP_NEXT], 1u);
    idx = __shfl_sync(kFullMask, idx, 0);
    if (idx >= count) return;
    run_piece<NARROW>(a, T, s_lut, a.long_idx[idx], smem, lane);
  }
}

// The super-pass engine, same ticketing (used unless a pass cap, a trace or
// caller tokens ask for the pass-by-pass engine above).
// Two instances: PIPE = pieces longer than kPipeMin positions (by default
// the shared working set's capacity), which stream from L2 and prefetch the
// next batch in every sweep; the other instance takes the rest and lists
// those for it. Separate kernels keep each one's register allocation free of
// the other's prefetch buffers, and give PIPE its own residency: no shared
// working set, so BBPE_PIPE_MINB CTAs per SM (5: 20 warps, 96 registers,
// phases B/C unrolled 2 segments deep); the shared-memory instance runs
// kLpMinBlocks (4: 16 warps, 128 registers, 8 KB slices).
#ifndef BBPE_PIPE_MIN_SEGS
#define BBPE_PIPE_MIN_SEGS 1
#endif
constexpr uint64_t kPipeMin = BBPE_PIPE_MIN_SEGS * (kLpSmemBytes / 8);
#ifndef BBPE_PIPE_MINB
#define BBPE_PIPE_MINB 5
#endif
template <bool NARROW, bool PIPE>
__global__ void __launch_bounds__(kLpWarps * 32, PIPE ? BBPE_PIPE_MINB : kLpMinBlocks) k_long_sp(EncodeArgs a, DevTable T) {
  __shared__ uint32_t s_lut[256];
  extern __shared__ __align__(16) unsigned char s_lp[];
  // PIPE = false: every long piece by ticket; the ones above kPipeMin are
  // listed for the PIPE instance, which runs after it on the same stream.
  const uint32_t count =
      static_cast<uint32_t>(min((uint64_t)a.counters[PIPE ? CNT_LONG2 : CNT_LONG], (uint64_t)a.long_cap));
  if (count == 0) return;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned char* smem = s_lp + size_t(wid) * lp_warp_bytes<NARROW>();
  for (;;) {
    uint32_t idx = 0;
    if (lane == 0) idx = atomicAdd(&a.counters[PIPE ? CNT_LP_NEXT2 : CNT_LP_NEXT], 1u);
    idx = __shfl_sync(kFullMask, idx, 0);
    if (idx >= count) return;
    const uint32_t ridx = PIPE ? a.long_idx2[idx] : a.long_idx[idx];
    if (!PIPE && a.lrec[ridx].len > kPipeMin) {
      if (lane == 0) a.long_idx2[atomicAdd(&a.counters[CNT_LONG2], 1u)] = ridx;
      continue;
    }
    run_piece_sp<NARROW, PIPE>(a, T, s_lut, ridx, smem, lane);
  }
}

// k_long_copy: warp per long piece (by ticket; a piece's tokens are written
// with 8 independent loads in flight per lane). The last warp to finish
// resets the counters k_gather left for it.
__global__ void __launch_bounds__(256, 4) k_long_copy(EncodeArgs a, DevTable T) {
  const uint32_t nrec = static_cast<uint32_t>(min((uint64_t)a.counters[CNT_LREC], a.lp_cap));
  if (a.counters[CNT_LREC] == 0) return;  // nothing to copy, nothing to reset
  __shared__ uint32_t s_lut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t* d2id = T.d2id;
  for (;;) {
    uint32_t r = 0;
    if (lane == 0) r = atomicAdd(&a.counters[CNT_LCOPY], 1u);
    r = __shfl_sync(kFullMask, r, 0);
    if (r >= nrec) break;
    const LongRec R = a.lrec[r];
    const uint32_t* src = a.lpo + R.start;
    const bool unchanged = (__ldcg(src) & kUnchangedFlag) != 0;
    uint32_t* dst = a.out_ids + R.out;
    const uint32_t cnt = R.count;
    constexpr int U = 8;
    for (uint32_t i0 = 0; i0 < cnt; i0 += 32 * U) {
      uint32_t v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + 32 * u + lane;
        v[u] = i < cnt ? (unchanged ? s_lut[__ldg(a.bytes + R.start + i)] : __ldcs(src + 1 + i)) : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = i0 + 32 * u + lane;
        if (i < cnt) dst[i] = d2id ? __ldg(d2id + v[u]) : v[u];
      }
    }
  }
  // Last warp out resets the counters (the next encode starts from zero).
  uint32_t done = 0;
  if (lane == 0) {
    __threadfence();
    done = atomicAdd(&a.counters[CNT_LDONE], 1u);
  }
  done = __shfl_sync(kFullMask, done, 0);
  if (done == gridDim.x * (blockDim.x / 32) - 1 && lane == 0) {
    a.counters[CNT_LREC] = 0;
    a.counters[CNT_LCOPY] = 0;
    a.counters[CNT_LDONE] = 0;
  }
}

}  // namespace

void launch_long_copy(const EncodeArgs& a, const DevTable& t, int grid, cudaStream_t stream) {
  k_long_copy<<<grid, 256, 0, stream>>>(a, t);
}

size_t long_pieces_smem(bool narrow) {
  return size_t(kLpWarps) * (narrow ? lp_warp_bytes<true>() : lp_warp_bytes<false>());
}

// Resident CTAs per SM of the PIPE instance (no shared working set: its
// pieces stream from the global scratch, so only registers bound it).
static int g_pipe_per_sm = 0, g_sm_count = 0;

int long_pieces_grid(int device, int sm_count) {
  (void)device;
  const size_t sn = long_pieces_smem(true), sw = long_pieces_smem(false);
  cudaFuncSetAttribute(k_long_pieces<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sn));
  cudaFuncSetAttribute(k_long_pieces<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sw));
  cudaFuncSetAttribute(k_long_sp<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sn));
  cudaFuncSetAttribute(k_long_sp<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sw));
  cudaFuncSetAttribute(k_long_sp<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sn));
  cudaFuncSetAttribute(k_long_sp<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sw));
  int per_sm = 0, pn = 0, pw = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_long_sp<true, false>, kLpWarps * 32, sn);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pn, k_long_sp<true, true>, kLpWarps * 32, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pw, k_long_sp<false, true>, kLpWarps * 32, 0);
  per_sm = per_sm > 0 ? per_sm : 1;
  g_pipe_per_sm = std::max(1, std::min(pn, pw));
  g_sm_count = sm_count;
  return sm_count * per_sm;
}

int launch_long_pieces(const EncodeArgs& a, const DevTable& t, int grid, cudaStream_t stream) {
  const bool by_pass = a.trace || a.max_passes > 0 || a.tokens_input;  // PassTrace, MaxPassesError
  const size_t sm = long_pieces_smem(t.key32 != 0);
  if (by_pass) {
    if (t.key32) k_long_pieces<true><<<grid, kLpWarps * 32, sm, stream>>>(a, t);
    else k_long_pieces<false><<<grid, kLpWarps * 32, sm, stream>>>(a, t);
    return 1;
  }
  // The PIPE instance: same SMs, its own residency (grid = SMs x its CTAs per SM).
  const int pgrid = g_sm_count > 0 ? g_sm_count * g_pipe_per_sm : grid;
  if (t.key32) {  // 16-bit ids and ranks
    k_long_sp<true, false><<<grid, kLpWarps * 32, sm, stream>>>(a, t);
    k_long_sp<true, true><<<pgrid, kLpWarps * 32, 0, stream>>>(a, t);
  } else {
    k_long_sp<false, false><<<grid, kLpWarps * 32, sm, stream>>>(a, t);
    k_long_sp<false, true><<<pgrid, kLpWarps * 32, 0, stream>>>(a, t);
  }
  return 2;
}

}  // namespace bbpe
