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
        const unsigned Mb = __ballot_sync(kFullMask, ((L >> lane) & 1u) && PT::rank(e) == m);
        // Left-greedy in live order (fill_merge_flags 103-128).
        uint32_t merged = 0, kill = 0;
        int64_t out_kill = -1;
        for (unsigned mm = Mb; mm; mm &= mm - 1) {
          const uint32_t b = __ffs(mm) - 1;
          if ((kill >> b) & 1u) continue;  // consumed by the previous merge of the run
          merged |= 1u << b;
          const uint32_t nb = L & above(b);
          if (nb) kill |= 1u << (__ffs(nb) - 1);
          else out_kill = first_live_from(V, s + 1);  // the pair's right token is in a later segment
        }
        if (!merged) continue;
        merges += __popc(merged);
        const uint32_t Ln = L & ~kill;
        const bool me = (merged >> lane) & 1u;
        // The left neighbour of a merged token: its pair changed.
        const uint32_t nbx = Ln & above(lane);
        const bool left_of_merge = ((Ln >> lane) & 1u) && !me && nbx && ((merged >> (__ffs(nbx) - 1)) & 1u);
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

int long_pieces_grid(int device, int sm_count) {
  (void)device;
  const size_t sn = long_pieces_smem(true), sw = long_pieces_smem(false);
  cudaFuncSetAttribute(k_long_pieces<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sn));
  cudaFuncSetAttribute(k_long_pieces<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sw));
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_long_pieces<true>, kLpWarps * 32, sn);
  return sm_count * (per_sm > 0 ? per_sm : 1);
}

void launch_long_pieces(const EncodeArgs& a, const DevTable& t, int grid, cudaStream_t stream) {
  if (t.key32)  // 16-bit ids and ranks: the u32 position record
    k_long_pieces<true><<<grid, kLpWarps * 32, long_pieces_smem(true), stream>>>(a, t);
  else
    k_long_pieces<false><<<grid, kLpWarps * 32, long_pieces_smem(false), stream>>>(a, t);
}

}  // namespace bbpe
