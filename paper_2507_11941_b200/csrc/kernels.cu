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
//   k_tile_first  : first row of each tile, row-start bitmap, offsets check/rebase
//   k_pieces      : warp per tile: boundaries, piece list, single bytes and
//                   piece-memo hits staged; merge / long records for the rest
//   k_dedup       : (large batches) one owner per distinct merge piece
//   k_merge       : lane-per-piece pass loops over the merge records (owners)
//   k_refs        : (large batches) references copy their owner's tokens
//   k_long_pieces : CTA-per-piece pass loop over the long pieces k_pieces found
//                   (the paper's block engine; every row under BBPE_ENGINE_BLOCK)
//   k_tile_scan   : tile token counts -> tile bases (decoupled look-back)
//   k_gather      : staging compaction -> CSR ids + row offsets
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"
#include "pretok.cuh"
#include "probe.cuh"

namespace bbpe {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPrefix = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

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
// k_tile_first: F(t) = min{ s : offsets[s] >= t*kTile }, t in [0, num_tiles),
// and the row-start bitmap (one bit per input byte, zeroed by the host), which
// k_pieces copies into shared memory with its window.
// Row s owns tiles t with offsets[s-1] < t*kTile <= offsets[s].
__global__ void k_tile_first(EncodeArgs a) {
  uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (s > a.n_rows) return;
  const uint64_t* src = a.offsets_raw ? a.offsets_raw : a.offsets;
  uint64_t o = src[s] - a.offsets_base;
  const uint64_t prev = s == 0 ? 0 : src[s - 1] - a.offsets_base;
  if (o < prev || o > a.total || (s == a.n_rows && o != a.total) || (s == 0 && o != 0)) {
    // Offsets must be non-decreasing (the host raises UsageError); clamp so
    // that every kernel stays inside its buffers meanwhile.
    atomicMin(reinterpret_cast<unsigned long long*>(&a.err[ERR_BAD_OFFSETS]), (unsigned long long)s);
    o = min(max(o, prev), a.total);
  }
  uint64_t hi = o / kTile;
  uint64_t lo = (s == 0) ? 0 : min(prev, a.total) / kTile + 1;
  if (s == 0) hi = 0;  // offsets[0] == 0
  for (uint64_t t = lo; t <= hi && t < a.num_tiles; ++t) a.tile_first[t] = s;
  if (s == 0) {
    a.tile_first[a.num_tiles] = a.n_rows + 1;
    if (a.pstats) atomicAdd(reinterpret_cast<unsigned long long*>(a.pstats + PST_BYTES), (unsigned long long)a.total);
  }
  // A row starting at `total` has no bytes: no bit (it would land past the
  // last tile, where k_gather never clears it).
  if (a.rowbits && s < a.n_rows && o < a.total) atomicOr(&a.rowbits[o >> 5], 1u << (o & 31));
  if (a.offsets_raw) a.offsets_w[s] = o;  // the rebased copy the other kernels read
}

// ---------------------------------------------------------------------------
// Asynchronous global -> shared copies (LDGSTS), zero-filled past src_bytes.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint32_t src_bytes) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Junction test on the transposed bitmap: bit (c << 8 | a) for the bigram (a, c).
__device__ __forceinline__ bool is_junction_t(const uint32_t* jt, uint32_t a, uint32_t c) {
  const uint32_t bit = (c << 8) | a;
  return (jt[((bit >> 5) ^ bit) & 0x7FF] >> (bit & 31)) & 1u;  // swizzled words (table.cpp)
}

// Per-warp shared state of k_pieces (double-buffered input window).
struct PieceSmem {
  uint4 win[2][kWinVec];          // bytes [b0-16, b0+kTile+32): position q at byte q+16
  uint32_t rb[2][kRowWords];      // row-start bits of positions [0, 32*kRowWords)
  uint32_t cb[2][kRowWords];      // pattern mode: chunk-start bits, same positions
  uint32_t bd[kTile / 32 + 1];    // piece-start bits of positions [0, min(kTile, limit)); [16] = 0
  uint16_t wpre[kTile / 32 + 1];  // pieces starting in words < w
  uint16_t plist[kTile + 1];      // piece starts in order, then the end of the last piece
  uint16_t cnt[kTile + 1];        // staging slots before piece k (k <= npieces)
  uint16_t lk[kTile / (kLmax + 1) + 2];  // long pieces (piece indices), in order
};

// Issues the window + row-bit copies of `tile` into buffer `buf` (one group).
__device__ __forceinline__ void issue_window(PieceSmem& S, int buf, const EncodeArgs& a, uint64_t tile,
                                             int lane) {
  const int64_t g0 = int64_t(tile) * kTile - 16;
#pragma unroll
  for (int i = lane; i < kWinVec; i += 32) {
    const int64_t pos = g0 + 16 * i;
    const int64_t rem = int64_t(a.total) - pos;
    const uint32_t nb = pos < 0 ? 0u : uint32_t(rem >= 16 ? 16 : (rem > 0 ? rem : 0));
    cp_async16(&S.win[buf][i], nb ? static_cast<const void*>(a.bytes + pos) : a.bytes, nb);
  }
  if (lane < kRowWords / 4)
    cp_async16(&S.rb[buf][4 * lane], a.rowbits + tile * (kTile / 32) + 4 * lane, 16);
  else if (a.chunkbits && lane < kRowWords / 2)
    cp_async16(&S.cb[buf][4 * (lane - kRowWords / 4)], a.chunkbits + tile * (kTile / 32) + 4 * (lane - kRowWords / 4),
               16);
}

// Window load without cp.async (input pointer not 16-byte aligned): plain
// byte loads into the same layout.
__device__ __noinline__ void load_window_slow(PieceSmem& S, int buf, const uint8_t* bytes, uint64_t total,
                                              const uint32_t* rowbits, const uint32_t* chunkbits, uint64_t tile,
                                              int lane) {
  const int64_t g0 = int64_t(tile) * kTile - 16;
  uint8_t* w = reinterpret_cast<uint8_t*>(S.win[buf]);
  for (int i = lane; i < kWinVec * 16; i += 32) {
    const int64_t pos = g0 + i;
    w[i] = (pos >= 0 && pos < int64_t(total)) ? bytes[pos] : 0;
  }
  for (int i = lane; i < kRowWords; i += 32) {
    S.rb[buf][i] = rowbits[tile * (kTile / 32) + i];
    if (chunkbits) S.cb[buf][i] = chunkbits[tile * (kTile / 32) + i];
  }
}

// Length of a long piece starting at abs (warp-cooperative, rare path).
// In pattern mode a piece also ends at a chunk start (chunkbits).
__device__ __noinline__ uint64_t long_piece_length(const uint64_t* offsets, uint64_t n_rows, const uint8_t* bytes,
                                                   const uint32_t* jt, const uint32_t* chunkbits, uint64_t abs,
                                                   int lane) {
  uint64_t row_end = 0;
  if (lane == 0) {
    uint64_t lo = 0, hi = n_rows;  // max s with offsets[s] <= abs
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) >> 1;
      if (offsets[mid] <= abs) lo = mid; else hi = mid - 1;
    }
    row_end = max(offsets[lo + 1], abs + kLmax + 1);  // (max: guards bad offsets)
  }
  row_end = __shfl_sync(kFull, row_end, 0);
  for (uint64_t x = abs + kLmax + 1; x < row_end; x += 32) {
    const uint64_t y = x + lane;
    const bool bnd =
        y < row_end && (!is_junction_t(jt, bytes[y - 1], bytes[y]) || (chunkbits && ((chunkbits[y >> 5] >> (y & 31)) & 1u)));
    const unsigned bm = __ballot_sync(kFull, bnd);
    if (bm) return x + __ffs(bm) - 1 - abs;
  }
  return row_end - abs;
}

// Whole-piece memo lookup: the piece's bytes (window byte index `start`,
// 2..kMemoMaxLen bytes) as 5 zero-padded words, hashed, then linear probing
// over 32-byte entries. Exact: an entry holds this engine's own encoding of
// the same bytes, computed from the table alone at upload time.
__device__ __forceinline__ int memo_match(const ulonglong2 lo, const ulonglong2 hi, const uint32_t* w,
                                          int len, uint32_t& r0, uint32_t& r1, uint32_t& nres) {
  const uint32_t meta = uint32_t(hi.x >> 32), elen = meta & 0xFF;
  // Branch-free compare: with a short-circuit the compiler sinks the load of
  // `lo` behind the length test, i.e. a second dependent L2 round trip.
  const bool hit = (elen == uint32_t(len)) & (lo.x == (uint64_t(w[1]) << 32 | w[0])) &
                   (lo.y == (uint64_t(w[3]) << 32 | w[2])) & (uint32_t(hi.x) == w[4]);
  if (hit) {
    nres = (meta >> 8) & 0xFF;
    r0 = uint32_t(hi.y);
    r1 = uint32_t(hi.y >> 32);
    return 1;
  }
  return elen == 0 ? 0 : -1;  // empty slot: miss; occupied by another piece: keep probing
}

// Everything by value: a pointer would force the caller's key into local memory.
struct MemoHit {
  uint32_t r0, r1, nres;  // nres 0: miss
};
__device__ __noinline__ MemoHit memo_overflow(const MemoEntry* memo, uint64_t mask, uint32_t w0, uint32_t w1,
                                              uint32_t w2, uint32_t w3, uint32_t w4, int len, uint64_t b) {
  const uint32_t w[5] = {w0, w1, w2, w3, w4};
  for (;;) {
    b = (b + 1) & mask;
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(memo + b);
    MemoHit h{0, 0, 0};
    const int m = memo_match(__ldg(p), __ldg(p + 1), w, len, h.r0, h.r1, h.nres);
    if (m == 0) return MemoHit{0, 0, 0};
    if (m == 1) return h;
  }
}

// Byte masks of the 5 key words for each piece length (shared memory,
// s_mask[32 * i + len]: lanes reading word i for any mix of lengths hit
// distinct banks or broadcast), built once per CTA.
__device__ __forceinline__ void build_mask_table(uint32_t* s_mask) {
  for (int k = threadIdx.x; k < 5 * 32; k += blockDim.x) {
    const int len = k & 31, wi = k >> 5;
    const int nb = len - 4 * wi;
    s_mask[k] = nb >= 4 ? ~0u : (nb <= 0 ? 0u : (1u << (8 * nb)) - 1u);
  }
}

__device__ __forceinline__ bool memo_lookup(const DevTable& T, const uint32_t* ww, const uint32_t* s_mask,
                                            int start, int len, uint32_t& r0, uint32_t& r1, uint32_t& nres) {
  const int a = start >> 2;
  const uint32_t sh = uint32_t(start & 3) * 8;
  const uint32_t mk[5] = {s_mask[len], s_mask[32 + len], s_mask[64 + len], s_mask[96 + len], s_mask[128 + len]};
  uint32_t x[6], w[5];
#pragma unroll
  for (int i = 0; i < 6; ++i) x[i] = ww[a + i];
#pragma unroll
  for (int i = 0; i < 5; ++i) w[i] = __funnelshift_r(x[i], x[i + 1], sh) & mk[i];
  const uint64_t b = memo_hash(w, uint32_t(len)) & T.memo_mask;
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.memo + b);
  const int m = memo_match(__ldg(p), __ldg(p + 1), w, len, r0, r1, nres);
  if (m >= 0) return m == 1;
  const MemoHit h = memo_overflow(T.memo, T.memo_mask, w[0], w[1], w[2], w[3], w[4], len, b);
  r0 = h.r0;
  r1 = h.r1;
  nres = h.nres;
  return nres != 0;
}

// 128-bit compare-and-swap (sm_90+ atom.cas.b128); returns the old value.
__device__ __forceinline__ ulonglong2 cas128(ulonglong2* p, ulonglong2 cmp, ulonglong2 val) {
  ulonglong2 old;
  asm volatile(
      "{ .reg .b128 d, c, v; mov.b128 c, {%2, %3}; mov.b128 v, {%4, %5};\n"
      "  atom.global.cas.b128 d, [%6], c, v; mov.b128 {%0, %1}, d; }\n"
      : "=l"(old.x), "=l"(old.y)
      : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(p)
      : "memory");
  return old;
}

// Bytes [p, p + 8k) of the input as k little-endian u64 words (k <= 3),
// from the aligned 8-byte words that cover them: independent loads in flight
// together, instead of one dependent byte load per position. Words wholly
// inside [bytes, bytes + total) only; the rare span whose last word would
// reach past the end (the input's final bytes) is read byte by byte. Bytes at
// or past `total` read as 0 on that path; callers use the first len bytes.
template <int K>
__device__ __forceinline__ void ld_span(const uint8_t* __restrict__ bytes, uint64_t total, uint64_t p, uint64_t (&v)[K]) {
  const uintptr_t addr = reinterpret_cast<uintptr_t>(bytes + p);
  const uint64_t* w = reinterpret_cast<const uint64_t*>(addr & ~uintptr_t(7));
  const int sh = int(addr & 7) * 8;
  if (reinterpret_cast<uintptr_t>(w + K + 1) <= reinterpret_cast<uintptr_t>(bytes + total)) {
    uint64_t x[K + 1];
#pragma unroll
    for (int k = 0; k <= K; ++k) x[k] = __ldg(w + k);
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = sh ? (x[k] >> sh) | (x[k + 1] << (64 - sh)) : x[k];
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      v[k] = 0;
      for (int j = 0; j < 8; ++j)
        if (p + 8 * k + j < total) v[k] |= uint64_t(__ldg(bytes + p + 8 * k + j)) << (8 * j);
    }
  }
}

// Within-call dedupe of merge pieces: finds or claims the slot of `key`.
// Returns the slot (the caller owns it: its merge passes run), the slot with
// bit 63 set (another piece with the same bytes owns it: copy its result),
// or ~0 after BBPE_DEDUP_PROBES probes (no dedupe for this piece).
__device__ __forceinline__ uint64_t dedup_claim(ulonglong2* dkey, uint64_t dmask, ulonglong2 key) {
  uint64_t h = (key.x * 0x9E3779B97F4A7C15ull) ^ (key.y * 0xC2B2AE3D27D4EB4Full);
  h ^= h >> 29;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 32;
  uint64_t s = h & dmask;
  for (int i = 0; i < BBPE_DEDUP_PROBES; ++i) {
    ulonglong2 cur = __ldcg(dkey + s);
    if (cur.x == 0 && cur.y == 0) {
      cur = cas128(dkey + s, make_ulonglong2(0, 0), key);
      if (cur.x == 0 && cur.y == 0) return s;
    }
    if (cur.x == key.x && cur.y == key.y) return s | (1ull << 63);
    s = (s + 1) & dmask;
  }
  return ~0ull;
}

#ifndef BBPE_PIECES_MINB
#define BBPE_PIECES_MINB 4
#endif
#ifndef BBPE_PIECES_PER_LANE
#define BBPE_PIECES_PER_LANE 2
#endif
// k_pieces: warp per 512-byte tile, persistent over tiles by ticket, the next
// tile's window and row bits in flight (cp.async) while the current one is
// processed.
//  (1) piece-start bits: lane l tests positions [16l, 16l+16) against the
//      junction bitmap (a position is a hard boundary when its bigram is not a
//      merge junction), ORs in row starts; the end of the last
//      piece comes from a 32-position tail test.
//  (2) piece list (start positions, in order).
//  (3) resolve 32 pieces per round: single bytes and piece-memo hits are
//      final and go to the tile's staging slots; other pieces of <= kLmax
//      bytes reserve `len` slots and become merge records (k_merge); longer
//      pieces become long records (k_long_pieces).
//  (4) row offsets relative to the tile (staging slot | long pieces before).
__global__ void __launch_bounds__(kWarpsPerCta * 32, BBPE_PIECES_MINB) k_pieces(EncodeArgs a, DevTable T) {
  __shared__ uint32_t s_jt[2048];
  __shared__ uint32_t s_lo[256];
  static_assert(kMemoMaxLen < 32, "mask table columns");
  __shared__ __align__(16) uint32_t s_mask[5 * 32];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s_jt[i] = T.junction_t[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lo[i] = T.lut_out[i];
  build_mask_table(s_mask);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  PieceSmem& S = reinterpret_cast<PieceSmem*>(s_dyn)[wid];
  const bool async = a.bytes_aligned != 0;
  const bool chk = T.full_lut == 0;

  // Tiles by ticket, kTilesPerTicket consecutive tiles per ticket (in input
  // order); the next ticket is taken a whole group ahead.
  // (one tile per ticket when there are few tiles per warp: keep every warp busy)
  const uint64_t G = a.num_tiles >= uint64_t(gridDim.x) * kWarpsPerCta * 16 ? kTilesPerTicket : 1;
  uint32_t tk = 0;
  if (lane == 0) tk = atomicAdd(&a.counters[CNT_TILE_TICKET], 1u);
  uint64_t tile = uint64_t(__shfl_sync(kFull, tk, 0)) * G;
  if (tile >= a.num_tiles) return;
  if (async) issue_window(S, 0, a, tile, lane);
  cp_async_commit();
  if (lane == 0) tk = atomicAdd(&a.counters[CNT_TILE_TICKET], 1u);
  uint64_t nxt = tile + 1;
  if (G == 1) {
    nxt = __shfl_sync(kFull, tk, 0);
    if (lane == 0) tk = atomicAdd(&a.counters[CNT_TILE_TICKET], 1u);
  }
  uint64_t f = lane < 2 ? a.tile_first[tile + lane] : 0;
  int buf = 0;
  uint64_t mbase = 0;
  uint32_t mleft = 0;
  uint32_t st_pieces = 0, st_merge = 0, st_long = 0, st_lbytes = 0;  // piece statistics (warp-uniform)

  while (tile < a.num_tiles) {
    // Prefetch: the next tile's window and row range.
    if (async && nxt < a.num_tiles) issue_window(S, buf ^ 1, a, nxt, lane);
    cp_async_commit();
    const uint64_t nf = (lane < 2 && nxt < a.num_tiles) ? a.tile_first[nxt + lane] : 0;
    if (async) {
      cp_async_wait<1>();
    } else {
      load_window_slow(S, buf, a.bytes, a.total, a.rowbits, a.chunkbits, tile, lane);
    }
    __syncwarp();

    const uint64_t b0 = tile * kTile;
    const int64_t limit = int64_t(a.total - b0);  // positions >= limit are past the input
    const uint64_t s0 = __shfl_sync(kFull, f, 0), s1 = __shfl_sync(kFull, f, 1);
    const uint32_t* ww = reinterpret_cast<const uint32_t*>(S.win[buf]);
    const uint8_t* wb = reinterpret_cast<const uint8_t*>(S.win[buf]);
    // Row offsets of the rows starting in this tile: loads issued now, used in (4).
    uint64_t my_off = 0;
    const uint64_t my_s = s0 + lane;
    if (my_s < s1 && my_s <= a.n_rows) my_off = a.offsets[my_s];

    // (1) Piece-start bits, 16 positions per lane: bigram (q-1, q) as the
    // 16-bit little-endian pair at window byte q+15.
    {
      const uint32_t y0 = ww[4 * lane + 3];
      const uint4 yv = S.win[buf][lane + 1];
      const uint32_t y[5] = {y0, yv.x, yv.y, yv.z, yv.w};
      uint32_t jm = 0;
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        // Pairs j and j+1 at once: V = a1 | c1 << 8 | a2 << 16 | c2 << 24
        // (bytes j+3, j+4, j+4, j+5), both swizzled word indices from one
        // shift + mask (the shift's bleed from the upper half lands in bits
        // 11-15 of the lower half, which the mask clears).
        const int r = j + 3, b = r & 3;
        const uint32_t V = __byte_perm(y[r >> 2], y[(r >> 2) + 1],
                                       uint32_t(b | ((b + 1) << 4) | ((b + 1) << 8) | ((b + 2) << 12)));
        const uint32_t idx = ((V >> 5) ^ V) & 0x07FF07FFu;
        const uint32_t w1 = s_jt[idx & 0xFFFFu], w2 = s_jt[idx >> 16];
        jm |= ((__funnelshift_r(w1, w1, V) & 1u) << j) | ((__funnelshift_r(w2, w2, V >> 16) & 1u) << (j + 1));
      }
      uint32_t m = (~jm) & 0xFFFFu;  // not a junction: boundary
      if (chk) {
        uint32_t bad = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int q = 16 * lane + j;
          const uint32_t byte = (y[(j + 4) >> 2] >> (8 * ((j + 4) & 3))) & 0xFFu;
          if (q < limit && s_lo[byte] == kInvalidToken && bad == 0xFFFFFFFFu) bad = uint32_t(q);
        }
        bad = __reduce_min_sync(kFull, bad);
        if (bad != 0xFFFFFFFFu && lane == 0)
          atomicMin(reinterpret_cast<unsigned long long*>(&a.err[ERR_BAD_BYTE_POS]),
                    (unsigned long long)(b0 + bad));
      }
      const uint32_t other = __shfl_down_sync(kFull, m, 1);
      if ((lane & 1) == 0) {
        uint32_t wbits = m | (other << 16) | S.rb[buf][lane >> 1] | (a.chunkbits ? S.cb[buf][lane >> 1] : 0u);
        const int64_t q0 = 16 * lane;  // word (lane/2) covers [q0, q0 + 32)
        if (q0 + 32 > limit) wbits &= limit <= q0 ? 0u : ((1u << (limit - q0)) - 1u);
        S.bd[lane >> 1] = wbits;
      }
    }
    // Tail: first cut in [kTile, kTile + 32) ends the tile's last piece.
    int last_end;
    {
      const int p = kTile + lane;
      const uint32_t pa = wb[p + 15], pc = wb[p + 16];
      const bool cut = p >= limit || (((S.rb[buf][p >> 5] | (a.chunkbits ? S.cb[buf][p >> 5] : 0u)) >> (p & 31)) & 1u) ||
                       !is_junction_t(s_jt, pa, pc);
      const unsigned cm = __ballot_sync(kFull, cut);
      last_end = cm ? kTile + __ffs(cm) - 1 : kTile + 32;
      if (limit < kTile) last_end = int(limit);
    }
    if (lane == 0) S.bd[kTile / 32] = 0;
    __syncwarp();

    // (2) Piece list: two lanes per boundary word (16 positions each).
    static_assert(kTile / 32 * 2 == 32, "two lanes per boundary word");
    int npieces;
    {
      const uint32_t m = (S.bd[lane >> 1] >> (16 * (lane & 1))) & 0xFFFFu;
      const uint32_t c = __popc(m);
      const uint32_t inc = warp_incl_sum(c, lane);
      const uint32_t tot = __shfl_sync(kFull, inc, 31);
      if ((lane & 1) == 0) S.wpre[lane >> 1] = static_cast<uint16_t>(inc - c);
      if (lane == 0) S.wpre[kTile / 32] = static_cast<uint16_t>(tot);
      int pos = int(inc - c);
      uint32_t mm = m;
      while (mm) {
        S.plist[pos++] = static_cast<uint16_t>(16 * lane + __ffs(mm) - 1);
        mm &= mm - 1;
      }
      npieces = int(__shfl_sync(kFull, inc, 31));
      if (lane == 0) S.plist[npieces] = static_cast<uint16_t>(last_end);
    }
    __syncwarp();

    // (3) Resolve 64 pieces per round: lane l takes the adjacent pieces
    // k0 + 2l and k0 + 2l + 1 (two memo lookups in flight per lane, one slot
    // scan per 64 pieces).
    constexpr int PPL = BBPE_PIECES_PER_LANE;
    uint32_t* stage = a.staging + tile * kStage;
    uint32_t run = 0, nlong = 0;
    for (int k0 = 0; k0 < npieces; k0 += 32 * PPL) {
      int len[PPL], q[PPL];
      uint32_t c[PPL], r0[PPL], r1[PPL];
      bool merge[PPL], lg[PPL];
#pragma unroll
      for (int u = 0; u < PPL; ++u) {
        const int k = k0 + PPL * lane + u;
        len[u] = 0;
        q[u] = 0;
        c[u] = r0[u] = r1[u] = 0;
        merge[u] = lg[u] = false;
        if (k < npieces) {
          q[u] = S.plist[k];
          len[u] = S.plist[k + 1] - q[u];
          if (len[u] > kLmax) {
            lg[u] = true;  // long: k_long_pieces, no staging slots
          } else if (len[u] == 1 && !a.use_memo) {  // (with the memo, single bytes are entries)
            c[u] = 1;
            r0[u] = s_lo[wb[q[u] + 16]];
          } else {
            uint32_t nres = 0;
            if (a.use_memo && len[u] <= kMemoMaxLen &&
                memo_lookup(T, ww, s_mask, q[u] + 16, len[u], r0[u], r1[u], nres)) {
              c[u] = nres;
            } else {
              merge[u] = true;  // k_merge fills the `len` reserved slots
              c[u] = uint32_t(len[u]);
            }
          }
        }
      }
      uint32_t cl = 0;
#pragma unroll
      for (int u = 0; u < PPL; ++u) cl += c[u];
      const uint32_t inc = warp_incl_sum(cl, lane);
      uint32_t slot[PPL];
      unsigned mmu[PPL], lmu[PPL], mm_any = 0, lm_any = 0;
#pragma unroll
      for (int u = 0; u < PPL; ++u) {
        slot[u] = (u ? slot[u - 1] + c[u - 1] : run + inc - cl);
        mmu[u] = __ballot_sync(kFull, merge[u]);
        lmu[u] = __ballot_sync(kFull, lg[u]);
        mm_any |= mmu[u];
        lm_any |= lmu[u];
        st_merge += __popc(mmu[u]);
        st_long += __popc(lmu[u]);
      }
#pragma unroll
      for (int u = 0; u < PPL; ++u) {
        const int k = k0 + PPL * lane + u;
        if (k < npieces) S.cnt[k] = static_cast<uint16_t>(slot[u]);
        if (!merge[u] && c[u]) {
          stage[slot[u]] = r0[u];
          if (c[u] > 1) stage[slot[u] + 1] = r1[u];
        }
      }
      if (mm_any) {
        uint32_t nm = 0;
#pragma unroll
        for (int u = 0; u < PPL; ++u) nm += __popc(mmu[u]);
        if (nm > mleft) {  // new chunk of merge records; the old chunk's tail becomes holes
          for (uint32_t i = lane; i < mleft; i += 32)
            if (mbase + i < a.mrec_cap) a.mrec[mbase + i] = make_ulonglong2(~0ull, 0);
          uint32_t cc = 0;
          if (lane == 0) cc = atomicAdd(&a.counters[CNT_MREC], uint32_t(kMrecChunk));
          mbase = __shfl_sync(kFull, cc, 0);
          mleft = kMrecChunk;
        }
        uint32_t before_u = 0;  // merges of the earlier piece positions, all lanes
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          if (merge[u]) {
            // The piece's first 8 bytes ride in its record (k_merge needs no
            // dependent load for pieces of <= 8 bytes); window byte q+16.
            const int st = q[u] + 16, wa = st >> 2;
            const uint32_t sh = uint32_t(st & 3) * 8;
            const uint32_t x0 = ww[wa], x1 = ww[wa + 1], x2 = ww[wa + 2];
            const uint64_t b8 = uint64_t(__funnelshift_r(x0, x1, sh)) | (uint64_t(__funnelshift_r(x1, x2, sh)) << 32);
            const uint64_t at = mbase + before_u + __popc(mmu[u] & lanemask_lt(lane));
            if (at < a.mrec_cap) a.mrec[at] = make_ulonglong2(pack_mrec(b0 + q[u], slot[u], uint32_t(len[u])), b8);
          }
          before_u += __popc(mmu[u]);
        }
        mbase += nm;
        mleft -= nm;
      }
      if (lm_any) {  // (rare) long pieces, listed in piece order
        uint32_t before = nlong;
#pragma unroll
        for (int u = 0; u < PPL; ++u) before += __popc(lmu[u] & lanemask_lt(lane));
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
          if (lg[u]) S.lk[before++] = static_cast<uint16_t>(k0 + PPL * lane + u);
          nlong += __popc(lmu[u]);
        }
      }
      run += __shfl_sync(kFull, inc, 31);
    }
    if (lane == 0) S.cnt[npieces] = static_cast<uint16_t>(run);
    __syncwarp();

    // Long pieces (rare): full length to the next hard boundary or row end.
    uint64_t lfirst = 0;
    if (nlong) {
      uint64_t l0 = 0, x0 = 0;
      if (lane == 0) {
        l0 = atomicAdd(&a.counters[CNT_LREC], nlong);
        x0 = atomicAdd(&a.counters[CNT_LONG], nlong);
      }
      lfirst = __shfl_sync(kFull, l0, 0);
      x0 = __shfl_sync(kFull, x0, 0);
      for (uint32_t i = 0; i < nlong; ++i) {
        const int k = S.lk[i];
        const uint64_t abs = b0 + S.plist[k];
        const uint64_t len = long_piece_length(a.offsets, a.n_rows, a.bytes, s_jt, a.chunkbits, abs, lane);
        st_lbytes += uint32_t(len);
        if (lane == 0) {
          if (lfirst + i < a.lp_cap) a.lrec[lfirst + i] = LongRec{abs, len, 0, S.cnt[k], 0u, 0};
          if (x0 + i < a.long_cap) a.long_idx[x0 + i] = uint32_t(lfirst + i);
        }
      }
    }
    st_pieces += uint32_t(npieces);
    if (lane == 0) {
      a.tile_lrec[tile] = nlong ? ((lfirst << 24) | nlong) : 0;
      a.tile_count[tile] = run;
      a.tile_slots[tile] = run;
    }
    // (4) Row offsets relative to the tile: staging slots before the row's
    // first piece (low 40 bits) and long pieces before it (above).
    for (uint64_t s = my_s, o = my_off;;) {
      if (!(s < s1 && s <= a.n_rows)) break;
      const int r = int(min(max(o, b0), b0 + kTile) - b0);  // in [0, kTile] (clamped: bad offsets)
      const int w = r >> 5;
      const int kk = S.wpre[w] + __popc(S.bd[w] & ((1u << (r & 31)) - 1u));
      uint64_t lb = 0;
      while (lb < nlong && S.lk[lb] < kk) ++lb;
      a.out_offsets[s] = uint64_t(S.cnt[kk]) | (lb << 40);
      s += 32;
      if (s < s1 && s <= a.n_rows) o = a.offsets[s];
    }
    __syncwarp();
    tile = nxt;
    if (G > 1 && (nxt + 1) % G) {
      nxt = nxt + 1;
    } else {  // next group: the ticket taken a group ago, and the one after it
      nxt = uint64_t(__shfl_sync(kFull, tk, 0)) * G;
      if (lane == 0) tk = atomicAdd(&a.counters[CNT_TILE_TICKET], 1u);
    }
    f = nf;
    buf ^= 1;
  }
  cp_async_wait<0>();
  for (uint32_t i = lane; i < mleft; i += 32)
    if (mbase + i < a.mrec_cap) a.mrec[mbase + i] = make_ulonglong2(~0ull, 0);
  if (a.pstats && lane == 0) {  // piece statistics: one set of atomics per warp
    auto add = [&](int k, uint64_t v) {
      if (v) atomicAdd(reinterpret_cast<unsigned long long*>(a.pstats + k), (unsigned long long)v);
    };
    add(PST_PIECES, st_pieces);
    add(PST_MEMO, st_pieces - st_merge - st_long);
    add(PST_MERGE, st_merge);
    add(PST_LONG, st_long);
    add(PST_LONG_BYTES, st_lbytes);
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
  uint32_t rnk[kLmax][32];  // rk of pair (i, i+1) once resolved
  uint8_t pq[kLmax][32];   // pairs waiting for a probe (positions)
};

// k_merge: every pass of the reference loop (block_engine.hpp:286-307) for a
// piece held in one lane's column of the [slot][lane] arrays:
//   probe : resolve the pending pairs, four bucket loads in flight, folding
//           their ranks into the running minimum m;
//   stop  : m == NONE (no pair in the table, block_engine.hpp:288-289);
//   sweep : compact in place -- a pair at rank m merges unless its left token
//           was just consumed (flags[i+1] = (ranks[i] == m && !flags[i]),
//           103-128) into M = r2m[m] (ranks are unique per pair, so this is
//           the merged id compact_into looks up, 173); pairs touching a merged
//           token become pending, the others keep their rank (cached ranks
//           are exact: a pair's rank depends on its two tokens only) and
//           give the next pass's minimum.
// Lanes refill from the merge-record list as their pieces finish.
#ifndef BBPE_MERGE_MINB
#define BBPE_MERGE_MINB 3
#endif
#ifndef BBPE_MERGE_PROBES
#define BBPE_MERGE_PROBES 3
#endif
template <typename Tk>
__global__ void __launch_bounds__(kWarpsPerCta * 32, BBPE_MERGE_MINB) k_merge(EncodeArgs a, DevTable T) {
  constexpr bool K32 = sizeof(Tk) == 2;  // narrow: 32-bit keys, merged id in the slot
  constexpr uint32_t NONE = kNoRank;
  __shared__ uint32_t s_lut[256];
  extern __shared__ __align__(16) unsigned char s_dyn[];
  MergeSmem<Tk>* s_m = reinterpret_cast<MergeSmem<Tk>*>(s_dyn);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) s_lut[i] = T.lut[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Tk(*tok)[32] = s_m[wid].tok;
  uint32_t(*rnk)[32] = s_m[wid].rnk;
  uint8_t(*pq)[32] = s_m[wid].pq;
  // Records to merge: all of them, or (dedupe on) the owners k_dedup listed.
  const bool listed = a.dmask != 0;
  const uint32_t nrec = min((uint64_t)a.counters[listed ? CNT_OWNERS : CNT_MREC], (uint64_t)a.mrec_cap);
  const uint32_t* d2id = T.d2id;
  // Records come 32 at a time: lane i holds record base + i of the current
  // batch in registers and idle lanes take theirs by shuffle (no dependent
  // global load on refill); the next batch is in flight meanwhile.
  const ulonglong2 kHole = make_ulonglong2(~0ull, 0ull);
  uint32_t base = 0, next = 0, avail = 0;  // warp-uniform slice of record indices
  uint32_t pbase = 0, pidx = 0;  // record index held by this lane (prefetched batch)
  uint32_t pslot = 0, cslot = 0;           // its dedupe slot + 1 (0: none)
  ulonglong2 cur = kHole, pre = kHole;
  auto fetch = [&]() {
    uint32_t c0 = 0;
    if (lane == 0) c0 = atomicAdd(&a.counters[CNT_MERGE_TICKET], 32u);
    pbase = __shfl_sync(kFull, c0, 0);
    pidx = pbase + lane;
    pslot = 0;
    if (pidx < nrec) {
      if (listed) {
        const uint64_t o = __ldcs(a.owners + pidx);
        pidx = uint32_t(o);
        pslot = uint32_t(o >> 32);
      }
      pre = __ldcs(a.mrec + pidx);
    } else {
      pre = kHole;
    }
  };
  fetch();
  bool exhausted = false;
  int n = 0;      // my piece's current length (0 = idle)
  int np = 0;     // pending probes
  uint32_t m = NONE;  // minimum over resolved ranks
  uint64_t rec = 0;
  uint32_t rslot = 0;
  for (;;) {
    const bool idle = n == 0;
    const unsigned im = __ballot_sync(kFull, idle);
    if (im && next >= avail && !exhausted) {
      base = pbase;
      cur = pre;
      cslot = pslot;
      next = 0;
      avail = base < nrec ? min(32u, nrec - base) : 0u;
      exhausted = avail == 0;
      if (!exhausted) fetch();
    }
    const uint32_t take = min(uint32_t(__popc(im)), avail - next);
    const uint32_t rank = __popc(im & lanemask_lt(lane));
    const bool takes = idle && rank < take;
    const int src_lane = takes ? int(next + rank) : lane;
    const uint64_t hdr = __shfl_sync(kFull, cur.x, src_lane);
    const uint64_t b8 = __shfl_sync(kFull, cur.y, src_lane);
    const uint32_t hslot = __shfl_sync(kFull, cslot, src_lane);
    if (takes) {
      rec = hdr;
      rslot = hslot;
      if (rec != ~0ull) {
        n = int(rec & 63);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (i < n) tok[i][lane] = Tk(s_lut[(b8 >> (8 * i)) & 0xFF]);
          pq[i][lane] = static_cast<uint8_t>(i);
        }
        if (n > 8) {  // bytes past the record's 8: word loads, then the lut
          static_assert(kLmax <= 32, "three words past the record's 8 bytes");
          const uint8_t* src = a.bytes + (rec >> 16);
          for (int i = 8; i < n; ++i) {
            tok[i][lane] = Tk(s_lut[__ldg(src + i)]);
            pq[i][lane] = static_cast<uint8_t>(i);
          }
        }
        np = n - 1;
        m = NONE;
      }
    }
    next += take;
    const bool busy = n > 0;
    if (!__any_sync(kFull, busy)) {
      if (exhausted) break;
      continue;
    }
    if (!busy) continue;
    // probe: pending pairs, BBPE_MERGE_PROBES in flight.
    constexpr int PB = BBPE_MERGE_PROBES;
    for (int p = 0; p < np; p += PB) {
      ProbeReq r[PB];
      int at[PB];
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        at[u] = p + u < np ? int(pq[p + u][lane]) : -1;
        if (at[u] >= 0) probe_issue<K32>(r[u], T, tok[at[u]][lane], tok[at[u] + 1][lane]);
      }
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        if (at[u] >= 0) {
          const uint32_t rk = probe_resolve<K32>(r[u], T);
          rnk[at[u]][lane] = rk;
          m = min(m, rk);
        }
      }
    }
    if (m == NONE || n < 2) {
      // Done: tokens into the reserved slots, kSentinel into the rest; the
      // tile's token count drops by the slots left empty.
      const uint64_t start = rec >> 16;
      const int len = int(rec & 63);
      uint32_t* dst = a.staging + (start / kTile) * kStage + ((rec >> 6) & 1023);
      for (int i = 0; i < n; ++i) {
        const uint32_t v = tok[i][lane];
        dst[i] = d2id ? __ldg(d2id + v) : v;
      }
      for (int i = n; i < len; ++i) dst[i] = kSentinel;
      if (len > n) atomicSub(&a.tile_count[start / kTile], uint32_t(len - n));
      if (rslot) {  // owner of a dedupe slot: its result for the references (DedupRes)
        const uint64_t at = (start / kTile) * kStage + ((rec >> 6) & 1023);
        uint32_t v[kInlineRes];
#pragma unroll
        for (int i = 0; i < kInlineRes; ++i) {
          const uint32_t t = i < n ? uint32_t(tok[i][lane]) : 0u;
          v[i] = d2id && i < n ? __ldg(d2id + t) : t;
        }
        ulonglong2* e = reinterpret_cast<ulonglong2*>(a.dres + 4 * uint64_t(rslot - 1));
        e[0] = make_ulonglong2(at | (uint64_t(n) << 48), uint64_t(v[0]) | (uint64_t(v[1]) << 32));
        e[1] = make_ulonglong2(uint64_t(v[2]) | (uint64_t(v[3]) << 32), uint64_t(v[4]) | (uint64_t(v[5]) << 32));
      }
      n = 0;
      continue;
    }
    // sweep at rank m.
    const Tk M = Tk(K32 ? (m & 0xFFFFu) : __ldg(T.r2m + m));
    const uint32_t mm = m;
    int j = 0, i = 0;
    np = 0;
    m = NONE;
    uint32_t hold = NONE;  // rank of pair (j-1, j) if it survives
    bool prev_merged = false;
    // Branch-free (lanes sweep different pieces): selects and predicated
    // stores instead of an if/else per position.
    while (i < n) {
      const uint32_t ri = (i < n - 1) ? rnk[i][lane] : NONE;
      const bool mg = ri == mm;
      const Tk ti = tok[i][lane];
      tok[j][lane] = mg ? M : ti;
      if (mg && j > 0 && !prev_merged) pq[np++][lane] = static_cast<uint8_t>(j - 1);
      if (mg) pq[np++][lane] = static_cast<uint8_t>(j);
      if (!mg) rnk[j][lane] = ri;
      m = mg ? m : min(m, hold);  // pair (j-1, j) keeps its rank
      hold = mg ? NONE : ri;      // rank of pair (j, j+1), kept unless the next output is a merge
      prev_merged = mg;
      i += mg ? 2 : 1;
      ++j;
    }
    m = min(m, hold);
    n = j;
    // The last merged token has no right pair.
    if (np > 0 && int(pq[np - 1][lane]) >= n - 1) --np;
  }
}

// ---------------------------------------------------------------------------
// k_dedup: thread per merge record. Pieces of <= kDedupMax bytes claim their
// bytes' slot (dedup_claim); the first claimer of each distinct piece is its
// owner and is listed for k_merge, the others become references (k_refs copies
// the owner's tokens). Exact: a piece's encoding depends on its bytes only.
// Longer pieces (and full neighbourhoods) are listed as owners of themselves.
// Owners are listed through one atomicAdd per CTA and step (warp counts
// scanned in shared memory), not one per warp on the shared counter.
constexpr int kDedupThreads = 256;
__global__ void __launch_bounds__(kDedupThreads) k_dedup(EncodeArgs a) {
  __shared__ uint32_t s_cnt[kDedupThreads / 32 + 1];
  const uint64_t nrec = min((uint64_t)a.counters[CNT_MREC], a.mrec_cap);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t stride = uint64_t(gridDim.x) * kDedupThreads;
  for (uint64_t b0 = blockIdx.x * uint64_t(kDedupThreads); b0 < nrec; b0 += stride) {  // CTA-uniform trip count
    const uint64_t i = b0 + threadIdx.x;
    bool owner = false;
    uint64_t oslot = 0;
    if (i < nrec) {
      const ulonglong2 r = __ldcs(a.mrec + i);
      if (r.x != ~0ull) {
        const int len = int(r.x & 63);
        uint64_t res = ~0ull;
        if (len <= kDedupMax) {
          const uint64_t k0 = len >= 8 ? r.y : (r.y & ((1ull << (8 * len)) - 1));
          uint64_t k1 = 0;
          if (len > 8) {  // bytes 8 .. len-1 (<= 7 of them)
            static_assert(kDedupMax < 16, "one word past the record's 8 bytes");
            uint64_t v[1];
            ld_span<1>(a.bytes, a.total, (r.x >> 16) + 8, v);
            k1 = v[0] & ((1ull << (8 * (len - 8))) - 1);
          }
          res = dedup_claim(a.dkey, a.dmask, make_ulonglong2(k0, k1 | (uint64_t(len) << 56)));
        }
        if (res != ~0ull && (res >> 63)) {
          a.mrec[i] = make_ulonglong2(r.x | kRefFlag, res & ~(1ull << 63));
        } else {
          owner = true;
          oslot = res == ~0ull ? 0 : res + 1;
        }
      }
    }
    const unsigned om = __ballot_sync(kFull, owner);
    if (lane == 0) s_cnt[wid] = __popc(om);
    __syncthreads();
    if (wid == 0) {
      const uint32_t c = lane < kDedupThreads / 32 ? s_cnt[lane] : 0u;
      uint32_t inc = c;
#pragma unroll
      for (int d = 1; d < kDedupThreads / 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(kFull, inc, d);
        if (lane >= d) inc += u;
      }
      const uint32_t tot = __shfl_sync(kFull, inc, kDedupThreads / 32 - 1);
      uint32_t b = 0;
      if (lane == 0 && tot) b = atomicAdd(&a.counters[CNT_OWNERS], tot);
      b = __shfl_sync(kFull, b, 0);
      if (lane < kDedupThreads / 32) s_cnt[lane] = b + inc - c;
    }
    __syncthreads();
    if (owner) a.owners[s_cnt[wid] + __popc(om & lanemask_lt(lane))] = i | (oslot << 32);
    __syncthreads();  // s_cnt is rewritten by the next step
  }
}

// k_refs: references (k_dedup) take their owner's tokens: thread per merge
// record, copy from the owner's staging slots (k_merge left its count in the
// record), kSentinel into the rest of the reserved slots, tile count adjusted.
__global__ void __launch_bounds__(256) k_refs(EncodeArgs a) {
  // Warp per 32 records: each lane loads one record and its owner's result,
  // then the records are written out by half-warps, lane j writing slot j
  // (coalesced stores into the reference's contiguous slots).
  static_assert(kDedupMax < 16, "a half-warp covers a reference's slots");
  const uint64_t nrec = min((uint64_t)a.counters[CNT_MREC], a.mrec_cap);
  const int lane = threadIdx.x & 31, h = lane >> 4, j = lane & 15;
  const uint64_t wstride = uint64_t(gridDim.x) * (blockDim.x / 32) * 32;
  for (uint64_t w0 = (blockIdx.x * uint64_t(blockDim.x / 32) + (threadIdx.x >> 5)) * 32; w0 < nrec; w0 += wstride) {
    const uint64_t i = w0 + lane;
    bool ref = false;
    uint64_t hdr = 0;
    ulonglong2 d0 = make_ulonglong2(0, 0), d1 = make_ulonglong2(0, 0);
    if (i < nrec) {
      const ulonglong2 r = __ldcs(a.mrec + i);
      ref = r.x != ~0ull && (r.x & kRefFlag);
      if (ref) {
        hdr = r.x & ~kRefFlag;
        const ulonglong2* de = reinterpret_cast<const ulonglong2*>(a.dres + 4 * r.y);
        d0 = __ldcg(de);
        d1 = __ldcg(de + 1);
      }
    }
    // References two at a time (the two lowest left in `m`): half-warp h
    // takes the (h+1)-th; iterations = ceil(references / 2), warp-uniform.
    for (unsigned m = __ballot_sync(kFull, ref); m;) {
      const unsigned m2 = m & (m - 1);
      const int s0 = __ffs(m) - 1, s1 = m2 ? __ffs(m2) - 1 : -1;
      m = m2 ? m2 & (m2 - 1) : 0u;
      const int src = h ? (s1 < 0 ? s0 : s1) : s0;
      const uint64_t rh = __shfl_sync(kFull, hdr, src);
      const uint64_t e0 = __shfl_sync(kFull, d0.x, src);
      const uint64_t t01 = __shfl_sync(kFull, d0.y, src);
      const uint64_t t23 = __shfl_sync(kFull, d1.x, src);
      const uint64_t t45 = __shfl_sync(kFull, d1.y, src);
      if (h && s1 < 0) continue;
      const int len = int(rh & 63), cnt = int(e0 >> 48);
      const uint64_t start = rh >> 16;
      uint32_t* dst = a.staging + (start / kTile) * kStage + ((rh >> 6) & 1023);
      if (j < len) {
        uint32_t v = kSentinel;
        if (j < cnt) {
          if (cnt <= kInlineRes) {
            const uint64_t pair = j < 2 ? t01 : (j < 4 ? t23 : t45);
            v = uint32_t(pair >> (32 * (j & 1)));
          } else {
            v = __ldcg(a.staging + (e0 & ((1ull << 48) - 1)) + j);
          }
        }
        dst[j] = v;
      }
      if (j == 0 && len > cnt) atomicSub(&a.tile_count[start / kTile], uint32_t(len - cnt));
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
          a.lrec[first + before] = LongRec{o, e - o, s, 0u, 0u, 0};
          if (lfirst + before < a.long_cap) a.long_idx[lfirst + before] = uint32_t(first + before);
        }
        ri += __popc(nm);
      }
      if (lane == 0) {
        a.tile_lrec[tile] = ne ? ((first << 24) | ne) : 0;
        a.tile_count[tile] = 0;
        a.tile_slots[tile] = 0;
        if (a.pstats) {  // every non-empty row is one long piece
          unsigned long long* ps = reinterpret_cast<unsigned long long*>(a.pstats);
          if (ne) {
            atomicAdd(ps + PST_PIECES, (unsigned long long)ne);
            atomicAdd(ps + PST_LONG, (unsigned long long)ne);
          }
          atomicAdd(ps + PST_LONG_BYTES, (unsigned long long)tl);
        }
      }
        }
}

// ---------------------------------------------------------------------------
// k_tile_scan: exclusive scan of the final tile token counts into
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
  if (cta == 0 && tid == 0 && a.pstats && a.dmask)  // k_dedup's owners (k_gather zeroes the counters)
    atomicAdd(reinterpret_cast<unsigned long long*>(a.pstats + PST_OWNERS),
              (unsigned long long)a.counters[CNT_OWNERS]);
  const uint64_t t0 = cta * kScanTiles + uint64_t(tid) * kScanPer;
  uint64_t v[kScanPer];
  uint64_t sum = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    const uint64_t t = t0 + i;
    v[i] = t < a.num_tiles ? __ldcg(a.tile_count + t) : 0;
    sum += v[i];
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
// k_gather: warp per tile. Compacts the tile's staging slots (kSentinel =
// slot a merge piece left empty) into its final CSR place, interleaving the
// tile's long pieces (rare) at their slot positions, and resolves the row
// offsets written by k_pieces. The compacted prefix of every 4-slot group is
// kept in shared memory for the row offsets.
constexpr int kStageIt = (kStage + 31) / 32;  // 32-slot steps per tile
constexpr int kLongCache = kTile / (kLmax + 1) + 2;  // long pieces of a k_pieces tile
struct GatherSmem {
  uint16_t pre[kStageIt + 1];   // valid slots before 32-slot step j
  uint32_t bal[kStageIt + 1];   // valid-slot ballot of step j
  uint32_t lsp[kLongCache];     // long pieces: slot position
  uint32_t lcnt[kLongCache];    // long pieces: token count
};
// Long-piece slot / count: cached in shared memory, or read from the records
// when a tile has more than kLongCache of them (block engine: one per row).
struct LongView {
  const GatherSmem& G;
  const LongRec* r;
  uint32_t n;
  __device__ __forceinline__ uint32_t sp(uint32_t i) const { return n <= kLongCache ? G.lsp[i] : r[i].spref; }
  __device__ __forceinline__ uint32_t cnt(uint32_t i) const {
    return n <= kLongCache ? G.lcnt[i] : __ldcg(&r[i].count);
  }
};

__device__ __forceinline__ uint32_t compact_at(const GatherSmem& G, uint32_t slot, uint32_t nslots,
                                               uint32_t total) {
  if (slot >= nslots) return total;
  return G.pre[slot >> 5] + __popc(G.bal[slot >> 5] & ((1u << (slot & 31)) - 1u));
}

#ifndef BBPE_GATHER_MINB
#define BBPE_GATHER_MINB 4
#endif
#ifndef BBPE_GATHER_EAGER
#define BBPE_GATHER_EAGER 6  // 32-slot steps loaded before the tile's slot count is known to need more
#endif
__global__ void __launch_bounds__(kWarpsPerCta * 32, BBPE_GATHER_MINB) k_gather(EncodeArgs a, DevTable T) {
  __shared__ GatherSmem s_g[kWarpsPerCta];
  (void)T;
  const int lane = threadIdx.x & 31;
  GatherSmem& G = s_g[threadIdx.x >> 5];
  const uint64_t nwarps = uint64_t(gridDim.x) * kWarpsPerCta;
  // Tile metadata is prefetched one tile ahead; a tile's staged slots and row
  // offsets are all loaded before any is used (one round trip, not one per
  // 128-slot chunk).
  uint64_t t = blockIdx.x * uint64_t(kWarpsPerCta) + (threadIdx.x >> 5);
  uint64_t m_tb = 0, m_rec = 0, m_s0 = 0, m_s1 = 0;
  uint32_t m_ns = 0;
  auto meta = [&](uint64_t u) {
    if (u < a.num_tiles) {
      m_tb = __ldcg(a.tile_base + u);
      m_rec = __ldcg(a.tile_lrec + u);
      m_ns = __ldcg(a.tile_slots + u);
      m_s0 = a.tile_first[u];
      m_s1 = a.tile_first[u + 1];
    }
  };
  meta(t);
  for (; t < a.num_tiles; t += nwarps) {
    const uint64_t tbase = m_tb, rec = m_rec, s0 = m_s0, s1 = m_s1;
    const uint32_t nslots = m_ns;
    meta(t + nwarps);
    const uint32_t* stage = a.staging + t * kStage;
    uint32_t* out = a.out_ids + tbase;
    // Typical tiles use ~130 slots: the first kGatherEager steps are loaded
    // unconditionally (all in flight at once), the rest only when the tile
    // has that many slots (warp-uniform branch), so rare full tiles do not
    // cost every tile their load instructions.
    constexpr int kGatherEager = BBPE_GATHER_EAGER;
    uint32_t xs[kStageIt];
#pragma unroll
    for (int j = 0; j < kGatherEager; ++j) {
      const uint32_t v = 32 * j + lane;
      xs[j] = v < nslots ? __ldcs(stage + v) : kSentinel;
    }
    if (nslots > 32u * kGatherEager) {
#pragma unroll
      for (int j = kGatherEager; j < kStageIt; ++j) {
        const uint32_t v = 32 * j + lane;
        xs[j] = v < nslots ? __ldcs(stage + v) : kSentinel;
      }
    } else {
#pragma unroll
      for (int j = kGatherEager; j < kStageIt; ++j) xs[j] = kSentinel;
    }
    uint64_t roff = 0;
    if (s0 + lane < s1 && s0 + lane <= a.n_rows) roff = __ldcg(a.out_offsets + s0 + lane);
    // Leave the look-back status and the counters zero for the next encode.
    if (t < a.num_groups && lane == 0) a.status[t] = 0;
    if (t == 0 && lane < CNT_N && lane != CNT_LREC && lane != CNT_LCOPY && lane != CNT_LDONE) a.counters[lane] = 0;
    // The tile's row-start bits are consumed: leave them zero for the next encode.
    if (a.rowbits && lane < kTile / 32) a.rowbits[t * (kTile / 32) + lane] = 0;
    if (a.chunkbits && lane < kTile / 32) a.chunkbits[t * (kTile / 32) + lane] = 0;
    const uint32_t nl = uint32_t(rec & 0xFFFFFF);
    const uint64_t lfirst = rec >> 24;
    const LongView LV{G, a.lrec + lfirst, nl};
    if (nl && nl <= kLongCache) {  // long pieces: slot positions and counts
      for (uint32_t i = lane; i < nl; i += 32) {
        const LongRec& r = a.lrec[lfirst + i];
        G.lsp[i] = r.spref;
        G.lcnt[i] = __ldcg(&r.count);
      }
      __syncwarp();
    }
    // Staged slots, one per lane per step: compaction by ballot.
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < kStageIt; ++j) {
      if (32u * j >= nslots) break;
      const bool valid = xs[j] != kSentinel;
      const uint32_t bal = __ballot_sync(kFull, valid);
      if (lane == 0) {
        G.pre[j] = static_cast<uint16_t>(run);
        G.bal[j] = bal;
      }
      if (valid) {
        uint32_t o = run + __popc(bal & lanemask_lt(lane));
        if (nl) {  // tokens after the long pieces that precede this slot
          const uint32_t slot = 32 * j + lane;
          for (uint32_t li = 0; li < nl && LV.sp(li) <= slot; ++li) o += LV.cnt(li);
        }
        __stcs(out + o, xs[j]);
      }
      run += __popc(bal);
    }
    __syncwarp();
    if (nl) {  // long pieces: their CSR positions (k_long_copy moves the tokens)
      uint32_t before = 0;
      for (uint32_t li = 0; li < nl; ++li) {
        const uint32_t cnt = LV.cnt(li);
        if (lane == 0) a.lrec[lfirst + li].out = tbase + compact_at(G, LV.sp(li), nslots, run) + before;
        before += cnt;
      }
    }
    // Row offsets: compacted staging slots before the row plus the tokens of
    // the first (v >> 40) long pieces of the tile.
    for (uint64_t s = s0 + lane; s < s1 && s <= a.n_rows; s += 32) {
      const uint64_t v = s == s0 + lane ? roff : __ldcg(a.out_offsets + s);
      const uint32_t lb = uint32_t(v >> 40);
      uint64_t lsum = 0;
      for (uint32_t li = 0; li < lb; ++li) lsum += LV.cnt(li);
      a.out_offsets[s] = tbase + compact_at(G, uint32_t(v & ((1ull << 40) - 1)), nslots, run) + lsum;
    }
    __syncwarp();
  }
}

__global__ void k_advance_base(uint64_t* run_base, const uint64_t* wave_total) {
  *run_base += *wave_total;
}
}  // namespace

// k_copy_out: one wave's results -> the caller's pinned buffers through their
// device mappings: row offsets (wave-relative + *run_base) and ids [0, n) to
// dst[*run_base, ...), clamped to cap; 16-byte stores to host memory after an
// aligning head, posted over PCIe. The waves' copy-outs run in order on one
// stream; k_advance_base moves *run_base on after each.
__global__ void k_copy_out(const uint32_t* __restrict__ src, uint32_t* dst, const uint64_t* __restrict__ d_off,
                           uint64_t* dst_off, uint64_t nr, const uint64_t* run_base, uint64_t cap) {
  const uint64_t rb = *run_base;
  const uint64_t tid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = tid; i <= nr; i += stride) dst_off[i] = rb + __ldcs(d_off + i);
  const uint64_t o0 = rb, end = min(rb + d_off[nr], cap);
  if (o0 >= end) return;
  const uint64_t n = end - o0;
  const uint64_t mis = (reinterpret_cast<uintptr_t>(dst + o0) >> 2) & 3;
  const uint64_t head = min(n, (4 - mis) & 3);
  if (tid < head) dst[o0 + tid] = src[tid];
  const uint64_t nv = (n - head) / 4;
  uint4* dv = reinterpret_cast<uint4*>(dst + o0 + head);
  for (uint64_t v = tid; v < nv; v += stride) {
    const uint64_t i = head + 4 * v;
    dv[v] = make_uint4(__ldcs(src + i), __ldcs(src + i + 1), __ldcs(src + i + 2), __ldcs(src + i + 3));
  }
  const uint64_t t0 = head + 4 * nv;
  if (tid < n - t0) dst[o0 + t0 + tid] = src[t0 + tid];
}

__global__ void k_add_u64(uint64_t* p, uint64_t n, uint64_t v) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    p[i] += v;
}

void launch_add_u64(uint64_t* d_p, uint64_t n, uint64_t v, int sm_count, cudaStream_t stream) {
  if (n && v) k_add_u64<<<unsigned(std::max(sm_count, 1) * 2), 256, 0, stream>>>(d_p, n, v);
}

void launch_copy_out(const uint32_t* d_ids, uint32_t* mapped_out, const uint64_t* d_wave_offsets,
                     uint64_t* mapped_offsets, uint64_t nr, uint64_t* run_base, uint64_t cap, int sm_count,
                     cudaStream_t stream) {
  k_copy_out<<<unsigned(std::max(sm_count, 1)), 256, 0, stream>>>(d_ids, mapped_out, d_wave_offsets, mapped_offsets,
                                                                   nr, run_base, cap);
  k_advance_base<<<1, 1, 0, stream>>>(run_base, d_wave_offsets + nr);
}

size_t pieces_smem() { return sizeof(PieceSmem) * kWarpsPerCta; }
static_assert(sizeof(PieceSmem) % 16 == 0, "per-warp window buffers stay 16-byte aligned");

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
  p.lp_grid = long_pieces_grid(device, p.sm_count);
  p.gather_grid = grid(k_gather, kWarpsPerCta * 32, 0);
  return p;
}

namespace {
__global__ void k_or_words(uint32_t* out, const uint32_t* x, const uint32_t* y, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = x[i] | y[i];
}
}  // namespace

int launch_pretok_only(const EncodeArgs& a, const LaunchPlan& p, uint32_t* d_out_bits, cudaStream_t stream) {
  const unsigned threads = 256, blocks = unsigned((a.n_rows + 1 + threads - 1) / threads);
  k_tile_first<<<blocks, threads, 0, stream>>>(a);
  launch_pretok_gpt2(a.bytes, a.offsets, a.tile_first, a.n_rows, a.total, a.rowbits, a.chunkbits,
                     a.counters + CNT_PRETOK, p.sm_count, stream);
  const uint64_t words = (a.total + 31) / 32;
  if (words) k_or_words<<<unsigned(std::max(p.sm_count, 1) * 2), 256, 0, stream>>>(d_out_bits, a.rowbits, a.chunkbits, words);
  return 4;
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
    if (a.pattern && a.engine != BBPE_ENGINE_BLOCK) {  // (timed with k_tile_first)
      launch_pretok_gpt2(a.bytes, a.offsets, a.tile_first, a.n_rows, a.total, a.rowbits, a.chunkbits,
                         a.counters + CNT_PRETOK, p.sm_count, stream);
      ++launched;
    }
  }
  if (ev) cudaEventRecord(ev[1], stream);
  if (a.engine == BBPE_ENGINE_BLOCK) {
    k_block_rows<<<p.gather_grid, kWarpsPerCta * 32, 0, stream>>>(a, t);
    ++launched;
    if (ev) for (int k = 2; k <= 5; ++k) cudaEventRecord(ev[k], stream);
  } else {
    k_pieces<<<p.main_grid, kWarpsPerCta * 32, pieces_smem(), stream>>>(a, t);
    ++launched;
    if (ev) cudaEventRecord(ev[2], stream);
    if (a.dmask) {
      k_dedup<<<unsigned(p.sm_count * 8), 256, 0, stream>>>(a);
      ++launched;
    }
    if (ev) cudaEventRecord(ev[3], stream);
    if (a.narrow)
      k_merge<uint16_t><<<p.merge_grid, kWarpsPerCta * 32, sizeof(MergeSmem<uint16_t>) * kWarpsPerCta,
                          stream>>>(a, t);
    else
      k_merge<uint32_t><<<p.merge_grid_wide, kWarpsPerCta * 32, sizeof(MergeSmem<uint32_t>) * kWarpsPerCta,
                          stream>>>(a, t);
    ++launched;
    if (ev) cudaEventRecord(ev[4], stream);
    if (a.dmask) {
      k_refs<<<unsigned(p.sm_count * 8), 256, 0, stream>>>(a);
      ++launched;
    }
    if (ev) cudaEventRecord(ev[5], stream);
  }
  launched += launch_long_pieces(a, t, p.lp_grid, stream);
  if (ev) cudaEventRecord(ev[6], stream);
  k_tile_scan<<<unsigned((a.num_tiles + kScanTiles - 1) / kScanTiles), kScanThreads, 0, stream>>>(a);
  ++launched;
  if (ev) cudaEventRecord(ev[7], stream);
  k_gather<<<p.gather_grid, kWarpsPerCta * 32, 0, stream>>>(a, t);
  ++launched;
  launch_long_copy(a, t, p.gather_grid, stream);
  ++launched;
  if (ev) cudaEventRecord(ev[8], stream);
  return launched;
}

int launch_block_bpe(const EncodeArgs& a, const DevTable& t, const LaunchPlan& p,
                     cudaStream_t stream) {
  (void)p;
  return launch_long_pieces(a, t, 1, stream);
}

}  // namespace bbpe
