// specials.cu -- special tokens on the device.
//
// encode_batch (batch.hpp:64-126) splits every row at special tokens
// (split_specials, pretokenize.hpp:32-57: at each position the longest
// special that fits in the row is consumed, SpecialTokenSet::match
// merge_table.hpp:336-344), BPE-encodes the literal segments and passes the
// special ids through, with optional BOS/EOS. Here:
//   k_sp_cand    position-parallel candidate bits (a special matches at p,
//                row ends ignored: a superset of the real matches)
//   k_sp_rows    thread per row: the greedy walk over the row's candidates
//                (sequential by definition; candidates are rare) -> counts
//   scan         match / literal-byte bases
//   k_sp_emit    thread per row: literal segment offsets and special ids
//   k_sp_copy    warp per segment: literal bytes compacted (special bytes are
//                never BPE-encoded, so a special may hold bytes with no token)
//   (encode of the literal segments as rows: the ordinary pipeline)
//   k_sp_len     row lengths; scan -> output offsets
//   k_sp_stitch  warp per row: BOS, segment tokens, special ids, EOS
#include "specials.cuh"

#include "scan.cuh"

namespace bbpe {
namespace {

constexpr int kScanThreads = 256;

__global__ void __launch_bounds__(kScanThreads) k_scan_blocks(uint64_t* v, uint64_t n, uint64_t* sums) {
  __shared__ uint64_t s_warp[kScanThreads / 32];
  const uint64_t i = blockIdx.x * uint64_t(kScanThreads) + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t x = i < n ? v[i] : 0;
  uint64_t inc = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint64_t w = lane < kScanThreads / 32 ? s_warp[lane] : 0;
    uint64_t wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, wi, d);
      if (lane >= d) wi += u;
    }
    if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
    if (lane == 31) sums[blockIdx.x] = wi;
  }
  __syncthreads();
  if (i < n) v[i] = s_warp[wid] + inc - x;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_add(uint64_t* v, uint64_t n, const uint64_t* sums,
                                                           uint64_t nb) {
  const uint64_t i = blockIdx.x * uint64_t(kScanThreads) + threadIdx.x;
  if (i < n) v[i] += sums[blockIdx.x];
  if (i == 0) v[n] = sums[nb];
}

// The 4 bytes at b[p..p+4) as a little-endian word (byte loads: p is unaligned).
__device__ __forceinline__ uint32_t load4(const uint8_t* b) {
  return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
}

__device__ __forceinline__ uint32_t sp_match(const SpecArgs& S, const uint8_t* b, uint64_t p, uint64_t end,
                                             uint32_t& id) {
  for (uint32_t i = 0; i < S.n; ++i) {
    const uint32_t o = S.off[i], len = S.off[i + 1] - o;
    if (len > end - p) continue;
    uint32_t k = 0;
    // four bytes per step (all loads of a step independent), then the tail
    while (k + 4 <= len && load4(b + p + k) == load4(S.blob + o + k)) k += 4;
    if (k + 4 <= len) continue;  // a word differed
    while (k < len && b[p + k] == S.blob[o + k]) ++k;
    if (k == len) {
      id = S.id[i];
      return len;
    }
  }
  return 0;
}

// Thread per 32-byte word of the candidate bitmap.
__global__ void __launch_bounds__(256) k_sp_cand(const uint8_t* bytes, uint64_t total, SpecArgs sp,
                                                 uint32_t* cand) {
  __shared__ uint32_t s_first[8];
  __shared__ uint32_t s_fb[4];  // up to 4 distinct first bytes, each replicated into the 4 byte lanes
  __shared__ int s_nfb;         // their number, or -1 for more (bitmap test per byte)
  if (threadIdx.x < 8) s_first[threadIdx.x] = sp.first[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    int k = 0;
    for (int c = 0; c < 256; ++c)
      if ((s_first[c >> 5] >> (c & 31)) & 1u) {
        if (k < 4) s_fb[k] = uint32_t(c) * 0x01010101u;
        ++k;
      }
    s_nfb = k <= 4 ? k : -1;
  }
  __syncthreads();
  const int nfb = s_nfb;
  // the first bytes in registers; unused ones repeat the first (no effect on the OR)
  const uint32_t fb0 = nfb > 0 ? s_fb[0] : 0u, fb1 = nfb > 1 ? s_fb[1] : fb0, fb2 = nfb > 2 ? s_fb[2] : fb0,
                 fb3 = nfb > 3 ? s_fb[3] : fb0;
  const uint64_t nw = (total + 31) / 32, stride = uint64_t(gridDim.x) * blockDim.x;
  const bool aligned = (reinterpret_cast<uintptr_t>(bytes) & 15) == 0;
  for (uint64_t w = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; w < nw; w += stride) {
    uint32_t bits = 0;
    const uint64_t p0 = w * 32, p1 = min(total, p0 + 32);
    uint32_t v[8];
    if (aligned && p1 - p0 == 32) {  // two 16-byte loads
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(bytes + p0));
      const uint4 y = __ldg(reinterpret_cast<const uint4*>(bytes + p0 + 16));
      v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w, v[4] = y.x, v[5] = y.y, v[6] = y.z, v[7] = y.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0;
      for (uint64_t p = p0; p < p1; ++p) v[(p - p0) >> 2] |= uint32_t(__ldg(bytes + p)) << (8 * ((p - p0) & 3));
    }
    uint32_t maybe = 0;  // bit k: byte k is a special's first byte
    if (nfb > 0) {       // few first bytes: 4-byte SIMD compares
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t m = __vcmpeq4(v[k], fb0) | __vcmpeq4(v[k], fb1) | __vcmpeq4(v[k], fb2) | __vcmpeq4(v[k], fb3);
        maybe |= (((m >> 7) & 1u) | ((m >> 14) & 2u) | ((m >> 21) & 4u) | ((m >> 28) & 8u)) << (4 * k);
      }
    } else if (nfb < 0) {
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const uint32_t c = (v[k >> 2] >> (8 * (k & 3))) & 0xFFu;
        maybe |= ((s_first[c >> 5] >> (c & 31)) & 1u) << k;
      }
    }
    if (p1 - p0 < 32) maybe &= (1u << (p1 - p0)) - 1u;
    for (; maybe; maybe &= maybe - 1) {  // rare: the full match at each candidate
      const int k = __ffs(maybe) - 1;
      uint32_t id;
      if (sp_match(sp, bytes, p0 + k, total, id)) bits |= 1u << k;
    }
    cand[w] = bits;
  }
}

// The greedy walk of one row; f(pos_of_match, len, id) per special consumed.
template <typename F>
__device__ __forceinline__ void sp_walk(const SpecArgs& sp, const uint8_t* bytes, const uint32_t* cand,
                                        uint64_t rs, uint64_t re, F f) {
  uint64_t pos = rs;
  for (uint64_t w = rs >> 5; rs < re && w <= (re - 1) >> 5; ++w) {
    uint32_t bits = cand[w];
    while (bits) {
      const uint64_t p = w * 32 + __ffs(bits) - 1;
      bits &= bits - 1;
      if (p < pos) continue;
      if (p >= re) return;
      uint32_t id = 0;
      const uint32_t len = sp_match(sp, bytes, p, re, id);
      if (len) {
        f(p, len, id);
        pos = p + len;
      }
    }
  }
}

__global__ void k_sp_rows(const uint8_t* bytes, const uint64_t* offsets, uint64_t n_rows, SpecArgs sp,
                          const uint32_t* cand, uint64_t* cnt, uint64_t* lit) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (r >= n_rows) return;
  const uint64_t rs = offsets[r], re = offsets[r + 1];
  uint64_t k = 0, sb = 0;
  sp_walk(sp, bytes, cand, rs, re, [&](uint64_t, uint32_t len, uint32_t) {
    ++k;
    sb += len;
  });
  cnt[r] = k;
  lit[r] = (re - rs) - sb;
}

__global__ void k_sp_emit(const uint8_t* bytes, const uint64_t* offsets, uint64_t n_rows, SpecArgs sp,
                          const uint32_t* cand, const uint64_t* match_base, const uint64_t* lit_base,
                          uint64_t* seg_off, uint64_t* seg_src, uint32_t* sp_ids, int inplace) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (r >= n_rows) return;
  const uint64_t rs = offsets[r], re = offsets[r + 1];
  const uint64_t mb = match_base[r];
  if (inplace) {  // segments tile the input: literal, special, literal, ..., literal
    uint64_t seg = r + 2 * mb, src = rs, j = 0;
    sp_walk(sp, bytes, cand, rs, re, [&](uint64_t p, uint32_t len, uint32_t id) {
      seg_off[seg++] = src;
      seg_off[seg++] = p;
      sp_ids[mb + j++] = id;
      src = p + len;
    });
    seg_off[seg] = src;
    if (r + 1 == n_rows) seg_off[seg + 1] = re;
    return;
  }
  uint64_t seg = r + mb, at = lit_base[r], src = rs, j = 0;
  sp_walk(sp, bytes, cand, rs, re, [&](uint64_t p, uint32_t len, uint32_t id) {
    seg_off[seg] = at;  // literal segment [src, p)
    seg_src[seg] = src;
    at += p - src;
    ++seg;
    sp_ids[mb + j++] = id;
    src = p + len;
  });
  seg_off[seg] = at;  // the row's last literal segment [src, re)
  seg_src[seg] = src;
  if (r + 1 == n_rows) seg_off[seg + 1] = at + (re - src);
}

// Warp per segment (grid-stride): literal bytes to their compacted place.
__global__ void __launch_bounds__(256) k_sp_copy(const uint8_t* bytes, uint64_t n_seg, const uint64_t* seg_off,
                                                 const uint64_t* seg_src, uint8_t* compact) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x / 32);
  for (uint64_t s = blockIdx.x * uint64_t(blockDim.x / 32) + (threadIdx.x >> 5); s < n_seg; s += nw) {
    const uint64_t d0 = seg_off[s], len = seg_off[s + 1] - d0, s0 = seg_src[s];
    for (uint64_t i = lane; i < len; i += 32) compact[d0 + i] = __ldg(bytes + s0 + i);
  }
}

__global__ void k_sp_len(uint64_t n_rows, const uint64_t* match_base, const uint64_t* seg_tok_off, int add_bos,
                         int add_eos, int stride, uint64_t* out_len) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (r >= n_rows) return;
  const uint64_t k = match_base[r + 1] - match_base[r], s0 = r + stride * match_base[r];
  uint64_t lit = 0;
  if (stride == 1) {
    lit = seg_tok_off[s0 + k + 1] - seg_tok_off[s0];  // the row's literal segments are contiguous
  } else {
    for (uint64_t j = 0; j <= k; ++j) lit += seg_tok_off[s0 + 2 * j + 1] - seg_tok_off[s0 + 2 * j];
  }
  out_len[r] = uint64_t(add_bos) + uint64_t(add_eos) + k + lit;
}

// Warp per 32 rows (grid-stride): lane l loads row l's metadata (match base,
// output offset, the first segments' token ranges) so the rows' dependent
// loads overlap; the warp then copies row by row, lanes along the tokens.
__global__ void __launch_bounds__(256) k_sp_stitch(uint64_t n_rows, const uint64_t* match_base,
                                                   const uint64_t* seg_tok_off, const uint32_t* seg_ids,
                                                   const uint32_t* sp_ids, const uint64_t* out_off, uint32_t bos_id,
                                                   uint32_t eos_id, int stride, uint32_t* out_ids) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x / 32);
  for (uint64_t r0 = (blockIdx.x * uint64_t(blockDim.x / 32) + (threadIdx.x >> 5)) * 32; r0 < n_rows; r0 += nw * 32) {
    const uint64_t r = r0 + lane;
    uint64_t mb = 0, k = 0, at = 0, t0 = 0, t1 = 0;
    if (r < n_rows) {
      mb = match_base[r];
      k = match_base[r + 1] - mb;
      at = out_off[r];
      const uint64_t s0 = r + stride * mb;
      t0 = seg_tok_off[s0];
      t1 = seg_tok_off[s0 + 1];
    }
    const uint32_t live = __ballot_sync(0xFFFFFFFFu, r < n_rows);
    for (int i = 0; i < 32 && ((live >> i) & 1u); ++i) {
      const uint64_t rmb = __shfl_sync(0xFFFFFFFFu, mb, i), rk = __shfl_sync(0xFFFFFFFFu, k, i);
      uint64_t o = __shfl_sync(0xFFFFFFFFu, at, i);
      uint64_t a = __shfl_sync(0xFFFFFFFFu, t0, i), b = __shfl_sync(0xFFFFFFFFu, t1, i);
      const uint64_t s0 = (r0 + i) + stride * rmb;
      if (bos_id != 0xFFFFFFFFu) {
        if (lane == 0) out_ids[o] = bos_id;
        ++o;
      }
      for (uint64_t j = 0;; ++j) {  // literal segment j: tokens [a, b)
        for (uint64_t q = lane; q < b - a; q += 32) out_ids[o + q] = seg_ids[a + q];
        o += b - a;
        if (j == rk) break;
        if (lane == 0) out_ids[o] = sp_ids[rmb + j];
        ++o;
        a = seg_tok_off[s0 + stride * (j + 1)];
        b = seg_tok_off[s0 + stride * (j + 1) + 1];
      }
      if (eos_id != 0xFFFFFFFFu && lane == 0) out_ids[o] = eos_id;
    }
  }
}

unsigned blocks_for(uint64_t n, unsigned threads) { return unsigned((n + threads - 1) / threads); }

}  // namespace

uint64_t scan_sums_len(uint64_t n) { return (n + kScanThreads - 1) / kScanThreads + 1; }

void launch_scan_u64(uint64_t* v, uint64_t n, uint64_t* sums, cudaStream_t s) {
  const uint64_t nb = (n + kScanThreads - 1) / kScanThreads;
  if (nb == 0) {
    cudaMemsetAsync(v, 0, 8, s);
    return;
  }
  k_scan_blocks<<<unsigned(nb), kScanThreads, 0, s>>>(v, n, sums);
  k_scan_totals<<<1, 1024, 0, s>>>(sums, nb);
  k_scan_add<<<unsigned(nb), kScanThreads, 0, s>>>(v, n, sums, nb);
}

void launch_sp_candidates(const uint8_t* bytes, uint64_t total, SpecArgs sp, uint32_t* cand, int sm_count,
                          cudaStream_t s) {
  const uint64_t nw = (total + 31) / 32;
  if (!nw) return;
  const unsigned blocks = unsigned(std::min<uint64_t>(blocks_for(nw, 256), uint64_t(sm_count) * 8));
  k_sp_cand<<<blocks, 256, 0, s>>>(bytes, total, sp, cand);
}

void launch_sp_rows(const uint8_t* bytes, const uint64_t* offsets, uint64_t n_rows, SpecArgs sp,
                    const uint32_t* cand, uint64_t* cnt, uint64_t* lit, cudaStream_t s) {
  if (n_rows) k_sp_rows<<<blocks_for(n_rows, 128), 128, 0, s>>>(bytes, offsets, n_rows, sp, cand, cnt, lit);
}

void launch_sp_emit(const uint8_t* bytes, const uint64_t* offsets, uint64_t n_rows, SpecArgs sp,
                    const uint32_t* cand, const uint64_t* match_base, const uint64_t* lit_base, uint64_t* seg_off,
                    uint64_t* seg_src, uint32_t* sp_ids, int inplace, cudaStream_t s) {
  if (n_rows)
    k_sp_emit<<<blocks_for(n_rows, 128), 128, 0, s>>>(bytes, offsets, n_rows, sp, cand, match_base, lit_base,
                                                     seg_off, seg_src, sp_ids, inplace);
}

void launch_sp_copy(const uint8_t* bytes, uint64_t n_seg, const uint64_t* seg_off, const uint64_t* seg_src,
                    uint8_t* compact, int sm_count, cudaStream_t s) {
  if (n_seg) k_sp_copy<<<unsigned(sm_count * 8), 256, 0, s>>>(bytes, n_seg, seg_off, seg_src, compact);
}

void launch_sp_lengths(uint64_t n_rows, const uint64_t* match_base, const uint64_t* seg_tok_off, int add_bos,
                       int add_eos, int stride, uint64_t* out_len, cudaStream_t s) {
  if (n_rows)
    k_sp_len<<<blocks_for(n_rows, 256), 256, 0, s>>>(n_rows, match_base, seg_tok_off, add_bos, add_eos, stride,
                                                    out_len);
}

void launch_sp_stitch(uint64_t n_rows, const uint64_t* match_base, const uint64_t* seg_tok_off,
                      const uint32_t* seg_ids, const uint32_t* sp_ids, const uint64_t* out_off, uint32_t bos_id,
                      uint32_t eos_id, int stride, uint32_t* out_ids, int sm_count, cudaStream_t s) {
  if (n_rows)
    k_sp_stitch<<<unsigned(sm_count * 8), 256, 0, s>>>(n_rows, match_base, seg_tok_off, seg_ids, sp_ids, out_off,
                                                       bos_id, eos_id, stride, out_ids);
}

}  // namespace bbpe
