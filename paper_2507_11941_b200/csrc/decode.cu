// decode.cu -- batch decode on the device: CSR token ids ->
// CSR bytes, the inverse of the encode path; and the JSON-lines text of a
// batch (write_batch_jsonl). Semantics of
// decode (merge_table.hpp:565-579: concatenate each id's bytes, DecodeError
// "unknown token id X at index i") and decode_batch (batch.hpp:128-154: per
// row, error prefixed "row r: ").
//
// Device table: dec[id] = byte start << 24 | byte length (~0: no such token),
// dense over ids 0..max_id, and the token bytes; built once per device.
// Kernels: k_dec_mark (row-start tokens as bits), k_dec_len (block byte
// totals, first bad token), k_scan_totals (scan.cuh: block totals -> block
// bases, one CTA), k_dec_copy (block-local scan again; the block's bytes
// assembled in shared memory and written with aligned 16-byte stores;
// row-start tokens record their byte position), k_dec_rows (row byte offsets).
#include <cuda_runtime.h>

#include <cstdint>

#include "decode.cuh"
#include "scan.cuh"

namespace bbpe {
namespace {

constexpr int kDecThreads = 256;

// decode (merge_table.hpp:565-579) of one id: the table's bytes, else the
// special's; decode_batch's skip_specials drops special ids first
// (batch.hpp:134-139). Returns false for an unknown id.
__device__ __forceinline__ bool dec_entry(const DecodeArgs& a, uint32_t id, const uint8_t*& src, uint64_t& len,
                                          bool& from_table) {
  from_table = false;
  int k = -1;
  if (a.sp_n) {
    uint32_t lo = 0, hi = a.sp_n;
    while (lo < hi) {
      const uint32_t m = (lo + hi) >> 1;
      if (a.sp_ids[m] < id) lo = m + 1;
      else hi = m;
    }
    if (lo < a.sp_n && a.sp_ids[lo] == id) k = int(lo);
    if (k >= 0 && a.skip) {
      len = 0;
      src = nullptr;
      return true;
    }
  }
  const uint64_t e = id < a.dec_n ? __ldg(a.dec + id) : ~0ull;
  if (e != ~0ull) {
    len = e & 0xFFFFFF;
    src = a.dec_bytes + (e >> 24);
    from_table = true;
    return true;
  }
  if (k < 0) return false;
  len = a.sp_len[k];
  src = a.sp_blob + a.sp_off[k];
  return true;
}

// Row starts as token bits (k_dec_copy records their byte positions).
__global__ void k_dec_mark(DecodeArgs a) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (r >= a.n_rows) return;
  const uint64_t t = a.tok_off[r] - a.tok_off[0];
  if (t < a.n_ids) atomicOr(a.rowstart + (t >> 5), 1u << (t & 31));
}

// A block decodes kDecBlockTok tokens: warp w takes tokens [256 w, 256 w +
// 256) of the block in kDecTok rounds of 32 consecutive tokens (lane l: token
// 32 k + l), so id loads are coalesced and the lanes of a round write
// neighbouring bytes; the table lookups of a lane's rounds are in flight
// together.
constexpr int kDecTok = 8;
constexpr int kDecBlockTok = kDecThreads * kDecTok;
static_assert(kDecBlockTok == kDecodeBlockTokens, "host block count");

__device__ __forceinline__ void dec_round_lengths(const DecodeArgs& a, uint64_t wbase, int lane,
                                                  uint32_t (&len)[kDecTok], const uint8_t* (&src)[kDecTok],
                                                  bool record_err, bool (&tabk)[kDecTok]) {
  uint32_t id[kDecTok];
#pragma unroll
  for (int k = 0; k < kDecTok; ++k) {
    const uint64_t t = wbase + 32 * k + lane;
    id[k] = t < a.n_ids ? __ldg(a.ids + t) : 0u;
  }
#pragma unroll
  for (int k = 0; k < kDecTok; ++k) {
    const uint64_t t = wbase + 32 * k + lane;
    uint64_t l = 0;
    bool tab = false;
    src[k] = nullptr;
    if (t < a.n_ids && !dec_entry(a, id[k], src[k], l, tab)) {
      l = 0;
      if (record_err) atomicMin(reinterpret_cast<unsigned long long*>(a.err), (unsigned long long)t);
    }
    len[k] = uint32_t(l);
    tabk[k] = tab;
  }
}

__device__ __forceinline__ uint32_t warp_sum32(uint32_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
  return v;
}

// Token lengths -> block byte totals, and the first unknown id.
__global__ void __launch_bounds__(kDecThreads) k_dec_len(DecodeArgs a) {
  __shared__ uint64_t s_w[kDecThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t wbase = blockIdx.x * uint64_t(kDecBlockTok) + uint64_t(wid) * (32 * kDecTok);
  uint32_t len[kDecTok];
  bool tab[kDecTok];
  const uint8_t* src[kDecTok];
  dec_round_lengths(a, wbase, lane, len, src, true, tab);
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < kDecTok; ++k) sum += len[k];
  sum = warp_sum32(sum);
  if (lane == 0) s_w[wid] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t tot = 0;
#pragma unroll
    for (int w = 0; w < kDecThreads / 32; ++w) tot += s_w[w];
    a.block_sums[blockIdx.x] = tot;
  }
}

// The block's bytes: assembled in shared memory, then written as aligned
// 16-byte stores (byte stores for the unaligned head and tail); blocks with
// more than kDecStage bytes (very long tokens or specials) copy byte by byte.
constexpr int kDecStage = 24576;
__global__ void __launch_bounds__(kDecThreads) k_dec_copy(DecodeArgs a) {
  __shared__ uint64_t s_w[kDecThreads / 32 + 1];
  __shared__ __align__(16) uint8_t s_out[kDecStage + 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t wbase = blockIdx.x * uint64_t(kDecBlockTok) + uint64_t(wid) * (32 * kDecTok);
  uint32_t len[kDecTok];
  bool tab[kDecTok];
  const uint8_t* src[kDecTok];
  dec_round_lengths(a, wbase, lane, len, src, false, tab);
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < kDecTok; ++k) sum += len[k];
  sum = warp_sum32(sum);
  if (lane == 0) s_w[wid] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive warp bases, block total last
    uint64_t run = 0;
#pragma unroll
    for (int w = 0; w < kDecThreads / 32; ++w) {
      const uint64_t v = s_w[w];
      s_w[w] = run;
      run += v;
    }
    s_w[kDecThreads / 32] = run;
  }
  __syncthreads();
  const uint64_t btot = s_w[kDecThreads / 32];
  const uint64_t base = a.block_sums[blockIdx.x];
  const bool stage = btot <= kDecStage;
  uint64_t off = s_w[wid];  // this round's first byte, block-relative
#pragma unroll
  for (int k = 0; k < kDecTok; ++k) {
    uint32_t inc = len[k];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, d);
      if (lane >= d) inc += u;
    }
    const uint64_t o = off + inc - len[k];
    off += __shfl_sync(0xFFFFFFFFu, inc, 31);
    const uint64_t t = wbase + 32 * k + lane;
    if (t < a.n_ids && ((a.rowstart[t >> 5] >> (t & 31)) & 1u)) a.pos[t] = base + o;
    if (stage) {
      for (uint32_t j = 0; j < len[k]; ++j) s_out[o + j] = __ldg(src[k] + j);
    } else {
      for (uint32_t j = 0; j < len[k] && base + o + j < a.cap; ++j) a.out[base + o + j] = __ldg(src[k] + j);
    }
  }
  if (!stage) return;
  __syncthreads();
  const uint64_t end = min(base + btot, a.cap);
  if (end <= base) return;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(a.out);
  const uint64_t a0 = min(end, base + ((16 - ((addr + base) & 15)) & 15));  // first 16-byte aligned position
  const uint64_t a1 = a0 + ((end - a0) & ~uint64_t(15));                     // end of the aligned body
  for (uint64_t p = base + threadIdx.x; p < a0; p += kDecThreads) a.out[p] = s_out[p - base];
  for (uint64_t p = a1 + threadIdx.x; p < end; p += kDecThreads) a.out[p] = s_out[p - base];
  const uint32_t* w = reinterpret_cast<const uint32_t*>(s_out);
  for (uint64_t p = a0 + 16 * uint64_t(threadIdx.x); p < a1; p += 16 * uint64_t(kDecThreads)) {
    const uint32_t q = uint32_t(p - base), k = q >> 2, sh = (q & 3) * 8;
    const uint32_t x0 = w[k], x1 = w[k + 1], x2 = w[k + 2], x3 = w[k + 3], x4 = w[k + 4];
    *reinterpret_cast<uint4*>(a.out + p) = make_uint4(__funnelshift_r(x0, x1, sh), __funnelshift_r(x1, x2, sh),
                                                      __funnelshift_r(x2, x3, sh), __funnelshift_r(x3, x4, sh));
  }
}

__global__ void k_dec_rows(DecodeArgs a) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (r > a.n_rows) return;
  const uint64_t t = a.tok_off[r] - a.tok_off[0];
  a.out_off[r] = t >= a.n_ids ? a.block_sums[a.n_blocks] : a.pos[t];
}

// ---- JSON-lines text (write_batch_jsonl, batch.hpp:157-166): per row
// {"ids":[i0,i1,...],"len":n}\n, the compact nlohmann dump. Token i takes
// digits(id) + 1 characters (its comma, or the row's closing bracket is
// accounted in the row frame); row r's frame is 18 + digits(n) - (n > 0).
__device__ __forceinline__ uint32_t ndigits(uint64_t v) {
  uint32_t d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

__device__ __forceinline__ void put_digits(uint8_t* out, uint64_t pos, uint64_t cap, uint64_t v, uint32_t d) {
  for (int k = int(d) - 1; k >= 0; --k) {
    if (pos + k < cap) out[pos + k] = uint8_t('0' + v % 10);
    v /= 10;
  }
}

__device__ __forceinline__ void put_str(uint8_t* out, uint64_t pos, uint64_t cap, const char* s, int n) {
  for (int k = 0; k < n; ++k)
    if (pos + k < cap) out[pos + k] = uint8_t(s[k]);
}

// Block-local exclusive scan of v over kDecThreads threads; block total to sums[block].
__device__ __forceinline__ uint64_t block_excl(uint64_t v, uint64_t* sums) {
  __shared__ uint64_t s_warp[kDecThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint64_t x = lane < kDecThreads / 32 ? s_warp[lane] : 0;
    uint64_t xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, xi, d);
      if (lane >= d) xi += u;
    }
    if (lane < kDecThreads / 32) s_warp[lane] = xi - x;
    if (lane == 31) sums[blockIdx.x] = xi;
  }
  __syncthreads();
  return s_warp[wid] + inc - v;
}

// Decimal digits of a u32 id (branch-free compares).
__device__ __forceinline__ uint32_t ndigits32(uint32_t v) {
  return 1u + (v >= 10u) + (v >= 100u) + (v >= 1000u) + (v >= 10000u) + (v >= 100000u) + (v >= 1000000u) +
         (v >= 10000000u) + (v >= 100000000u) + (v >= 1000000000u);
}

// Row text lengths (warp per row): the frame plus every token's digits and comma.
__global__ void __launch_bounds__(256) k_json_rowlen(JsonArgs a) {
  const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x / 32) + (threadIdx.x >> 5); r < a.n_rows; r += nw) {
    const uint64_t t0 = a.tok_off[r] - a.tok_off[0], t1 = a.tok_off[r + 1] - a.tok_off[0];
    uint64_t s = 0;
    for (uint64_t i = t0 + lane; i < t1; i += 32) s += ndigits32(__ldg(a.ids + i)) + 1;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, d);
    const uint64_t len = t1 - t0;
    if (lane == 0) a.row_pos[r] = 18 + ndigits(len) - (len > 0 ? 1 : 0) + s;
  }
}

// Row lengths -> exclusive positions within blocks of 256 rows, block totals.
__global__ void __launch_bounds__(kDecThreads) k_json_rowscan(JsonArgs a) {
  const uint64_t r = blockIdx.x * uint64_t(kDecThreads) + threadIdx.x;
  const uint64_t v = r < a.n_rows ? a.row_pos[r] : 0;
  const uint64_t e = block_excl(v, a.row_sums);
  if (r < a.n_rows) a.row_pos[r] = e;
}

// The text (warp per row): tokens 32 at a time, their digits and commas laid
// out in a per-warp shared buffer by a warp scan, then written with
// consecutive lanes on consecutive bytes.
__global__ void __launch_bounds__(256) k_json_write(JsonArgs a) {
  __shared__ uint8_t s_buf[8][32 * 11 + 8];
  const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  uint8_t* buf = s_buf[threadIdx.x >> 5];
  const uint64_t tb = a.tok_off[0];
  // The next row's offsets and position are loaded while this row is written.
  uint64_t r = blockIdx.x * uint64_t(blockDim.x / 32) + (threadIdx.x >> 5);
  uint64_t n_o0 = 0, n_o1 = 0, n_s = 0, n_p = 0;
  if (r < a.n_rows) {
    n_o0 = a.tok_off[r];
    n_o1 = a.tok_off[r + 1];
    n_s = a.row_sums[r / kDecThreads];
    n_p = a.row_pos[r];
  }
  for (; r < a.n_rows; r += nw) {
    const uint64_t t0 = n_o0 - tb, t1 = n_o1 - tb;
    const uint64_t len = t1 - t0;
    const uint64_t start = n_s + n_p;
    const uint64_t rn = r + nw;
    if (rn < a.n_rows) {
      n_o0 = a.tok_off[rn];
      n_o1 = a.tok_off[rn + 1];
      n_s = a.row_sums[rn / kDecThreads];
      n_p = a.row_pos[rn];
    }
    if (lane == 0) put_str(a.out, start, a.cap, "{\"ids\":[", 8);
    uint64_t pos = start + 8;
    for (uint64_t c0 = t0; c0 < t1; c0 += 32) {
      const uint64_t i = c0 + lane;
      const bool valid = i < t1;
      const uint32_t id = valid ? __ldg(a.ids + i) : 0u;
      const uint32_t d = valid ? ndigits32(id) : 0u;
      const bool comma = valid && i + 1 < t1;
      const uint32_t w = d + (comma ? 1u : 0u);
      uint32_t inc = w;
#pragma unroll
      for (int k = 1; k < 32; k <<= 1) {
        const uint32_t u = __shfl_up_sync(0xFFFFFFFFu, inc, k);
        if (lane >= k) inc += u;
      }
      const uint32_t total = __shfl_sync(0xFFFFFFFFu, inc, 31);
      const uint32_t o = inc - w;
      uint32_t v = id;
      for (int k = int(d) - 1; k >= 0; --k) {
        buf[o + k] = uint8_t('0' + v % 10);
        v /= 10;
      }
      if (comma) buf[o + d] = ',';
      __syncwarp();
      for (uint32_t b = lane; b < total; b += 32)
        if (pos + b < a.cap) a.out[pos + b] = buf[b];
      __syncwarp();
      pos += total;
    }
    if (lane == 0) {
      put_str(a.out, pos, a.cap, "],\"len\":", 8);
      const uint32_t d = ndigits(len);
      put_digits(a.out, pos + 8, a.cap, len, d);
      put_str(a.out, pos + 8 + d, a.cap, "}\n", 2);
    }
  }
}

}  // namespace

void launch_jsonl(const JsonArgs& a, int sm_count, cudaStream_t s) {
  // Row positions carry the whole text: the token-level total stays zero.
  cudaMemsetAsync(a.tok_sums + a.n_tok_blocks, 0, 8, s);
  if (a.n_rows) {
    k_json_rowlen<<<unsigned(sm_count * 8), 256, 0, s>>>(a);
    k_json_rowscan<<<unsigned(a.n_row_blocks), kDecThreads, 0, s>>>(a);
    k_scan_totals<<<1, 1024, 0, s>>>(a.row_sums, a.n_row_blocks);
    k_json_write<<<unsigned(sm_count * 8), 256, 0, s>>>(a);
  } else {
    cudaMemsetAsync(a.row_sums, 0, 8, s);
  }
}

void launch_decode(const DecodeArgs& a, cudaStream_t s) {
  if (a.n_ids) {
    cudaMemsetAsync(a.rowstart, 0, ((a.n_ids + 31) / 32) * 4, s);
    if (a.n_rows) k_dec_mark<<<unsigned((a.n_rows + 255) / 256), 256, 0, s>>>(a);
    k_dec_len<<<unsigned(a.n_blocks), kDecThreads, 0, s>>>(a);
    k_scan_totals<<<1, 1024, 0, s>>>(a.block_sums, a.n_blocks);
    k_dec_copy<<<unsigned(a.n_blocks), kDecThreads, 0, s>>>(a);
  } else {
    cudaMemsetAsync(a.block_sums, 0, 8, s);
  }
  k_dec_rows<<<unsigned((a.n_rows + 1 + 255) / 256), 256, 0, s>>>(a);
}

}  // namespace bbpe
