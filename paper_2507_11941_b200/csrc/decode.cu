// decode.cu -- batch decode on the device: CSR token ids ->
// CSR bytes, the inverse of the encode path; and the JSON-lines text of a
// batch (write_batch_jsonl). Semantics of
// decode (merge_table.hpp:565-579: concatenate each id's bytes, DecodeError
// "unknown token id X at index i") and decode_batch (batch.hpp:128-154: per
// row, error prefixed "row r: ").
//
// Device table: dec[id] = byte start << 24 | byte length (~0: no such token),
// dense over ids 0..max_id, and the token bytes; built once per device.
// Kernels: k_dec_len (token lengths, block-local exclusive scan, first bad
// token), k_scan_totals (scan.cuh: block totals -> block bases, one CTA), k_dec_copy
// (bytes gathered to their output position), k_dec_rows (row byte offsets).
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
__device__ __forceinline__ bool dec_entry(const DecodeArgs& a, uint32_t id, const uint8_t*& src, uint64_t& len) {
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
    return true;
  }
  if (k < 0) return false;
  len = a.sp_len[k];
  src = a.sp_blob + a.sp_off[k];
  return true;
}

__global__ void __launch_bounds__(kDecThreads) k_dec_len(DecodeArgs a) {
  __shared__ uint64_t s_warp[kDecThreads / 32];
  const uint64_t i = blockIdx.x * uint64_t(kDecThreads) + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t len = 0;
  if (i < a.n_ids) {
    const uint8_t* src;
    if (!dec_entry(a, a.ids[i], src, len)) {
      len = 0;
      atomicMin(reinterpret_cast<unsigned long long*>(a.err), (unsigned long long)i);
    }
  }
  uint64_t inc = len;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) s_warp[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint64_t x = lane < kDecThreads / 32 ? s_warp[lane] : 0;
    uint64_t xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, xi, d);
      if (lane >= d) xi += u;
    }
    if (lane < kDecThreads / 32) s_warp[lane] = xi - x;
    if (lane == 31) a.block_sums[blockIdx.x] = xi;
  }
  __syncthreads();
  if (i < a.n_ids) a.pos[i] = s_warp[wid] + inc - len;
}

__global__ void __launch_bounds__(kDecThreads) k_dec_copy(DecodeArgs a) {
  const uint64_t i = blockIdx.x * uint64_t(kDecThreads) + threadIdx.x;
  if (i >= a.n_ids) return;
  const uint8_t* src;
  uint64_t len;
  if (!dec_entry(a, a.ids[i], src, len)) return;
  const uint64_t pos = a.block_sums[blockIdx.x] + a.pos[i];
  for (uint64_t k = 0; k < len && pos + k < a.cap; ++k) a.out[pos + k] = __ldg(src + k);
}

__global__ void k_dec_rows(DecodeArgs a) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (r > a.n_rows) return;
  const uint64_t t = a.tok_off[r] - a.tok_off[0];
  const uint64_t b = t / kDecThreads;
  a.out_off[r] = t >= a.n_ids ? a.block_sums[a.n_blocks] : a.block_sums[b] + a.pos[t];
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

__global__ void __launch_bounds__(kDecThreads) k_json_tok(JsonArgs a) {
  const uint64_t i = blockIdx.x * uint64_t(kDecThreads) + threadIdx.x;
  const uint64_t v = i < a.n_ids ? ndigits(a.ids[i]) + 1 : 0;
  const uint64_t e = block_excl(v, a.tok_sums);
  if (i < a.n_ids) a.tok_pos[i] = e;
}

__global__ void __launch_bounds__(kDecThreads) k_json_row(JsonArgs a) {
  const uint64_t r = blockIdx.x * uint64_t(kDecThreads) + threadIdx.x;
  uint64_t v = 0;
  if (r < a.n_rows) {
    const uint64_t len = a.tok_off[r + 1] - a.tok_off[r];
    v = 18 + ndigits(len) - (len > 0 ? 1 : 0);
  }
  const uint64_t e = block_excl(v, a.row_sums);
  if (r < a.n_rows) a.row_pos[r] = e;
}

__device__ __forceinline__ uint64_t tok_text_pos(const JsonArgs& a, uint64_t i) {  // exclusive, i <= n_ids
  return i >= a.n_ids ? a.tok_sums[a.n_tok_blocks] : a.tok_sums[i / kDecThreads] + a.tok_pos[i];
}

// Warp per row: lane per token; lane 0 writes the frame.
__global__ void k_json_write(JsonArgs a) {
  const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x / 32);
  const int lane = threadIdx.x & 31;
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x / 32) + (threadIdx.x >> 5); r < a.n_rows; r += nw) {
    const uint64_t t0 = a.tok_off[r] - a.tok_off[0], t1 = a.tok_off[r + 1] - a.tok_off[0];
    const uint64_t len = t1 - t0;
    const uint64_t p0 = tok_text_pos(a, t0);
    const uint64_t start = a.row_sums[r / kDecThreads] + a.row_pos[r] + p0;
    for (uint64_t i = t0 + lane; i < t1; i += 32) {
      const uint32_t id = a.ids[i];
      const uint32_t d = ndigits(id);
      const uint64_t pos = start + 8 + (tok_text_pos(a, i) - p0);
      put_digits(a.out, pos, a.cap, id, d);
      if (i + 1 < t1 && pos + d < a.cap) a.out[pos + d] = ',';
    }
    if (lane == 0) {
      put_str(a.out, start, a.cap, "{\"ids\":[", 8);
      const uint64_t q = start + 8 + (tok_text_pos(a, t1) - p0) - (len > 0 ? 1 : 0);
      put_str(a.out, q, a.cap, "],\"len\":", 8);
      const uint32_t d = ndigits(len);
      put_digits(a.out, q + 8, a.cap, len, d);
      put_str(a.out, q + 8 + d, a.cap, "}\n", 2);
    }
  }
}

}  // namespace

void launch_jsonl(const JsonArgs& a, int sm_count, cudaStream_t s) {
  if (a.n_ids) {
    k_json_tok<<<unsigned(a.n_tok_blocks), kDecThreads, 0, s>>>(a);
    k_scan_totals<<<1, 1024, 0, s>>>(a.tok_sums, a.n_tok_blocks);
  } else {
    cudaMemsetAsync(a.tok_sums, 0, 8, s);
  }
  if (a.n_rows) {
    k_json_row<<<unsigned(a.n_row_blocks), kDecThreads, 0, s>>>(a);
    k_scan_totals<<<1, 1024, 0, s>>>(a.row_sums, a.n_row_blocks);
    k_json_write<<<unsigned(sm_count * 8), 256, 0, s>>>(a);
  } else {
    cudaMemsetAsync(a.row_sums, 0, 8, s);
  }
}

void launch_decode(const DecodeArgs& a, cudaStream_t s) {
  if (a.n_ids) {
    k_dec_len<<<unsigned(a.n_blocks), kDecThreads, 0, s>>>(a);
    k_scan_totals<<<1, 1024, 0, s>>>(a.block_sums, a.n_blocks);
    k_dec_copy<<<unsigned(a.n_blocks), kDecThreads, 0, s>>>(a);
  } else {
    cudaMemsetAsync(a.block_sums, 0, 8, s);
  }
  k_dec_rows<<<unsigned((a.n_rows + 1 + 255) / 256), 256, 0, s>>>(a);
}

}  // namespace bbpe
