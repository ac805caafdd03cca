// epilogue.cu -- encode_batch's padded BatchEncoding on the device
// (reference batch.hpp:64-126): row r = [bos] + its CSR ids +
// [eos], right-truncated to max_len (truncated_rows counts the cut rows),
// written into N x max_len ids (pad_id elsewhere), u32 lengths and a u8 mask.
#include <cuda_runtime.h>

#include <cstdint>

#include "epilogue.cuh"

namespace bbpe {
namespace {

// Widest row (ids + extra BOS/EOS slots).
__global__ void k_row_max(const uint64_t* off, uint64_t n, uint32_t extra, unsigned long long* out) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  unsigned long long v = r < n ? (off[r + 1] - off[r]) + extra : 0;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, d));
  if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// Lengths and the truncated-row count (thread per row).
__global__ void k_pad_lengths(PadArgs a) {
  const uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  bool cut = false;
  if (r < a.n_rows) {
    const uint64_t len = (a.off[r + 1] - a.off[r]) + (a.bos != kNoId) + (a.eos != kNoId);
    cut = len > a.max_len;
    a.lengths[r] = uint32_t(cut ? a.max_len : len);
  }
  const unsigned m = __ballot_sync(0xFFFFFFFFu, cut);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(a.truncated, (unsigned long long)__popc(m));
}

// The N x max_len matrix, one thread per 4 consecutive cells of a row.
__global__ void k_pad_fill(PadArgs a) {
  const uint64_t L = a.max_len;
  const uint64_t per_row = (L + 3) / 4;
  const uint64_t total = a.n_rows * per_row;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint32_t nb = a.bos != kNoId ? 1u : 0u;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += stride) {
    const uint64_t r = i / per_row;
    const uint64_t c0 = (i - r * per_row) * 4;
    const uint64_t o0 = a.off[r], body = a.off[r + 1] - o0;
    const uint64_t len = min(body + nb + (a.eos != kNoId ? 1 : 0), L);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t c = c0 + k;
      if (c >= L) break;
      uint32_t v = a.pad;
      if (c < len) {
        if (c < nb) v = a.bos;
        else if (c - nb < body) v = a.ids[o0 + c - nb];
        else v = a.eos;
      }
      a.out_ids[r * L + c] = v;
      a.out_mask[r * L + c] = c < len ? 1 : 0;
    }
  }
}

}  // namespace

void launch_row_max(const uint64_t* d_off, uint64_t n, uint32_t extra, unsigned long long* d_out, cudaStream_t s) {
  cudaMemsetAsync(d_out, 0, 8, s);
  if (n) k_row_max<<<unsigned((n + 255) / 256), 256, 0, s>>>(d_off, n, extra, d_out);
}

void launch_pad(const PadArgs& a, int sm_count, cudaStream_t s) {
  cudaMemsetAsync(a.truncated, 0, 8, s);
  if (!a.n_rows) return;
  k_pad_lengths<<<unsigned((a.n_rows + 255) / 256), 256, 0, s>>>(a);
  if (a.max_len) k_pad_fill<<<unsigned(sm_count * 8), 256, 0, s>>>(a);
}

}  // namespace bbpe
