// scan.cuh -- one-CTA exclusive scan of per-block totals (shared by
// decode.cu and specials.cu). Internal linkage: each includer gets its copy.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bbpe {
namespace {

// One CTA: exclusive scan of the block totals in place, total at [n_blocks].
__global__ void __launch_bounds__(1024) k_scan_totals(uint64_t* sums, uint64_t n_blocks) {
  __shared__ uint64_t s_warp[32];
  __shared__ uint64_t s_carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint64_t b0 = 0; b0 < n_blocks; b0 += 1024) {
    const uint64_t b = b0 + threadIdx.x;
    const uint64_t v = b < n_blocks ? sums[b] : 0;
    uint64_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, inc, d);
      if (lane >= d) inc += u;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      const uint64_t x = s_warp[lane];
      uint64_t xi = x;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t u = __shfl_up_sync(0xFFFFFFFFu, xi, d);
        if (lane >= d) xi += u;
      }
      s_warp[lane] = xi - x;
    }
    __syncthreads();
    const uint64_t carry = s_carry;
    if (b < n_blocks) sums[b] = carry + s_warp[wid] + inc - v;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = carry + s_warp[wid] + inc;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[n_blocks] = s_carry;
}

}  // namespace
}  // namespace bbpe
