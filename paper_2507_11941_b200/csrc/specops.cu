// specops.cu -- the reference's spec-level operations on the device: a
// per-phase replay of one block_bpe pass (block_engine.hpp:189-256), with the
// same contract checks and ContractViolation messages.
//
//   pair_ranks       (189-199)  k_spec_ranks   thread per pair: probe -> original rank
//   min_rank_reduce  (201-206)  k_spec_min     grid-stride min, warp REDUX + atomicMin
//   mark_merges      (211-220)  k_spec_runs    thread per run start of the rank-m pairs,
//                                              left-greedy alternate flags (fill_merge_flags 103-128)
//   exclusive_scan   (223-235)  k_spec_check   flags 0/1 and no two adjacent (lowest index wins)
//                               k_spec_scan    one CTA, carry across 1024-element chunks
//   compact          (238-256)  k_spec_check_offsets, then k_spec_compact (compact_into 166-182:
//                                              ContractViolation when a flagged pair is not a merge)
// These are the test/debug surface of the engine (the encode path never calls
// them); the kernels are simple and one-thread-per-element on purpose.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
#include "probe.cuh"

namespace bbpe {
namespace {

__global__ void k_spec_ranks(const uint32_t* tok, uint64_t n, DevTable T, uint32_t* ranks) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i + 1 < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t rk = probe(T, tok[i], tok[i + 1]);
    ranks[i] = rk == kNoRank ? kNoRank : T.rank_orig[rk_rank(T, rk)];
  }
}

__global__ void k_spec_min(const uint32_t* ranks, uint64_t n, uint32_t* out) {
  uint32_t m = kNoRank;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    m = min(m, ranks[i]);
  m = __reduce_min_sync(0xFFFFFFFFu, m);
  if ((threadIdx.x & 31) == 0 && m != kNoRank) atomicMin(out, m);
}

// ranks: n - 1 pairs. A run of rank-m pairs starting at i marks f[i+1],
// f[i+3], ... while the run lasts (f[0] = 0; f[j+1] = r[j] == m && !f[j]).
__global__ void k_spec_runs(const uint32_t* ranks, uint64_t n, uint32_t m, uint8_t* flags) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i + 1 < n; i += uint64_t(gridDim.x) * blockDim.x) {
    if (ranks[i] != m || (i > 0 && ranks[i - 1] == m)) continue;
    for (uint64_t j = i; j + 1 < n && ranks[j] == m; j += 2) {
      flags[j + 1] = 1;
      if (j + 1 + 1 >= n || ranks[j + 1] != m) break;
    }
  }
}

// err = min over failing i of (i << 1 | kind): kind 0 = flag value > 1,
// kind 1 = flags i-1 and i both set (the reference checks in that order).
__global__ void k_spec_check(const uint8_t* flags, uint64_t n, unsigned long long* err) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint8_t f = flags[i];
    if (f > 1) atomicMin(err, (unsigned long long)(i << 1));
    else if (i > 0 && f && flags[i - 1]) atomicMin(err, (unsigned long long)((i << 1) | 1));
  }
}

// Exclusive prefix sum of u8 flags into u32 offsets; one CTA of 1024 threads.
__global__ void __launch_bounds__(1024) k_spec_scan(const uint8_t* flags, uint64_t n, uint32_t* offsets,
                                                    uint32_t* total) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint64_t base = 0; base < n; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint32_t v = i < n ? flags[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t s = warp_sums[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, d);
        if (lane >= d) s += y;
      }
      warp_sums[lane] = s;
    }
    __syncthreads();
    const uint32_t before = carry + (wid ? warp_sums[wid - 1] : 0u) + x - v;
    if (i < n) offsets[i] = before;
    __syncthreads();
    if (threadIdx.x == 1023) carry = before + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_spec_check_offsets(const uint32_t* offsets, const uint32_t* scan, uint64_t n,
                                     unsigned long long* err) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    if (offsets[i] != scan[i]) atomicMin(err, (unsigned long long)i);
}

// compact_into (166-182): dense tokens for the probe, original ids out.
__global__ void k_spec_compact(const uint32_t* dtok, const uint32_t* orig, const uint8_t* flags,
                               const uint32_t* offsets, uint64_t n, DevTable T, uint32_t* out,
                               unsigned long long* err) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    if (flags[i]) continue;
    const uint64_t dst = i - offsets[i];
    if (i + 1 < n && flags[i + 1]) {
      const uint32_t rk = probe(T, dtok[i], dtok[i + 1]);
      if (rk == kNoRank) {
        atomicMin(err, (unsigned long long)i);
        continue;
      }
      const uint32_t m = rk_merged(T, rk);
      out[dst] = T.d2id ? T.d2id[m] : m;
    } else {
      out[dst] = orig[i];
    }
  }
}

constexpr int kSpecThreads = 256;
int spec_grid(uint64_t n) { return int(std::min<uint64_t>((n + kSpecThreads - 1) / kSpecThreads + 1, 4096)); }

}  // namespace

void launch_spec_ranks(const uint32_t* tok, uint64_t n, const DevTable& t, uint32_t* ranks, cudaStream_t s) {
  k_spec_ranks<<<spec_grid(n), kSpecThreads, 0, s>>>(tok, n, t, ranks);
}
void launch_spec_min(const uint32_t* ranks, uint64_t n, uint32_t* out, cudaStream_t s) {
  k_spec_min<<<spec_grid(n), kSpecThreads, 0, s>>>(ranks, n, out);
}
void launch_spec_runs(const uint32_t* ranks, uint64_t n, uint32_t m, uint8_t* flags, cudaStream_t s) {
  k_spec_runs<<<spec_grid(n), kSpecThreads, 0, s>>>(ranks, n, m, flags);
}
void launch_spec_check(const uint8_t* flags, uint64_t n, unsigned long long* err, cudaStream_t s) {
  k_spec_check<<<spec_grid(n), kSpecThreads, 0, s>>>(flags, n, err);
}
void launch_spec_scan(const uint8_t* flags, uint64_t n, uint32_t* offsets, uint32_t* total, cudaStream_t s) {
  k_spec_scan<<<1, 1024, 0, s>>>(flags, n, offsets, total);
}
void launch_spec_check_offsets(const uint32_t* offsets, const uint32_t* scan, uint64_t n, unsigned long long* err,
                               cudaStream_t s) {
  k_spec_check_offsets<<<spec_grid(n), kSpecThreads, 0, s>>>(offsets, scan, n, err);
}
void launch_spec_compact(const uint32_t* dtok, const uint32_t* orig, const uint8_t* flags, const uint32_t* offsets,
                         uint64_t n, const DevTable& t, uint32_t* out, unsigned long long* err, cudaStream_t s) {
  k_spec_compact<<<spec_grid(n), kSpecThreads, 0, s>>>(dtok, orig, flags, offsets, n, t, out, err);
}

}  // namespace bbpe
