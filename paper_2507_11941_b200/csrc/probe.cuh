// probe.cuh -- device lookups in the pair table (DevTable, bbpe_internal.h):
// the reference's PairMap::find (merge_table.hpp:168-176) over the device
// layout the host builds (table.cpp). Shared by the encode kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bbpe_internal.h"

namespace bbpe {

__device__ __forceinline__ uint64_t dmix64(uint64_t h) {
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdULL;
  h ^= h >> 33;
  return h;
}

// Probe results ("rk"): for narrow tables (T.key32) rank << 16 | merged id,
// for wide tables the dense rank (merged id = r2m[rank]). Both order like the
// rank (ranks are unique), kNoRank when the pair is not in the table.
__device__ __forceinline__ uint32_t rk_merged(const DevTable& T, uint32_t rk) {
  return T.key32 ? (rk & 0xFFFFu) : __ldg(T.r2m + rk);
}
__device__ __forceinline__ uint32_t rk_rank(const DevTable& T, uint32_t rk) { return T.key32 ? rk >> 16 : rk; }

// Pair -> rk (kNoRank when absent). One 32-byte bucket per step.
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

// Batched probe: issue the bucket loads, resolve later. K32: narrow tables
// (ids < 2^16) with 32-bit keys, slot = key32 << 32 | rank.
struct ProbeReq {
  uint64_t key;
  ulonglong2 s01, s23;
};
template <bool K32>
__device__ __forceinline__ uint64_t probe_bucket(const DevTable& T, uint64_t key) {
  return (K32 ? uint64_t(mix32(uint32_t(key))) : dmix64(key)) & T.bucket_mask;
}
template <bool K32>
__device__ __forceinline__ void probe_issue(ProbeReq& q, const DevTable& T, uint32_t l, uint32_t r) {
  q.key = K32 ? uint64_t((l << 16) | r) : ((uint64_t(l) << T.id_bits) | uint64_t(r));
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(T.slots + probe_bucket<K32>(T, q.key) * kBucketSlots);
  q.s01 = __ldg(p);
  q.s23 = __ldg(p + 1);
}

// Bucket full without a hit: keep probing linearly (rare at load <= 0.5).
template <bool K32>
__device__ __noinline__ uint32_t probe_overflow(const uint64_t* slots, uint64_t bucket_mask, uint32_t rank_bits,
                                                uint64_t key, uint64_t b) {
  const uint64_t rmask = (1ull << rank_bits) - 1;
  for (;;) {
    b = (b + 1) & bucket_mask;
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(slots + b * kBucketSlots);
    const ulonglong2 x = __ldg(p), y = __ldg(p + 1);
    const uint64_t t[4] = {x.x, x.y, y.x, y.y};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (t[j] == kEmptySlot) return kNoRank;
      if (K32 ? (uint32_t(t[j] >> 32) == uint32_t(key)) : ((t[j] >> rank_bits) == key))
        return K32 ? uint32_t(t[j]) : static_cast<uint32_t>(t[j] & rmask);
    }
  }
}

template <bool K32>
__device__ __forceinline__ uint32_t probe_resolve(const ProbeReq& q, const DevTable& T) {
  // Branch-free over the bucket (both halves of the 32-byte load are used
  // unconditionally, so the compiler cannot sink one behind the other): a key
  // occupies at most one slot and slots fill left to right, so the result is
  // the matching slot, else no rank if the bucket has an empty slot, else the
  // next bucket (rare at load <= 0.5).
  const uint64_t s[4] = {q.s01.x, q.s01.y, q.s23.x, q.s23.y};
  uint32_t res = kNoRank;
  bool any_empty = false;
#pragma unroll
  for (int j = 3; j >= 0; --j) {
    const bool hit = K32 ? (uint32_t(s[j] >> 32) == uint32_t(q.key)) : ((s[j] >> T.rank_bits) == q.key);
    const uint32_t v = K32 ? uint32_t(s[j]) : static_cast<uint32_t>(s[j] & ((1ull << T.rank_bits) - 1));
    res = hit ? v : res;
    any_empty |= s[j] == kEmptySlot;
  }
  if (res != kNoRank || any_empty) return res;
  return probe_overflow<K32>(T.slots, T.bucket_mask, T.rank_bits, q.key, probe_bucket<K32>(T, q.key));
}

}  // namespace bbpe
