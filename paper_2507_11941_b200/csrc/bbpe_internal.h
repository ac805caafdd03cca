// bbpe_internal.h -- shared host/device definitions of the B200 BlockBPE engine.
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/bbpe_b200.h"

namespace bbpe {

constexpr uint32_t kNoRank = 0xFFFFFFFFu;     // block_engine.hpp:16
constexpr uint32_t kInvalidToken = 0xFFFFFFFFu;  // merge_table.hpp:22
constexpr uint64_t kEmptySlot = ~0ull;
#ifndef BBPE_PAIR_SLOTS_PER_MERGE
#define BBPE_PAIR_SLOTS_PER_MERGE 8  // pair-table slots per merge (load <= 1/8: full home buckets are rare, so misses end at one 32-byte load)
#endif
constexpr int kBucketSlots = 4;               // 4 x 8 B = one 32 B sector per bucket

// Exceptions mirror the reference taxonomy (types.hpp:32-70); the C-ABI maps
// each to its bbpe_status.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
inline Error usage_error(const std::string& m) { return Error(BBPE_USAGE, m); }
inline Error parse_error(const std::string& m) { return Error(BBPE_PARSE, m); }
inline Error integrity_error(const std::string& m) { return Error(BBPE_INTEGRITY, m); }

// The device view of a merge table, passed by value to every kernel.
//
// Pair key  = (left << id_bits) | right  over DENSE token ids.
// Slot (u64)= (key << rank_bits) | dense_rank, empty = all ones.
// Buckets of 4 slots (32 B, one sector), linear probing bucket to bucket.
// dense_rank = position of the merge in rank order (order preserving, so
// min-rank comparisons are unchanged); r2m[dense_rank] = dense merged id.
struct DevTable {
  const uint64_t* slots = nullptr;
  uint64_t bucket_mask = 0;
  const uint32_t* r2m = nullptr;    // dense rank -> dense merged id
  const uint32_t* d2id = nullptr;   // dense id -> original id (null = identity)
  const uint32_t* lut = nullptr;    // 256: byte -> dense id or kInvalidToken
  const uint32_t* junction = nullptr;  // 2048 words: bit (a<<8|b) set iff some merge spans a|b
  const uint32_t* junction_t = nullptr;  // the same, transposed: bit (b<<8|a) (k_pieces' byte-pair order)
  const uint32_t* lut_out = nullptr;   // 256: byte -> ORIGINAL id of its token, or kInvalidToken
  const uint32_t* rank_orig = nullptr; // dense rank -> original rank (traces)
  // Piece memo (optional): exact encodings of whole pieces that equal a
  // vocabulary token's bytes, computed by this engine at table upload.
  const struct MemoEntry* memo = nullptr;
  uint64_t memo_mask = 0;
  uint32_t id_bits = 0;
  uint32_t rank_bits = 0;
  uint32_t n_merges = 0;
  uint32_t key32 = 0;  // 1: 32-bit pair keys (ids, ranks < 2^16): slot = key32 << 32 | rank << 16 | merged
  uint32_t full_lut = 0;  // 1: every byte value has a token (no invalid-byte checks)
};

// Bucket hash of a 32-bit pair key (murmur3 finaliser).
__host__ __device__ inline uint32_t mix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

// 32-byte memo entry: piece bytes (zero padded), length, 1-2 result tokens
// (original ids: memo results are final output). len == 0 marks an empty slot.
// Single bytes are entries too (one lookup path for every short piece).
constexpr int kMemoMaxLen = 20;
struct MemoEntry {
  uint32_t w[5];
  uint8_t len;
  uint8_t nres;
  uint16_t pad;
  uint32_t res[2];
};
static_assert(sizeof(MemoEntry) == 32, "memo entry is one sector");

// Hash of a piece given as 5 little-endian words (bytes past len are zero):
// the length and the first 12 bytes (99.5% of pieces are shorter; longer ones
// sharing a 12-byte prefix and a length just probe on), one xor-multiply per
// word, then a murmur-style finaliser. Lookups compare all 20 bytes.
__host__ __device__ inline uint32_t memo_hash(const uint32_t* w, uint32_t len) {
  uint32_t h = len * 0x9E3779B9u;
  for (int i = 0; i < 3; ++i) h = (h ^ w[i]) * 0x85EBCA6Bu;
  h ^= h >> 15;
  h *= 0xC2B2AE35u;
  h ^= h >> 13;
  return h;
}

struct DeviceReplica {
  DevTable view;
  void* base = nullptr;  // one cudaMalloc holding every array
  void* memo = nullptr;  // memo slots (separate allocation)
  int memo_state = 0;    // 0 not built, 1 building, 2 built (or not applicable)
  // Decode table (decode.cu), built on first device decode: dec_n u64
  // entries (byte start << 24 | length, ~0 = no token) then the token bytes.
  void* dec = nullptr;
  uint64_t dec_n = 0;
};

}  // namespace bbpe

// The opaque C-ABI table object.
struct bbpe_table {
  // Host copy in reference terms (MergeTable): tokens sorted by id, merges by rank.
  std::vector<uint32_t> ids;
  std::vector<uint64_t> tok_off;
  std::vector<uint8_t> tok_bytes;
  std::unordered_map<uint32_t, uint32_t> index_of;  // id -> position in ids
  std::vector<uint32_t> m_rank, m_left, m_right, m_merged;  // sorted by rank
  uint32_t byte_tokens[256];
  uint64_t base_size = 0;
  uint32_t max_id = 0;
  bool rank_consistent = true;

  // Device layout, built once on the host.
  uint32_t id_bits = 0, rank_bits = 0;
  bool remap = false;
  uint32_t max_dev_id = 0;  // largest id a byte token or merge mentions (non-remapped device ids)
  bool narrow = false;  // 16-bit device working arrays and 32-bit pair keys suffice
  std::unordered_map<uint32_t, uint32_t> dense_of;  // only when remap
  std::vector<uint32_t> dense_to_id;                // only when remap
  std::vector<uint64_t> slots;
  uint64_t bucket_mask = 0;
  std::vector<uint32_t> r2m;       // dense rank -> dense merged
  std::vector<uint32_t> lut;       // 256
  std::vector<uint32_t> junction;  // 2048
  uint64_t junction_count = 0;
  // Host-side pair lookup (rank_of / merged_of) over ORIGINAL ids.
  std::unordered_map<uint64_t, uint32_t> pair_index;  // pack(l,r) -> merge position

  std::mutex mu;
  std::map<int, bbpe::DeviceReplica> replicas;

  uint32_t dense(uint32_t id) const {
    if (!remap) return id;
    auto it = dense_of.find(id);
    return it == dense_of.end() ? bbpe::kInvalidToken : it->second;
  }
};

namespace bbpe {
// table.cpp
void build_device_layout(bbpe_table& t);
const DevTable& table_on_device(const bbpe_table& t, int device);
DeviceReplica& replica_of(const bbpe_table& t, int device);  // after table_on_device
void release_replicas(bbpe_table& t);
uint64_t mix64(uint64_t h);
}  // namespace bbpe
