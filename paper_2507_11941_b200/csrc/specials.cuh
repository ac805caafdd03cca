// specials.cuh -- device split of special tokens and the stitched encode_batch
// rows (specials.cu). SURVEY 8f(1).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bbpe {

// The special-token set on the device, entries longest first (the order
// SpecialTokenSet::add keeps, merge_table.hpp:311-319).
struct SpecArgs {
  const uint8_t* blob;
  const uint32_t* off;    // n + 1
  const uint32_t* id;     // n
  const uint32_t* first;  // 8 words: bitmap of first bytes
  uint32_t n;
};

// v[0..n) -> exclusive prefix sums in place, v[n] = total. sums: scan_sums_len(n) words.
uint64_t scan_sums_len(uint64_t n);
void launch_scan_u64(uint64_t* v, uint64_t n, uint64_t* sums, cudaStream_t s);

// cand bit p: some special matches at byte p (row ends ignored: a superset).
void launch_sp_candidates(const uint8_t* bytes, uint64_t total, SpecArgs sp, uint32_t* cand, int sm_count,
                          cudaStream_t s);
// Greedy split of each row (split_specials, pretokenize.hpp:32-57):
// cnt[r] = specials matched, lit[r] = literal bytes.
void launch_sp_rows(const uint8_t* bytes, const uint64_t* offsets, uint64_t n_rows, SpecArgs sp,
                    const uint32_t* cand, uint64_t* cnt, uint64_t* lit, cudaStream_t s);
// With match_base = scan(cnt), lit_base = scan(lit): row r owns literal
// segments r + match_base[r] + j, j = 0..cnt[r] (empty ones included), their
// offsets in the compacted literal bytes (seg_off, n_seg + 1), their source
// starts (seg_src), and the special ids sp_ids[match_base[r] + j].
// inplace != 0 (every byte has a token, so special bytes may be encoded and
// dropped): no compaction, row r owns segments r + 2 match_base[r] + i,
// literal at even i, special at odd i, offsets into the input bytes.
void launch_sp_emit(const uint8_t* bytes, const uint64_t* offsets, uint64_t n_rows, SpecArgs sp,
                    const uint32_t* cand, const uint64_t* match_base, const uint64_t* lit_base, uint64_t* seg_off,
                    uint64_t* seg_src, uint32_t* sp_ids, int inplace, cudaStream_t s);
void launch_sp_copy(const uint8_t* bytes, uint64_t n_seg, const uint64_t* seg_off, const uint64_t* seg_src,
                    uint8_t* compact, int sm_count, cudaStream_t s);
// out_len[r] = bos + literal tokens + specials + eos (then scanned into offsets).
// stride: 1 (compacted segments) or 2 (in place: literal segments at even offsets).
void launch_sp_lengths(uint64_t n_rows, const uint64_t* match_base, const uint64_t* seg_tok_off, int add_bos,
                       int add_eos, int stride, uint64_t* out_len, cudaStream_t s);
void launch_sp_stitch(uint64_t n_rows, const uint64_t* match_base, const uint64_t* seg_tok_off,
                      const uint32_t* seg_ids, const uint32_t* sp_ids, const uint64_t* out_off, uint32_t bos_id,
                      uint32_t eos_id, int stride, uint32_t* out_ids, int sm_count, cudaStream_t s);

}  // namespace bbpe
