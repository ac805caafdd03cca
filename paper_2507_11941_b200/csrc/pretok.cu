// pretok.cu -- the GPT-2 pattern splitter on the device:
// pattern_pretokenize("gpt2") of every row (reference pretokenize.hpp:79-243,
// the dedicated matcher for
//   's|'t|'re|'ve|'m|'ll|'d| ?\p{L}+| ?\p{N}+| ?[^\s\p{L}\p{N}]+|\s+(?!\S)|\s+
// with the reference's lenient UTF-8 decoder, merge_table.hpp:77-103, and its
// unicode category tables, pretokenize.hpp:94-150). Thread per row; every
// chunk start is ORed into the row-start bitmap, which k_pieces already treats
// as a piece boundary, so merges run within each chunk (encode_reference's
// pattern mode, ref_engines.hpp:119-146).
#include <cuda_runtime.h>

#include <cstdint>

#include "pretok.cuh"

namespace bbpe {
namespace {

__constant__ uint32_t c_letter[36][2] = {
    {0x00aa, 0x00aa}, {0x00b5, 0x00b5}, {0x00ba, 0x00ba}, {0x00c0, 0x00d6},
    {0x00d8, 0x00f6}, {0x00f8, 0x02c1}, {0x0370, 0x0374}, {0x0376, 0x0377},
    {0x037a, 0x037d}, {0x037f, 0x037f}, {0x0386, 0x0386}, {0x0388, 0x03f5},
    {0x03f7, 0x0481}, {0x048a, 0x052f}, {0x0531, 0x0556}, {0x0561, 0x0587},
    {0x05d0, 0x05ea}, {0x0620, 0x064a}, {0x0671, 0x06d3}, {0x0904, 0x0939},
    {0x0958, 0x0961}, {0x0e01, 0x0e30}, {0x10a0, 0x10c5}, {0x10d0, 0x10fa},
    {0x1e00, 0x1f15}, {0x1f18, 0x1f1d}, {0x1f20, 0x1f45}, {0x1f48, 0x1f4d},
    {0x1f50, 0x1f7d}, {0x1f80, 0x1fb4}, {0x2c60, 0x2c7f}, {0x3041, 0x3096},
    {0x30a1, 0x30fa}, {0x4e00, 0x9fff}, {0xa720, 0xa7ff}, {0xac00, 0xd7a3},
};
__constant__ uint32_t c_number[10][2] = {
    {0x00b2, 0x00b3}, {0x00b9, 0x00b9}, {0x00bc, 0x00be}, {0x0660, 0x0669},
    {0x06f0, 0x06f9}, {0x0966, 0x096f}, {0x0e50, 0x0e59}, {0x2070, 0x2079},
    {0x2080, 0x2089}, {0xff10, 0xff19},
};
__constant__ uint32_t c_space[19] = {
    0x0085, 0x00a0, 0x1680, 0x2000, 0x2001, 0x2002, 0x2003, 0x2004, 0x2005, 0x2006,
    0x2007, 0x2008, 0x2009, 0x200a, 0x2028, 0x2029, 0x202f, 0x205f, 0x3000,
};

enum Cls { kLetter = 0, kNumber = 1, kSpace = 2, kOther = 3 };

// next_utf8 (merge_table.hpp:77-103): lead byte only decides the length;
// continuation bytes are not validated; truncated or invalid -> the byte.
__device__ __forceinline__ uint32_t next_utf8(const uint8_t* s, uint64_t n, uint64_t& pos) {
  const uint32_t c0 = s[pos];
  if (c0 < 0x80) {
    pos += 1;
    return c0;
  }
  if ((c0 >> 5) == 0x6 && pos + 1 < n) {
    const uint32_t cp = ((c0 & 0x1fu) << 6) | (s[pos + 1] & 0x3fu);
    pos += 2;
    return cp;
  }
  if ((c0 >> 4) == 0xe && pos + 2 < n) {
    const uint32_t cp = ((c0 & 0x0fu) << 12) | ((s[pos + 1] & 0x3fu) << 6) | (s[pos + 2] & 0x3fu);
    pos += 3;
    return cp;
  }
  if ((c0 >> 3) == 0x1e && pos + 3 < n) {
    const uint32_t cp = ((c0 & 0x07u) << 18) | ((s[pos + 1] & 0x3fu) << 12) | ((s[pos + 2] & 0x3fu) << 6) |
                        (s[pos + 3] & 0x3fu);
    pos += 4;
    return cp;
  }
  pos += 1;
  return c0;
}

template <int N>
__device__ __forceinline__ bool in_ranges(uint32_t cp, const uint32_t (&r)[N][2]) {
  int lo = 0, hi = N;
  while (lo < hi) {  // in_ranges (pretokenize.hpp:119-131)
    const int mid = (lo + hi) / 2;
    if (cp > r[mid][1]) lo = mid + 1;
    else if (cp < r[mid][0]) hi = mid;
    else return true;
  }
  return false;
}

// classify (pretokenize.hpp:157-165) with is_letter / is_number / is_space (133-149).
__device__ __forceinline__ int classify(const uint8_t* s, uint64_t n, uint64_t pos, uint64_t& adv) {
  uint64_t next = pos;
  const uint32_t cp = next_utf8(s, n, next);
  adv = next - pos;
  if (cp < 0x80) {
    if ((cp >= 'A' && cp <= 'Z') || (cp >= 'a' && cp <= 'z')) return kLetter;
    if (cp >= '0' && cp <= '9') return kNumber;
    if (cp == ' ' || (cp >= 0x09 && cp <= 0x0d)) return kSpace;
    return kOther;
  }
  if (in_ranges(cp, c_letter)) return kLetter;
  if (in_ranges(cp, c_number)) return kNumber;
  for (int i = 0; i < 19; ++i)
    if (cp == c_space[i]) return kSpace;
  return kOther;
}

__device__ __forceinline__ uint64_t run_of(const uint8_t* s, uint64_t n, int want, uint64_t p) {
  while (p < n) {
    uint64_t adv;
    if (classify(s, n, p, adv) != want) break;
    p += adv;
  }
  return p;
}

// gpt2_chunk_end (pretokenize.hpp:168-219): end of the match starting at pos.
__device__ uint64_t gpt2_chunk_end(const uint8_t* s, uint64_t n, uint64_t pos) {
  uint64_t adv0;
  const int c0 = classify(s, n, pos, adv0);
  // 's|'t|'re|'ve|'m|'ll|'d (case-sensitive)
  if (s[pos] == '\'' && pos + 1 < n) {
    const uint8_t c1 = s[pos + 1];
    if (c1 == 's' || c1 == 't' || c1 == 'm' || c1 == 'd') return pos + 2;
    if (pos + 2 < n) {
      const uint8_t c2 = s[pos + 2];
      if ((c1 == 'l' && c2 == 'l') || (c1 == 'r' && c2 == 'e') || (c1 == 'v' && c2 == 'e')) return pos + 3;
    }
  }
  //  ?\p{L}+  and  ?\p{N}+  and  ?[^\s\p{L}\p{N}]+
  for (int want = kLetter; want <= kOther; ++want) {
    if (want == kSpace) continue;
    uint64_t p = pos;
    if (s[p] == ' ' && p + 1 < n) ++p;
    const uint64_t end = run_of(s, n, want, p);
    if (end > p) return end;
  }
  // \s+(?!\S)  then  \s+
  if (c0 == kSpace) {
    uint64_t p = pos, last_start = pos;
    while (p < n) {
      uint64_t adv;
      if (classify(s, n, p, adv) != kSpace) break;
      last_start = p;
      p += adv;
    }
    if (p >= n) return p;                     // trailing whitespace, lookahead holds
    if (last_start > pos) return last_start;  // back off one character, not one byte
    return p;
  }
  return pos + adv0;  // lone unclassifiable byte
}

// Thread per row; chunk-start bits are gathered per 32-bit word and ORed in
// once per word.
__global__ void __launch_bounds__(256) k_pretok_gpt2(const uint8_t* bytes, const uint64_t* offsets, uint64_t n_rows,
                                                     uint32_t* rowbits) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n_rows; r += stride) {
    const uint64_t base = offsets[r], n = offsets[r + 1] - base;
    const uint8_t* s = bytes + base;
    uint64_t word = ~0ull;
    uint32_t bits = 0;
    for (uint64_t pos = 0; pos < n;) {
      const uint64_t g = base + pos;
      if ((g >> 5) != word) {
        if (bits) atomicOr(&rowbits[word], bits);
        word = g >> 5;
        bits = 0;
      }
      bits |= 1u << (g & 31);
      pos = gpt2_chunk_end(s, n, pos);
    }
    if (bits) atomicOr(&rowbits[word], bits);
  }
}

}  // namespace

void launch_pretok_gpt2(const uint8_t* d_bytes, const uint64_t* d_offsets, uint64_t n_rows, uint32_t* d_rowbits,
                        int sm_count, cudaStream_t s) {
  if (n_rows) k_pretok_gpt2<<<unsigned(sm_count * 8), 256, 0, s>>>(d_bytes, d_offsets, n_rows, d_rowbits);
}

}  // namespace bbpe
