// pretok.cu -- the GPT-2 pattern splitter on the device:
// pattern_pretokenize("gpt2") of every row (reference pretokenize.hpp:79-243,
// the dedicated matcher for
//   's|'t|'re|'ve|'m|'ll|'d| ?\p{L}+| ?\p{N}+| ?[^\s\p{L}\p{N}]+|\s+(?!\S)|\s+
// with the reference's lenient UTF-8 decoder, merge_table.hpp:77-103, and its
// unicode category tables, pretokenize.hpp:94-150). Warp per tile, lane per
// span (see k_pretok_gpt2); chunk starts go to a bitmap that k_pieces ORs
// into its piece boundaries, so merges run within each chunk
// (encode_reference's pattern mode, ref_engines.hpp:119-146).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"
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
template <typename Txt>
__device__ __forceinline__ uint32_t next_utf8(const Txt& s, uint64_t n, uint64_t& pos) {
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

__host__ __device__ constexpr int ascii_class(uint32_t c) {
  return ((c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z')) ? kLetter
         : (c >= '0' && c <= '9')                            ? kNumber
         : (c == ' ' || (c >= 0x09 && c <= 0x0d))            ? kSpace
                                                             : kOther;
}

// The ASCII classes in shared memory (accessors carry the pointer): one load
// instead of compare chains, and no divergent branch per character.
__device__ __forceinline__ void build_ascii_classes(uint8_t* cls) {
  for (int i = threadIdx.x; i < 128; i += blockDim.x) cls[i] = uint8_t(ascii_class(i));
  __syncthreads();
}

// classify (pretokenize.hpp:157-165) with is_letter / is_number / is_space (133-149).
template <typename Txt>
__device__ __forceinline__ int classify(const Txt& s, uint64_t n, uint64_t pos, uint64_t& adv) {
  const uint32_t b0 = s[pos];
  if (b0 < 0x80) {
    adv = 1;
    return s.cls[b0];
  }
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

template <typename Txt>
__device__ __forceinline__ uint64_t run_of(const Txt& s, uint64_t n, int want, uint64_t p) {
  while (p < n) {
    uint64_t adv;
    if (classify(s, n, p, adv) != want) break;
    p += adv;
  }
  return p;
}

// gpt2_chunk_end (pretokenize.hpp:168-219): end of the match starting at pos.
template <typename Txt>
__device__ __forceinline__ uint64_t gpt2_chunk_end(const Txt& s, uint64_t n, uint64_t pos) {
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
  //  ?\p{L}+  and  ?\p{N}+  and  ?[^\s\p{L}\p{N}]+ : the three alternatives
  // test the same first character (after the optional space), so the one
  // that can match is that character's class.
  {
    uint64_t p = pos, advp = adv0;
    int cp = c0;
    if (s[p] == ' ' && p + 1 < n) {
      ++p;
      cp = classify(s, n, p, advp);
    }
    if (cp != kSpace) return run_of(s, n, cp, p + advp);
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

// Short rows (<= kShortRow bytes): thread per row, the reference scan as is.
constexpr uint64_t kShortRow = 4096;

// A 16-byte register window over 16-aligned global bytes: a sequential scan
// loads memory once per 16 bytes instead of once per byte (the row scan was
// load-latency bound). The last partial block is read bytewise (no read past
// `total`).
struct RegWin {
  const uint8_t* g;
  const uint8_t* cls;  // ascii_class table (shared memory)
  uint64_t total;
  mutable uint64_t base;
  mutable uint4 v;
  __device__ __forceinline__ uint8_t operator[](uint64_t p) const {
    const uint64_t b = p & ~15ull;
    if (b != base) {
      base = b;
      if (b + 16 <= total) {
        v = __ldg(reinterpret_cast<const uint4*>(g + b));
      } else {
        uint32_t w[4] = {0, 0, 0, 0};
        for (uint64_t i = b; i < total; ++i) w[(i - b) >> 2] |= uint32_t(g[i]) << (8 * ((i - b) & 3));
        v = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    const uint32_t k = uint32_t(p) & 15;
    const uint32_t x = (k & 8) ? ((k & 4) ? v.w : v.z) : ((k & 4) ? v.y : v.x);
    return uint8_t(x >> (8 * (k & 3)));
  }
};

struct Plain;
template <typename Txt>
__device__ __forceinline__ Txt make_txt(const uint8_t* bytes, const uint8_t* cls, uint64_t total);
template <>
__device__ __forceinline__ RegWin make_txt<RegWin>(const uint8_t* bytes, const uint8_t* cls, uint64_t total) {
  return RegWin{bytes, cls, total, ~0ull, make_uint4(0, 0, 0, 0)};
}

template <typename Txt>
__global__ void __launch_bounds__(256) k_pretok_rows(const uint8_t* bytes, uint64_t total, const uint64_t* offsets,
                                                     uint64_t n_rows, uint32_t* chunkbits, uint32_t* long_flag) {
  __shared__ uint8_t s_cls[128];
  build_ascii_classes(s_cls);
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const Txt txt = make_txt<Txt>(bytes, s_cls, total);
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n_rows; r += stride) {
    const uint64_t rs = offsets[r], re = offsets[r + 1];
    if (re - rs > kShortRow) {  // long rows: k_pretok_gpt2
      *long_flag = 1;
      continue;
    }
    uint64_t word = ~0ull;
    uint32_t bits = 0;
    for (uint64_t pos = rs; pos < re;) {
      if ((pos >> 5) != word) {
        if (bits) atomicOr(&chunkbits[word], bits);
        word = pos >> 5;
        bits = 0;
      }
      bits |= 1u << (pos & 31);
      pos = gpt2_chunk_end(txt, re, pos);
    }
    if (bits) atomicOr(&chunkbits[word], bits);
  }
}

// Long rows (> kShortRow bytes): thread per kSpan-byte span. A restart point
// is a position where the reference's left-to-right scan always starts a
// chunk, whatever came before:
//  * a row start;
//  * p with ' ' at p after an ASCII non-whitespace character at p-1: the
//    chunk holding p-1 is a letter/number/other run or a contraction, none of
//    which contains a space, so it ends at p;
//  * p with '\n' at p-1 and a non-whitespace character at p: a whitespace
//    chunk never extends past non-whitespace, and '\n' is never an optional
//    leading space.
// Both need p-1 to start a character under the reference's lenient UTF-8
// decoding (next_utf8 decides a length from the lead byte alone): no byte
// >= 0xC0 in p-4..p-2 within the row. A thread scans chunks from the first
// restart point of a long row in its span until it reaches a restart point
// at or past the span end (the next span's first one); spans without one are
// covered by an earlier thread. Chunk starts go to `chunkbits` (row starts
// stay read-only).
constexpr uint64_t kSpan = 1024;

// Plain byte loads (unaligned input).
struct Plain {
  const uint8_t* g;
  const uint8_t* cls;  // ascii_class table (shared memory)
  __device__ __forceinline__ uint8_t operator[](uint64_t p) const { return g[p]; }
};

template <>
__device__ __forceinline__ Plain make_txt<Plain>(const uint8_t* bytes, const uint8_t* cls, uint64_t) {
  return Plain{bytes, cls};
}

struct Bits {  // row-start bitmap
  const uint32_t* g;
  __device__ __forceinline__ bool operator()(uint64_t p) const { return (g[p >> 5] >> (p & 31)) & 1u; }
  __device__ __forceinline__ uint32_t word(uint64_t x) const { return g[x]; }
};

// min(next row start after p, p + lim, total): scans at most lim / 32 + 1 words.
__device__ __forceinline__ uint64_t row_end_near(const Bits& row, uint64_t total, uint64_t p, uint64_t lim) {
  const uint64_t cap = min(total, p + lim);
  for (uint64_t q = p + 1; q < cap; q = (q | 31) + 1) {
    const uint32_t v = row.word(q >> 5) >> (q & 31);
    if (v) return min(cap, q + __ffs(v) - 1);
  }
  return cap;
}

// First row index s with offsets[s] > p (p < total): the row holding p is s - 1
// and ends at offsets[s]. tile_first[t] (k_tile_first) brackets s in
// [tile_first[t], tile_first[t + 1]] for t = p / kTile.
struct Rows {
  const uint64_t* off;
  const uint64_t* tile_first;
  uint64_t n_rows, num_tiles;
  __device__ __forceinline__ uint64_t upper(uint64_t p) const {
    const uint64_t t = p / kTile;
    uint64_t lo = tile_first[t], hi = min(n_rows, t + 1 < num_tiles ? tile_first[t + 1] : n_rows);
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (off[m] > p) hi = m;
      else lo = m + 1;
    }
    return lo;
  }
};

template <typename Txt>
__device__ __forceinline__ bool is_restart(const Txt& s, const Bits& row, uint64_t total, uint64_t p) {
  if (p >= total) return false;
  if (row(p)) return true;
  if (p == 0) return true;
  const uint8_t a = s[p - 1], c = s[p];
  const bool sp = c == ' ' && a >= 0x21 && a <= 0x7E;
  if (!sp && a != '\n') return false;
  for (uint64_t k = 2; k <= 4 && p >= k; ++k) {
    if (row(p - k + 1)) break;  // earlier bytes belong to the previous row
    if (s[p - k] >= 0xC0) return false;  // p-1 might continue a multi-byte character
  }
  if (sp) return true;
  uint64_t adv;  // decoded within the row, like the reference (text = the row)
  return classify(s, row_end_near(row, total, p, 8), p, adv) != kSpace;  // reads < 8 bytes ahead
}

// Row [rs, re) of a restart point p, skipping short rows: returns false when
// no long row has a restart point in [p, se).
template <typename Txt>
__device__ __forceinline__ bool first_long_restart(const Txt& txt, const Bits& row, const Rows& rows,
                                                   uint64_t total, uint64_t short_row, uint64_t se, uint64_t& pos,
                                                   uint64_t& re) {
  for (;;) {
    uint64_t p = pos;
    while (p < se && !is_restart(txt, row, total, p)) ++p;
    if (p >= se) return false;
    const uint64_t u = rows.upper(p);
    re = rows.off[u];
    pos = p;
    if (re - rows.off[u - 1] > short_row) return true;
    pos = re;  // a short row (k_pretok_rows): its end is the next restart point
  }
}

template <typename Txt>
__global__ void __launch_bounds__(256) k_pretok_spans(const uint8_t* bytes, uint64_t total, const uint32_t* rowbits,
                                                      Rows rows, uint32_t* chunkbits, uint64_t short_row,
                                                      const uint32_t* long_flag) {
  if (short_row && *reinterpret_cast<const volatile uint32_t*>(long_flag) == 0) return;  // no long row
  __shared__ uint8_t s_cls[128];
  build_ascii_classes(s_cls);
  const Txt txt = make_txt<Txt>(bytes, s_cls, total);
  const Bits row{rowbits};
  const uint64_t spans = (total + kSpan - 1) / kSpan, stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t sp = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; sp < spans; sp += stride) {
    const uint64_t se = min(total, (sp + 1) * kSpan);
    uint64_t pos = sp * kSpan, re = 0;
    if (!first_long_restart(txt, row, rows, total, short_row, se, pos, re)) continue;
    uint64_t word = ~0ull;
    uint32_t bits = 0;
    for (;;) {
      if (pos >= re) {  // the next row's start is a restart point
        if (re >= total || re >= se) break;
        pos = re;
        if (!first_long_restart(txt, row, rows, total, short_row, se, pos, re)) break;
      }
      if (pos >= se && is_restart(txt, row, total, pos)) break;  // the next span's
      if ((pos >> 5) != word) {
        if (bits) atomicOr(&chunkbits[word], bits);
        word = pos >> 5;
        bits = 0;
      }
      bits |= 1u << (pos & 31);
      pos = gpt2_chunk_end(txt, re, pos);
    }
    if (bits) atomicOr(&chunkbits[word], bits);
  }
}

}  // namespace

void launch_pretok_gpt2(const uint8_t* d_bytes, const uint64_t* d_offsets, const uint64_t* d_tile_first,
                        uint64_t n_rows, uint64_t total, const uint32_t* d_rowbits, uint32_t* d_chunkbits,
                        uint32_t* d_long_flag, int sm_count, cudaStream_t s) {
  const uint64_t tiles = (total + kTile - 1) / kTile;
  if (!tiles) return;
  const Rows rows{d_offsets, d_tile_first, n_rows, tiles};
  const unsigned grid = unsigned(sm_count * 8);
  if ((reinterpret_cast<uintptr_t>(d_bytes) & 15) == 0) {  // 16-byte register windows
    k_pretok_rows<RegWin><<<grid, 256, 0, s>>>(d_bytes, total, d_offsets, n_rows, d_chunkbits, d_long_flag);
    k_pretok_spans<RegWin><<<grid, 256, 0, s>>>(d_bytes, total, d_rowbits, rows, d_chunkbits, kShortRow,
                                                d_long_flag);
  } else {
    k_pretok_rows<Plain><<<grid, 256, 0, s>>>(d_bytes, total, d_offsets, n_rows, d_chunkbits, d_long_flag);
    k_pretok_spans<Plain><<<grid, 256, 0, s>>>(d_bytes, total, d_rowbits, rows, d_chunkbits, kShortRow,
                                               d_long_flag);
  }
}

}  // namespace bbpe
