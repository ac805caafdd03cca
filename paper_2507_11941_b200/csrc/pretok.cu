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

// classify (pretokenize.hpp:157-165) with is_letter / is_number / is_space (133-149).
template <typename Txt>
__device__ __forceinline__ int classify(const Txt& s, uint64_t n, uint64_t pos, uint64_t& adv) {
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
__device__ uint64_t gpt2_chunk_end(const Txt& s, uint64_t n, uint64_t pos) {
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

struct Plain {
  const uint8_t* g;
  __device__ __forceinline__ uint8_t operator[](uint64_t p) const { return g[p]; }
};

__global__ void __launch_bounds__(256) k_pretok_rows(const uint8_t* bytes, const uint64_t* offsets, uint64_t n_rows,
                                                     uint32_t* chunkbits) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const Plain txt{bytes};
  for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < n_rows; r += stride) {
    const uint64_t rs = offsets[r], re = offsets[r + 1];
    if (re - rs > kShortRow || re == rs) continue;  // long rows: k_pretok_gpt2
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

// Long rows: warp per 512-byte tile, lane per 16-byte span. The tile's bytes (with 16
// bytes before and kAhead after) and its row-start bits sit in shared memory
// (coalesced loads); scans that run further read global memory. A restart
// point is a position where the reference's left-to-right scan always starts
// a chunk, whatever came before:
//  * a row start;
//  * p with ' ' at p after an ASCII non-whitespace character at p-1: the
//    chunk holding p-1 is a letter/number/other run or a contraction, none of
//    which contains a space, so it ends at p;
//  * p with '\n' at p-1 and a non-whitespace character at p: a whitespace
//    chunk never extends past non-whitespace, and '\n' is never an optional
//    leading space.
// Both need p-1 to start a character under the reference's lenient UTF-8
// decoding (next_utf8 decides a length from the lead byte alone): no byte
// >= 0xC0 in p-4..p-2 within the row. A lane scans chunks from the first
// restart point in its span until it reaches a restart point at or past the
// span end (the next owner's first one); spans without one are covered by an
// earlier lane. Chunk starts go to `chunkbits` (row starts stay read-only).
constexpr int kAhead = 128;
constexpr int kPreBytes = 16 + kTile + kAhead + 16;  // [b0 - 16, b0 + kTile + kAhead + 16)
constexpr int kPreWords = (kTile + kAhead) / 32 + 2;  // row / chunk bits of [b0 - 32, b0 + kTile + kAhead + 32)

struct __align__(16) PreSmem {
  uint8_t w[kPreBytes];
  uint32_t rb[kPreWords];
  uint32_t cb[kPreWords];
};

// Byte view: shared-memory window, global memory outside it.
struct Text {
  const uint8_t* w;  // window byte 0 = position lo
  const uint8_t* g;
  uint64_t lo, hi;
  __device__ __forceinline__ uint8_t operator[](uint64_t p) const { return p - lo < hi - lo ? w[p - lo] : g[p]; }
};
struct Bits {
  const uint32_t* w;  // window word 0 = word wlo
  const uint32_t* g;
  uint64_t wlo, whi;
  __device__ __forceinline__ bool operator()(uint64_t p) const {
    const uint64_t x = p >> 5;
    const uint32_t v = x - wlo < whi - wlo ? w[x - wlo] : g[x];
    return (v >> (p & 31)) & 1u;
  }
  __device__ __forceinline__ uint32_t word(uint64_t x) const { return x - wlo < whi - wlo ? w[x - wlo] : g[x]; }
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
  __device__ __forceinline__ uint64_t end_of(uint64_t p) const { return off[upper(p)]; }
};

__device__ __forceinline__ bool is_restart(const Text& s, const Bits& row, uint64_t total, uint64_t p) {
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

__global__ void __launch_bounds__(256) k_pretok_gpt2(const uint8_t* bytes, uint64_t total, uint64_t num_tiles,
                                                     const uint32_t* rowbits, Rows rows, uint32_t* chunkbits) {
  __shared__ PreSmem sm[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  PreSmem& S = sm[wid];
  const uint64_t nw = uint64_t(gridDim.x) * 8;
  for (uint64_t tile = blockIdx.x * uint64_t(8) + wid; tile < num_tiles; tile += nw) {
    const uint64_t b0 = tile * kTile;
    const uint64_t lo = b0 >= 16 ? b0 - 16 : 0;
    const uint64_t hi = min(total, b0 + kTile + kAhead + 16);
    constexpr int kVec = kPreBytes / 16;  // 42 16-byte chunks
    static_assert(kPreBytes % 16 == 0 && kVec <= 64, "window chunks");
    if ((reinterpret_cast<uintptr_t>(bytes) & 15) == 0 && b0 >= 16 && hi - lo == uint64_t(kPreBytes)) {
      // Interior tile, aligned input: two 16-byte loads per lane, both in flight.
      const uint4* src = reinterpret_cast<const uint4*>(bytes + lo);
      uint4 v0 = __ldg(src + lane), v1 = make_uint4(0, 0, 0, 0);
      if (lane + 32 < kVec) v1 = __ldg(src + lane + 32);
      reinterpret_cast<uint4*>(S.w)[lane] = v0;
      if (lane + 32 < kVec) reinterpret_cast<uint4*>(S.w)[lane + 32] = v1;
    } else {
      for (uint64_t i = lane; i < hi - lo; i += 32) S.w[i] = bytes[lo + i];
    }
    const uint64_t wlo = b0 / 32 >= 1 ? b0 / 32 - 1 : 0;
    const uint64_t whi = min((total + 31) / 32 + 1, wlo + kPreWords);
    for (uint64_t i = lane; i < whi - wlo; i += 32) {
      S.rb[i] = rowbits[wlo + i];
      S.cb[i] = 0;
    }
    __syncwarp();
    const Text txt{S.w, bytes, lo, hi};
    const Bits row{S.rb, rowbits, wlo, whi};
    const uint64_t sb = b0 + 16 * lane, se = min(total, sb + 16);
    uint64_t pos = se;
    if (sb < se) {  // spans of short rows belong to k_pretok_rows
      const uint64_t u = rows.upper(sb);
      if (rows.off[u] - rows.off[u - 1] <= kShortRow) pos = se + 1;  // skip
    }
    if (pos == se)
      for (uint64_t p = sb; p < se; ++p)
        if (is_restart(txt, row, total, p)) {
          pos = p;
          break;
        }
    if (pos < se) {
      uint64_t re = rows.end_of(pos);
      for (;;) {
        if (pos >= re) {
          if (re >= total) break;
          pos = re;  // the next row's start is a restart point
          re = rows.end_of(pos);
          if (pos >= se) break;
        }
        if (pos >= se && is_restart(txt, row, total, pos)) break;  // the next owner's
        const uint64_t x = pos >> 5;
        if (x - wlo < whi - wlo) atomicOr(&S.cb[x - wlo], 1u << (pos & 31));
        else atomicOr(&chunkbits[x], 1u << (pos & 31));
        pos = gpt2_chunk_end(txt, re, pos);
      }
    }
    __syncwarp();
    for (uint64_t i = lane; i < whi - wlo; i += 32)
      if (S.cb[i]) atomicOr(&chunkbits[wlo + i], S.cb[i]);
    __syncwarp();
  }
}

}  // namespace

void launch_pretok_gpt2(const uint8_t* d_bytes, const uint64_t* d_offsets, const uint64_t* d_tile_first,
                        uint64_t n_rows, uint64_t total, const uint32_t* d_rowbits, uint32_t* d_chunkbits, int sm_count, cudaStream_t s) {
  const uint64_t tiles = (total + kTile - 1) / kTile;
  if (!tiles) return;
  k_pretok_rows<<<unsigned(sm_count * 8), 256, 0, s>>>(d_bytes, d_offsets, n_rows, d_chunkbits);
  const Rows rows{d_offsets, d_tile_first, n_rows, tiles};
  k_pretok_gpt2<<<unsigned(sm_count * 4), 256, 0, s>>>(d_bytes, total, tiles, d_rowbits, rows, d_chunkbits);
}

}  // namespace bbpe
