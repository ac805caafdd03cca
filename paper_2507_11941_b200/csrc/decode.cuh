// decode.cuh -- device batch decode (decode.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bbpe {

constexpr uint64_t kDecodeBlockTokens = 2048;  // tokens per k_dec_len / k_dec_copy block (256 threads x 8)

struct DecodeArgs {
  const uint32_t* ids;       // n_ids token ids
  const uint64_t* tok_off;   // n_rows + 1 row offsets into ids (relative to tok_off[0])
  uint64_t n_rows;
  uint64_t n_ids;
  const uint64_t* dec;       // dec_n entries: byte start << 24 | length, ~0 = unknown id
  uint64_t dec_n;
  const uint8_t* dec_bytes;
  uint64_t* pos;             // n_ids: byte position of the row-start tokens (k_dec_copy)
  uint32_t* rowstart;        // (n_ids + 31) / 32 words: bit t = token t starts a row
  uint64_t* block_sums;      // n_blocks + 1: block byte totals -> exclusive bases, total last
  uint64_t n_blocks;
  uint8_t* out;              // cap bytes
  uint64_t cap;
  uint64_t* out_off;         // n_rows + 1 row byte offsets
  uint64_t* err;             // min index of an unknown id (~0 = none)
  // Special tokens (the ctx's set), sorted by id: ids the table lacks decode
  // to their bytes; with skip, special ids are dropped (decode_batch).
  const uint32_t* sp_ids;    // sp_n, ascending
  const uint32_t* sp_off;    // sp_n: byte start of each in sp_blob
  const uint32_t* sp_len;    // sp_n
  const uint8_t* sp_blob;
  uint32_t sp_n;
  int skip;
};

void launch_decode(const DecodeArgs& a, cudaStream_t s);

struct JsonArgs {
  const uint32_t* ids;
  const uint64_t* tok_off;   // n_rows + 1 (relative to tok_off[0])
  uint64_t n_rows;
  uint64_t n_ids;
  uint64_t* tok_pos;         // n_ids: text offset of each token within its block
  uint64_t* tok_sums;        // n_tok_blocks + 1
  uint64_t n_tok_blocks;
  uint64_t* row_pos;         // n_rows: frame offset of each row within its block
  uint64_t* row_sums;        // n_row_blocks + 1
  uint64_t n_row_blocks;
  uint8_t* out;
  uint64_t cap;
};

// JSON-lines text of a CSR batch; total length = tok_sums[n_tok_blocks] + row_sums[n_row_blocks].
void launch_jsonl(const JsonArgs& a, int sm_count, cudaStream_t s);

}  // namespace bbpe
