// epilogue.cuh -- device padded BatchEncoding (epilogue.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bbpe {

constexpr uint32_t kNoId = 0xFFFFFFFFu;  // no BOS / EOS

struct PadArgs {
  const uint32_t* ids;       // CSR ids
  const uint64_t* off;       // n_rows + 1 (absolute indices into ids)
  uint64_t n_rows;
  uint32_t pad, bos, eos;    // bos/eos kNoId: not added
  uint64_t max_len;
  uint32_t* out_ids;         // n_rows x max_len
  uint32_t* lengths;         // n_rows
  uint8_t* out_mask;         // n_rows x max_len
  unsigned long long* truncated;
};

void launch_row_max(const uint64_t* d_off, uint64_t n, uint32_t extra, unsigned long long* d_out, cudaStream_t s);
void launch_pad(const PadArgs& a, int sm_count, cudaStream_t s);

}  // namespace bbpe
