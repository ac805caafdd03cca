// pretok.cuh -- device GPT-2 pattern splitter (pretok.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bbpe {

// ORs the chunk starts of pattern_pretokenize("gpt2") of every row into the
// row-start bitmap (one bit per input byte; offsets rebased, offsets[0] == 0).
void launch_pretok_gpt2(const uint8_t* d_bytes, const uint64_t* d_offsets, uint64_t n_rows, uint32_t* d_rowbits,
                        int sm_count, cudaStream_t s);

}  // namespace bbpe
