// pretok.cuh -- device GPT-2 pattern splitter (pretok.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bbpe {

// ORs the chunk starts of pattern_pretokenize("gpt2") of every row into
// chunkbits (one bit per input byte); rowbits holds the row starts
// (k_tile_first), read-only here.
// Rows of <= 4 KiB: thread per row; longer rows: warp per tile, lane per span.
void launch_pretok_gpt2(const uint8_t* d_bytes, const uint64_t* d_offsets, const uint64_t* d_tile_first,
                        uint64_t n_rows, uint64_t total, const uint32_t* d_rowbits, uint32_t* d_chunkbits,
                        uint32_t* d_long_flag /* zero on entry; k_gather resets it */, int sm_count, cudaStream_t s);

}  // namespace bbpe
