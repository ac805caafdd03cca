// kernels.cuh -- launch interface of the sm_100a BlockBPE kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bbpe_internal.h"

namespace bbpe {

constexpr int kTile = 512;          // input bytes owned by one warp-tile
constexpr int kLmax = 32;           // longest piece merged by a single lane
constexpr int kWin = kTile + kLmax + 1;  // window positions [0, kWin) after b0
constexpr int kWarpsPerCta = 8;
constexpr int kLpThreads = 512;     // CTA size of the long-piece (block engine) kernel

// Counter slots (u32).
enum { CNT_TILE_TICKET = 0, CNT_LP_COUNT = 1, CNT_LP_NEXT = 2, CNT_N = 8 };
// Error slots (u64, initialised to ~0).
enum { ERR_BAD_BYTE_POS = 0, ERR_MAXPASS_ROW = 1, ERR_CONTRACT = 2, ERR_N = 4 };

struct LongPiece {
  uint64_t start;  // absolute byte position (or token position for token input)
  uint64_t len;
  uint64_t row;
};

struct EncodeArgs {
  const uint8_t* bytes;
  const uint64_t* offsets;  // n_rows + 1, offsets[0] == 0
  uint64_t n_rows;
  uint64_t total;           // offsets[n_rows]
  uint64_t num_tiles;
  uint32_t* out_ids;
  uint64_t* out_offsets;
  // scratch
  uint64_t* tile_first;     // num_tiles + 1
  uint64_t* status;         // num_tiles look-back words
  uint32_t* counters;       // CNT_N
  uint64_t* err;            // ERR_N
  LongPiece* lp;
  uint64_t lp_cap;
  uint32_t* lpo;            // total + 1: long-piece results {count, tokens...} at start
  uint64_t* lpx;            // total: long-piece working set {token | rank << 32}
  uint64_t* lpy;            // total: double buffer
  uint64_t* trace;          // optional per-pass trace (single piece), 3 x u64 per pass
  uint64_t trace_cap;
  uint64_t* trace_count;
  int engine;               // bbpe_engine
  int tokens_input;         // 1: lpx already holds initial tokens (bbpe_block_bpe)
  int64_t max_passes;       // <= 0: none
};

struct LaunchPlan {
  int main_grid = 0;
  int prepass_grid = 0;
  int lp_grid = 0;
  int sm_count = 0;
};

LaunchPlan plan_launch(int device);
// Enqueues the full encode on `stream`; returns the number of kernels launched.
// ev (optional): 5 events recorded before the first and after each kernel.
int launch_encode(const EncodeArgs& a, const DevTable& t, const LaunchPlan& p, cudaStream_t stream,
                  cudaEvent_t* ev = nullptr);
// Long-piece kernel only (token input, used by bbpe_block_bpe).
int launch_block_bpe(const EncodeArgs& a, const DevTable& t, const LaunchPlan& p,
                     cudaStream_t stream);

}  // namespace bbpe
