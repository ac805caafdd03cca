// capi.cu -- the extern "C" boundary (include/bbpe_b200.h): encode contexts,
// device scratch, host<->device staging, error mapping, multi-GPU sharding.
//
// The reference's batch path is encode_batch (proj/include/blockbpe/batch.hpp:64-126):
// validate config, fan rows out, encode each row, rethrow the first error with
// a "row r: " prefix, assemble. Here rows are packed (bytes + u64 offsets),
// encoded on the device into CSR, and errors raised on the device (invalid byte,
// pass cap) are re-materialised on the host with the reference's messages.
#include <cuda_runtime.h>
#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <cctype>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "bbpe_internal.h"
#include "decode.cuh"
#include "epilogue.cuh"
#include "kernels.cuh"
#include "specials.cuh"

namespace bbpe {
bbpe_table* table_load_files(const char* vocab, const char* merges, int format);
bbpe_table* table_create(size_t n_tokens, const uint32_t* ids, const uint64_t* tok_off,
                         const uint8_t* tok_bytes, size_t n_merges, const uint32_t* merges4);
void table_save_binary(const bbpe_table& t, const char* path);
}  // namespace bbpe

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define BBPE_TRY try {
#define BBPE_CATCH                                                      \
  }                                                                     \
  catch (const bbpe::Error& e) {                                        \
    return fail(e.code, e.what());                                      \
  }                                                                     \
  catch (const std::bad_alloc&) {                                       \
    return fail(BBPE_ERROR, "out of host memory");                      \
  }                                                                     \
  catch (const std::exception& e) {                                     \
    return fail(BBPE_ERROR, e.what());                                  \
  }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw bbpe::Error(BBPE_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  // Returns true when the buffer was (re)allocated (contents undefined).
  bool ensure(size_t bytes) {
    if (bytes <= cap && p) return false;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    want = want + want / 8;  // grow with slack so a sweep does not thrash
    ck(cudaMalloc(&p, want), "cudaMalloc (scratch)");
    cap = want;
    return true;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

bool is_pinned(const void* p) {
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeHost;
}


// Device scratch of one encode in flight (kernels.cuh EncodeArgs).
struct Scratch {
  DevBuf tile_first, status, counters, err, lpo, lpx, lpy, trace, trace_count;
  DevBuf staging, tile_count, tile_slots, tile_lrec, lrec, tile_base, long_idx, long_idx2, rowbits, mrec;
  DevBuf dkey, dres, owners, offs, chunkbits;
  uint64_t rowbits_zeroed = 0;  // words known to be zero (k_gather clears what k_tile_first set)
  uint64_t chunkbits_zeroed = 0;  // the same for the pattern splitter's chunk bits
  bool ctrl_dirty = true;       // counters/status not known to be zero (k_gather resets them)  // words known to be zero (k_pieces clears what it consumes)
  void release() {
    for (DevBuf* b : {&tile_first, &status, &counters, &err, &lpo, &lpx, &lpy, &trace, &trace_count, &staging,
                      &tile_count, &tile_slots, &tile_lrec, &lrec, &tile_base, &long_idx, &long_idx2, &rowbits, &mrec,
                      &dkey, &dres, &owners, &offs, &chunkbits})
      b->release();
    rowbits_zeroed = 0;
    chunkbits_zeroed = 0;
    ctrl_dirty = true;
  }
};

// One in-flight wave of the pipelined host encode: buffers, its own device
// scratch and compute stream (waves of different sets overlap on the device).
struct WaveSet {
  DevBuf in_bytes, in_offsets, out_ids, out_offsets, err;
  Scratch sc;
  cudaStream_t stream = nullptr;
  cudaGraphExec_t exec = nullptr;  // the wave's kernels as a CUDA graph (updated per wave)
  uint64_t* h_off = nullptr;  // pinned: the wave's CSR offsets
  uint64_t* h_rel = nullptr;  // pinned: the wave's input offsets, rebased
  uint64_t* h_err = nullptr;  // pinned: error slots
  uint64_t h_cap = 0;
  cudaEvent_t h2d_done = nullptr, comp_done = nullptr, off_done = nullptr, d2h_done = nullptr;
  uint64_t r0 = 0, r1 = 0;
  bool used = false;
  void init() {
    if (!stream) ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    if (h2d_done) return;
    for (cudaEvent_t* e : {&h2d_done, &comp_done, &off_done, &d2h_done})
      ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_err), bbpe::ERR_N * 8, 0), "cudaHostAlloc");
  }
  void reserve_host(uint64_t rows) {
    if (rows + 1 <= h_cap) return;
    if (h_off) cudaFreeHost(h_off);
    if (h_rel) cudaFreeHost(h_rel);
    h_cap = rows + 1 + (rows + 1) / 4;
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_off), h_cap * 8, 0), "cudaHostAlloc");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&h_rel), h_cap * 8, 0), "cudaHostAlloc");
  }
  void release() {
    for (DevBuf* b : {&in_bytes, &in_offsets, &out_ids, &out_offsets, &err}) b->release();
    sc.release();
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
    if (h_off) cudaFreeHost(h_off);
    if (h_rel) cudaFreeHost(h_rel);
    if (h_err) cudaFreeHost(h_err);
    for (cudaEvent_t e : {h2d_done, comp_done, off_done, d2h_done})
      if (e) cudaEventDestroy(e);
    h_off = h_rel = h_err = nullptr;
    h2d_done = comp_done = off_done = d2h_done = nullptr;
  }
};

}  // namespace

struct bbpe_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bbpe_config cfg{256, 0, BBPE_ENGINE_PIECES, 0, 1, 0, 0};
  bbpe::LaunchPlan plan;
  Scratch sc;  // device API / single-wave encodes (on `stream` or the caller's)
  DevBuf in_bytes, in_offsets, out_ids, out_offsets;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  uint64_t launches = 0;
  // Deferred device-side error check (bbpe_encode_device with sync == 0).
  bool pending = false;
  const uint64_t* pending_offsets = nullptr;
  cudaStream_t pending_stream = nullptr;
  uint64_t pending_rows = 0;
  uint64_t last_long_pieces = 0;
  // Per-kernel timing: one set of 5 events per enqueued encode.
  std::vector<std::array<cudaEvent_t, BBPE_N_KERNELS + 1>> ev_sets;
  std::vector<cudaStream_t> ev_streams;
  size_t ev_used = 0;
  double kernel_ms[BBPE_N_KERNELS] = {};
  uint64_t timed_calls = 0;
  // Pipelined host encode.
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr, off_stream = nullptr;
  static constexpr int kSets = 6;
  WaveSet sets[kSets];
  uint64_t* h_errs = nullptr;  // pinned: error slots of every wave of the last host encode
  size_t h_errs_cap = 0;
  // Device decode scratch and host-API staging.
  DevBuf dec_pos, dec_sums, dec_err, dec_ids, dec_toff, dec_out, dec_ooff, dec_rowbits;
  DevBuf pad_scalar;  // epilogue: widest row / truncated count
  DevBuf pstats;      // piece statistics (bbpe_ctx_piece_stats), PST_N u64
  bool stats_paused = false;  // the memo build's own encodes are not counted
  DevBuf run_base;
  // Special-token set (bbpe_ctx_set_specials), longest first, and the scratch
  // of bbpe_encode_batch_device.
  uint32_t sp_n = 0;
  DevBuf sp_blob, sp_off, sp_id, sp_first;
  DevBuf sp_dec;                  // decode: ids ascending | byte starts | lengths (u32 x 3 sp_dn)
  uint32_t sp_dn = 0;
  std::vector<uint32_t> sp_dec_ids;  // host copy (error-index rebasing under skip)
  DevBuf sp_cand, sp_cnt, sp_lit, sp_sums, sp_segoff, sp_segsrc, sp_ids, sp_compact, sp_segtok, sp_segtokoff;
};

namespace {

void validate_config(const bbpe_config& c) {
  // BlockConfig::validate (block_engine.hpp:26-31).
  if (c.block_size < 32 || c.block_size > 1024 || (c.block_size & (c.block_size - 1)) != 0)
    throw bbpe::usage_error("block_size must be a power of two in [32, 1024], got " +
                            std::to_string(c.block_size));
  if (c.engine != BBPE_ENGINE_PIECES && c.engine != BBPE_ENGINE_BLOCK)
    throw bbpe::usage_error("unknown engine " + std::to_string(c.engine));
  if (c.pattern != 0 && c.pattern != 1)
    throw bbpe::usage_error("unknown split pattern " + std::to_string(c.pattern) +
                            " (0 byte-level, 1 gpt2; other regexes run on the host reference only)");
  if (c.pattern && (c.engine != BBPE_ENGINE_PIECES || c.max_passes > 0))
    throw bbpe::usage_error("the gpt2 split pattern needs the pieces engine without a pass cap");
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

// Sizes scratch and fills EncodeArgs for a device-resident batch.
// Input offsets relative to `base` (pipelined waves) are rebased by
// k_tile_first into scratch; the other kernels read the rebased copy.
bbpe::EncodeArgs prepare_args(bbpe_ctx& c, Scratch& sc, const uint8_t* d_bytes, const uint64_t* d_offsets,
                              uint64_t n, uint64_t total, uint32_t* d_out, uint64_t* d_out_off,
                              cudaStream_t s, uint64_t* err = nullptr, uint64_t base = 0) {
  using namespace bbpe;
  EncodeArgs a{};
  a.bytes = d_bytes;
  a.offsets = d_offsets;
  if (base) {
    sc.offs.ensure((n + 1) * 8);
    a.offsets_raw = d_offsets;
    a.offsets_base = base;
    a.offsets = a.offsets_w = sc.offs.as<uint64_t>();
  }
  a.n_rows = n;
  a.total = total;
  a.num_tiles = (total + kTile - 1) / kTile;
  a.out_ids = d_out;
  a.out_offsets = d_out_off;
  a.num_groups = (a.num_tiles + kScanTilesPerCta - 1) / kScanTilesPerCta;
  sc.tile_first.ensure((a.num_tiles + 1) * 8);
  if (sc.status.ensure(std::max<uint64_t>(a.num_groups, 1) * 8)) sc.ctrl_dirty = true;
  sc.staging.ensure(std::max<uint64_t>(a.num_tiles, 1) * kStage * 4);
  sc.tile_count.ensure(std::max<uint64_t>(a.num_tiles, 1) * 4);
  sc.tile_slots.ensure(std::max<uint64_t>(a.num_tiles, 1) * 4);
  const uint64_t rb_words = (a.num_tiles + 1) * (kTile / 32) + kRowWords;
  sc.rowbits.ensure(rb_words * 4);
  sc.tile_lrec.ensure(std::max<uint64_t>(a.num_tiles, 1) * 8);
  sc.tile_base.ensure((a.num_tiles + 1) * 8);
  if (sc.counters.ensure(CNT_N * 4)) sc.ctrl_dirty = true;
  sc.err.ensure(ERR_N * 8);
  const bool block = c.cfg.engine == BBPE_ENGINE_BLOCK || c.cfg.max_passes > 0;
  // Long records: every row (block engine) or, worst case, one per kLmax+1
  // bytes. Merge records: at most one per 2 bytes, plus the unused tail of
  // each warp's record chunk (< 32 per refill of kMrecChunk, and the last
  // chunk of every warp).
  a.lp_cap = block ? n + 1 : total / (kLmax + 1) + 2;
  a.long_cap = a.lp_cap;
  a.mrec_cap = block ? 1 : total / 2 + total / 14 + uint64_t(std::max(c.plan.main_grid, 1)) * kWarpsPerCta * kMrecChunk;
  sc.mrec.ensure(a.mrec_cap * 16);
  a.mrec = sc.mrec.as<ulonglong2>();
  // Within-call dedupe of merge pieces (bbpe_config.no_dedup == 0): a table
  // of ~total/128 slots (the distinct merge pieces of text are far fewer;
  // a full neighbourhood just skips the dedupe for that piece).
  if (!block && !c.cfg.no_dedup && total >= kDedupMinBytes) {
    uint64_t slots = 4096;
    while (slots < total / BBPE_DEDUP_BYTES_PER_SLOT) slots <<= 1;
    sc.dkey.ensure(slots * 16);
    sc.dres.ensure(slots * 32);
    a.dkey = sc.dkey.as<ulonglong2>();
    a.dres = sc.dres.as<uint64_t>();
    a.dmask = slots - 1;
    sc.owners.ensure(a.mrec_cap * 8);
    a.owners = sc.owners.as<uint64_t>();
    ck(cudaMemsetAsync(a.dkey, 0, slots * 16, s), "memset dedupe keys");
  }
  sc.lrec.ensure(a.lp_cap * sizeof(LongRec));
  sc.long_idx.ensure(a.long_cap * 4);
  a.long_idx = sc.long_idx.as<uint32_t>();
  sc.long_idx2.ensure(a.long_cap * 4);
  a.long_idx2 = sc.long_idx2.as<uint32_t>();
  sc.lpo.ensure((total + 1) * 4);
  sc.lpx.ensure(std::max<uint64_t>(total, 1) * 8);
  sc.lpy.ensure(std::max<uint64_t>(total, 1) * 8);
  a.tile_first = sc.tile_first.as<uint64_t>();
  a.status = sc.status.as<uint64_t>();
  a.staging = sc.staging.as<uint32_t>();
  a.tile_count = sc.tile_count.as<uint32_t>();
  a.tile_slots = sc.tile_slots.as<uint32_t>();
  a.rowbits = sc.rowbits.as<uint32_t>();
  a.bytes_aligned = (reinterpret_cast<uintptr_t>(d_bytes) & 15) == 0 ? 1 : 0;
  a.tile_lrec = sc.tile_lrec.as<uint64_t>();
  a.tile_base = sc.tile_base.as<uint64_t>();
  a.lrec = sc.lrec.as<LongRec>();
  a.counters = sc.counters.as<uint32_t>();
  a.err = err ? err : sc.err.as<uint64_t>();
  a.lpo = sc.lpo.as<uint32_t>();
  a.lpx = sc.lpx.as<uint64_t>();
  a.lpy = sc.lpy.as<uint64_t>();
  a.engine = block ? BBPE_ENGINE_BLOCK : BBPE_ENGINE_PIECES;
  a.max_passes = c.cfg.max_passes;
  a.pattern = c.cfg.pattern;
  if (c.pstats.ensure(PST_N * 8)) ck(cudaMemsetAsync(c.pstats.p, 0, PST_N * 8, s), "memset pstats");
  a.pstats = c.stats_paused ? nullptr : c.pstats.as<uint64_t>();
  // Counters and look-back status are left zero by k_gather; rowbits too.
  if (sc.ctrl_dirty) {
    ck(cudaMemsetAsync(a.status, 0, sc.status.cap, s), "memset status");
    ck(cudaMemsetAsync(a.counters, 0, CNT_N * 4, s), "memset counters");
    sc.ctrl_dirty = false;
  }
  if (c.cfg.pattern && !block) {
    sc.chunkbits.ensure(rb_words * 4);
    a.chunkbits = sc.chunkbits.as<uint32_t>();
    if (sc.chunkbits_zeroed < rb_words) {
      ck(cudaMemsetAsync(a.chunkbits, 0, sc.chunkbits.cap, s), "memset chunkbits");
      sc.chunkbits_zeroed = sc.chunkbits.cap / 4;
    }
  }
  if (sc.rowbits_zeroed < rb_words) {
    ck(cudaMemsetAsync(a.rowbits, 0, sc.rowbits.cap, s), "memset rowbits");
    sc.rowbits_zeroed = sc.rowbits.cap / 4;
  }
  ck(cudaMemsetAsync(a.err, 0xFF, ERR_N * 8, s), "memset err");
  return a;
}

void ensure_plan(bbpe_ctx& c) {
  if (c.plan.sm_count == 0) c.plan = bbpe::plan_launch(c.device);
}

void ensure_memo(bbpe_ctx& c, const bbpe_table& t);

// Enqueue a device-resident encode. Handles the empty-input corner cases.
void enqueue_encode(bbpe_ctx& c, Scratch& sc, const bbpe_table& t, const uint8_t* d_bytes,
                    const uint64_t* d_offsets, uint64_t n, uint64_t total, uint32_t* d_out,
                    uint64_t* d_out_off, cudaStream_t s, bool allow_memo = true,
                    uint64_t* err = nullptr, bool timed = true, uint64_t base = 0) {
  if (total == 0) {
    ck(cudaMemsetAsync(d_out_off, 0, (n + 1) * 8, s), "memset out_offsets");
    sc.err.ensure(bbpe::ERR_N * 8);
    ck(cudaMemsetAsync(err ? err : sc.err.as<uint64_t>(), 0xFF, bbpe::ERR_N * 8, s), "memset err");
    return;
  }
  bbpe::table_on_device(t, c.device);
  ensure_plan(c);
  if (c.cfg.pattern && !t.rank_consistent)
    throw bbpe::usage_error("the gpt2 split pattern needs a rank-consistent merge table (the reference's pattern "
                            "mode runs heap_bpe, which equals the block engine only on such tables)");
  const bool memo = allow_memo && c.cfg.piece_memo && c.cfg.engine == BBPE_ENGINE_PIECES &&
                    c.cfg.max_passes <= 0;
  // The memo itself is built at API entry (maybe_build_memo), never here:
  // building encodes through the ctx's own staging buffers.
  const bbpe::DevTable dt = bbpe::table_on_device(t, c.device);
  bbpe::EncodeArgs a = prepare_args(c, sc, d_bytes, d_offsets, n, total, d_out, d_out_off, s, err, base);
  a.narrow = t.narrow ? 1 : 0;
  a.use_memo = memo && dt.memo ? 1 : 0;
  // Per-kernel timing events (BBPE_NO_KERNEL_TIMING=1 disables them, e.g.
  // for stream capture into a CUDA graph).
  static const bool no_timing = std::getenv("BBPE_NO_KERNEL_TIMING") != nullptr;
  if (no_timing || !timed) {
    c.launches += bbpe::launch_encode(a, dt, c.plan, s, nullptr);
  } else {
    if (c.ev_used == c.ev_sets.size()) {
      std::array<cudaEvent_t, BBPE_N_KERNELS + 1> set{};
      for (auto& e : set) ck(cudaEventCreate(&e), "cudaEventCreate");
      c.ev_sets.push_back(set);
      c.ev_streams.push_back(s);
    }
    c.ev_streams[c.ev_used] = s;
    c.launches += bbpe::launch_encode(a, dt, c.plan, s, c.ev_sets[c.ev_used++].data());
  }
  ck(cudaGetLastError(), "kernel launch");
}

void maybe_build_memo(bbpe_ctx& c, const bbpe_table& t) {
  if (c.cfg.piece_memo && c.cfg.engine == BBPE_ENGINE_PIECES && c.cfg.max_passes <= 0) {
    bbpe::table_on_device(t, c.device);
    ensure_plan(c);
    ensure_memo(c, t);
  }
}

uint64_t row_of(const uint64_t* host_offsets, uint64_t n, uint64_t pos) {
  // max r with offsets[r] <= pos, among r < n
  uint64_t lo = 0, hi = n ? n - 1 : 0;
  while (lo < hi) {
    uint64_t mid = (lo + hi + 1) / 2;
    if (host_offsets[mid] <= pos) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Reads the device error slots; throws the reference's exception for the
// lowest failing row (the inline encode_batch reports the first row).
void raise_device_errors(bbpe_ctx& c, const uint64_t* err, const uint64_t* host_offsets, uint64_t n,
                         uint64_t row_base, const uint8_t* host_bytes, const uint64_t* d_offsets,
                         const uint8_t* d_bytes);

void check_device_errors(bbpe_ctx& c, const uint64_t* host_offsets, uint64_t n, uint64_t row_base,
                         const uint8_t* host_bytes, const uint64_t* d_offsets,
                         const uint8_t* d_bytes) {
  uint64_t err[bbpe::ERR_N];
  ck(cudaMemcpy(err, c.sc.err.p, sizeof(err), cudaMemcpyDeviceToHost), "read error slots");
  raise_device_errors(c, err, host_offsets, n, row_base, host_bytes, d_offsets, d_bytes);
}

// Throws the reference's exception for the lowest failing row, if any.
void raise_device_errors(bbpe_ctx& c, const uint64_t* err, const uint64_t* host_offsets, uint64_t n,
                         uint64_t row_base, const uint8_t* host_bytes, const uint64_t* d_offsets,
                         const uint8_t* d_bytes) {
  const uint64_t none = ~0ull;
  if (err[bbpe::ERR_BAD_OFFSETS] != none)
    throw bbpe::usage_error("offsets must start at 0, be non-decreasing and end at total_bytes");
  if (err[bbpe::ERR_BAD_BYTE_POS] == none && err[bbpe::ERR_MAXPASS_ROW] == none) return;
  std::vector<uint64_t> tmp;
  if (!host_offsets) {
    tmp.resize(n + 1);
    ck(cudaMemcpy(tmp.data(), d_offsets, (n + 1) * 8, cudaMemcpyDeviceToHost), "read offsets");
    host_offsets = tmp.data();
  }
  uint64_t bad_row = none, mp_row = err[bbpe::ERR_MAXPASS_ROW];
  if (err[bbpe::ERR_BAD_BYTE_POS] != none) bad_row = row_of(host_offsets, n, err[bbpe::ERR_BAD_BYTE_POS]);
  if (bad_row != none && (mp_row == none || bad_row <= mp_row)) {
    uint8_t byte = 0;
    if (host_bytes)
      byte = host_bytes[err[bbpe::ERR_BAD_BYTE_POS]];
    else
      ck(cudaMemcpy(&byte, d_bytes + err[bbpe::ERR_BAD_BYTE_POS], 1, cudaMemcpyDeviceToHost), "read byte");
    throw bbpe::integrity_error("row " + std::to_string(bad_row + row_base) +
                                ": vocabulary has no single-byte token for byte value " +
                                std::to_string(byte));
  }
  // encode_batch rethrows MaxPassesError as a plain Error (batch.hpp:88-89).
  uint64_t len = host_offsets[mp_row + 1] - host_offsets[mp_row];
  throw bbpe::Error(BBPE_ERROR, "row " + std::to_string(mp_row + row_base) + ": block_bpe exceeded " +
                                    std::to_string(c.cfg.max_passes > 0 ? uint64_t(c.cfg.max_passes) : len) +
                                    " merge passes; the merge table is pathological for this input");
}

// Encodes rows [r0, r1) of a host batch as one wave. Returns tokens written.
uint64_t encode_wave(bbpe_ctx& c, const bbpe_table& t, const uint8_t* bytes,
                     const uint64_t* offsets, uint64_t r0, uint64_t r1, uint32_t* out_ids,
                     uint64_t out_pos, uint64_t out_capacity, uint64_t* out_offsets,
                     bbpe_stats* st, bool allow_memo = true) {
  const uint64_t n = r1 - r0;
  const uint64_t base = offsets[r0];
  const uint64_t total = offsets[r1] - base;
  std::vector<uint64_t> rel(n + 1);
  for (uint64_t i = 0; i <= n; ++i) rel[i] = offsets[r0 + i] - base;
  c.in_bytes.ensure(std::max<uint64_t>(total, 1) + 16);
  c.in_offsets.ensure((n + 1) * 8);
  c.out_ids.ensure(std::max<uint64_t>(total, 1) * 4);
  c.out_offsets.ensure((n + 1) * 8);
  auto t0 = std::chrono::steady_clock::now();
  if (total) ck(cudaMemcpyAsync(c.in_bytes.p, bytes + base, total, cudaMemcpyHostToDevice, c.stream), "H2D bytes");
  ck(cudaMemcpyAsync(c.in_offsets.p, rel.data(), (n + 1) * 8, cudaMemcpyHostToDevice, c.stream), "H2D offsets");
  ck(cudaStreamSynchronize(c.stream), "sync H2D");
  if (st) st->h2d_ms += ms_since(t0);
  ck(cudaEventRecord(c.ev0, c.stream), "event");
  enqueue_encode(c, c.sc, t, c.in_bytes.as<uint8_t>(), c.in_offsets.as<uint64_t>(), n, total,
                 c.out_ids.as<uint32_t>(), c.out_offsets.as<uint64_t>(), c.stream, allow_memo);
  ck(cudaEventRecord(c.ev1, c.stream), "event");
  std::vector<uint64_t> oo(n + 1);
  ck(cudaMemcpyAsync(oo.data(), c.out_offsets.p, (n + 1) * 8, cudaMemcpyDeviceToHost, c.stream), "D2H offsets");
  ck(cudaStreamSynchronize(c.stream), "encode");
  bbpe_ctx_kernel_times(&c, nullptr, nullptr, 0);
  float ms = 0;
  cudaEventElapsedTime(&ms, c.ev0, c.ev1);
  if (st) st->device_ms += ms;
  check_device_errors(c, rel.data(), n, r0, bytes + base, nullptr, nullptr);
  const uint64_t ntok = oo[n];
  if (out_pos + ntok > out_capacity)
    throw bbpe::usage_error("output capacity " + std::to_string(out_capacity) +
                            " is smaller than the " + std::to_string(out_pos + ntok) +
                            " tokens produced");
  auto t1 = std::chrono::steady_clock::now();
  if (ntok)
    ck(cudaMemcpyAsync(out_ids + out_pos, c.out_ids.p, ntok * 4, cudaMemcpyDeviceToHost, c.stream), "D2H ids");
  ck(cudaStreamSynchronize(c.stream), "D2H ids");
  if (st) st->d2h_ms += ms_since(t1);
  for (uint64_t i = 0; i <= n; ++i) out_offsets[r0 + i] = out_pos + oo[i];
  return ntok;
}

// Wave plan of a host batch: rows cut into waves whose byte sizes ramp up
// from 1 MiB (the first ids leave the device early), stay at `wave` bytes,
// and ramp down at the end (short drain). Every wave has at least one row.
std::vector<std::pair<uint64_t, uint64_t>> plan_waves(const uint64_t* offsets, uint64_t n, uint64_t wave) {
  const uint64_t total = offsets[n] - offsets[0];
  std::vector<uint64_t> front, back;
  uint64_t rem = total, f = std::min<uint64_t>(wave, 1ull << 20);
  while (rem > 0) {
    const uint64_t take = std::min(f, rem);
    front.push_back(take);
    rem -= take;
    if (f < wave && rem > 0) {
      const uint64_t b = std::min(f, rem);
      back.push_back(b);
      rem -= b;
    }
    f = std::min(wave, f * 2);
  }
  front.insert(front.end(), back.rbegin(), back.rend());
  std::vector<std::pair<uint64_t, uint64_t>> waves;
  uint64_t r0 = 0;
  size_t k = 0;
  do {
    const uint64_t target = k < front.size() ? front[k] : wave;
    ++k;
    // Rows of a wave: at least one, then as many as fit in `target` bytes
    // (binary search on the offsets: O(log n) per wave).
    uint64_t lo = r0 + 1, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) / 2;
      if (offsets[mid] - offsets[r0] <= target) lo = mid; else hi = mid - 1;
    }
    const uint64_t r1 = n == 0 ? 0 : std::min<uint64_t>(n, std::max<uint64_t>(lo, r0 + 1));
    waves.push_back({r0, r1});
    r0 = r1;
  } while (r0 < n);
  return waves;
}

// Host-buffer encode, pipelined over waves (plan_waves) with bbpe_ctx::kSets
// buffer sets, each with its own device scratch and compute stream: the H2D
// copies (one stream), the waves' kernels (overlapping across sets) and the
// D2H copies (one stream) run concurrently.
//  * Default: the host waits for each wave's row offsets (pinned staging),
//    rebases them into the caller's array and enqueues the wave's id copy
//    (copy engine) -- its size is only known once the wave is encoded.
//  * BBPE_COPY_OUT=kernel and pinned (device-mapped) outputs: everything is
//    enqueued up front and k_copy_out writes offsets and ids through the
//    mappings, carrying the running base on the copy stream (no host round
//    trip per wave; slower than the copy engines on the measured box).
uint64_t encode_host_pipelined(bbpe_ctx& c, const bbpe_table& t, const uint8_t* bytes,
                               const uint64_t* offsets, uint64_t n, uint32_t* out_ids,
                               uint64_t out_capacity, uint64_t* out_offsets, bbpe_stats* st) {
  using namespace bbpe;
  const uint64_t total_all = offsets[n] - offsets[0];
  uint64_t wave = c.cfg.wave_bytes;
  if (!wave) wave = std::max<uint64_t>(4ull << 20, std::min<uint64_t>(16ull << 20, total_all / 16 + 1));
  const std::vector<std::pair<uint64_t, uint64_t>> waves = plan_waves(offsets, n, wave);
  uint64_t max_rows = 0, max_bytes = 0;
  for (const auto& w : waves) {
    max_rows = std::max(max_rows, w.second - w.first);
    max_bytes = std::max(max_bytes, offsets[w.second] - offsets[w.first]);
  }
  // Device-mapped views of the caller's output buffers (pinned memory only).
  uint32_t* d_out_ids = nullptr;
  uint64_t* d_out_off = nullptr;
  if (is_pinned(out_offsets) && (total_all == 0 || is_pinned(out_ids))) {
    void* p = nullptr;
    if (total_all && cudaHostGetDevicePointer(&p, out_ids, 0) == cudaSuccess) d_out_ids = static_cast<uint32_t*>(p);
    if (cudaHostGetDevicePointer(&p, out_offsets, 0) == cudaSuccess) d_out_off = static_cast<uint64_t*>(p);
    cudaGetLastError();
  }
  // Device-driven copy-out is opt-in (BBPE_COPY_OUT=kernel): on B200 + PCIe
  // Gen5 the copy engines move D2H data faster than SM stores to host memory
  // and do not take SM time from the overlapping waves.
  static const bool copy_kernel = [] {
    const char* v = std::getenv("BBPE_COPY_OUT");
    return v && std::string(v) == "kernel";
  }();
  const bool async = copy_kernel && d_out_off && (total_all == 0 || d_out_ids);
  if (!c.h2d_stream) ck(cudaStreamCreateWithFlags(&c.h2d_stream, cudaStreamNonBlocking), "stream");
  if (!c.d2h_stream) ck(cudaStreamCreateWithFlags(&c.d2h_stream, cudaStreamNonBlocking), "stream");
  if (!c.off_stream) ck(cudaStreamCreateWithFlags(&c.off_stream, cudaStreamNonBlocking), "stream");
  for (WaveSet& w : c.sets) {
    w.init();
    w.in_bytes.ensure(std::max<uint64_t>(max_bytes, 1) + 16);
    w.in_offsets.ensure((max_rows + 1) * 8);
    w.out_ids.ensure(std::max<uint64_t>(max_bytes, 1) * 4);
    w.out_offsets.ensure((max_rows + 1) * 8);
    w.err.ensure(ERR_N * 8);
    w.used = false;
  }
  if (c.h_errs_cap < waves.size()) {
    if (c.h_errs) cudaFreeHost(c.h_errs);
    c.h_errs = nullptr;
    c.h_errs_cap = 0;
    ck(cudaHostAlloc(reinterpret_cast<void**>(&c.h_errs), waves.size() * ERR_N * 8, 0), "cudaHostAlloc");
    c.h_errs_cap = waves.size();
  }
  c.run_base.ensure(8);
  ck(cudaMemsetAsync(c.run_base.p, 0, 8, c.d2h_stream), "memset run_base");
  constexpr int K = bbpe_ctx::kSets;
  auto t0 = std::chrono::steady_clock::now();
  double k_before = 0;
  {
    double ms[BBPE_N_KERNELS];
    bbpe_ctx_kernel_times(&c, ms, nullptr, 0);
    for (double v : ms) k_before += v;
  }

  // Opt-in timeline (BBPE_TIMELINE=1): timing events around every copy and
  // kernel sequence, printed to stderr at the end (diagnostics only).
  static const bool tl_on = std::getenv("BBPE_TIMELINE") != nullptr;
  std::vector<std::array<cudaEvent_t, 6>> tl;
  cudaEvent_t tl0 = nullptr;
  auto tl_rec = [&](size_t k, int i, cudaStream_t s) {
    if (tl_on) ck(cudaEventRecord(tl[k][i], s), "event");
  };
  if (tl_on) {
    tl.resize(waves.size());
    for (auto& a : tl)
      for (auto& e : a) ck(cudaEventCreate(&e), "cudaEventCreate");
    ck(cudaEventCreate(&tl0), "cudaEventCreate");
    ck(cudaEventRecord(tl0, c.d2h_stream), "event");
    ck(cudaStreamWaitEvent(c.h2d_stream, tl0, 0), "wait");
  }

  static const bool use_graphs = [] {
    const char* v = std::getenv("BBPE_WAVE_GRAPHS");
    return !(v && std::string(v) == "0");
  }();
  if (use_graphs) {  // size every set's scratch for the largest wave before any capture
    table_on_device(t, c.device);
    ensure_plan(c);
    for (WaveSet& w : c.sets)
      prepare_args(c, w.sc, w.in_bytes.as<uint8_t>(), w.in_offsets.as<uint64_t>(), max_rows,
                   std::max<uint64_t>(max_bytes, 1), w.out_ids.as<uint32_t>(), w.out_offsets.as<uint64_t>(), w.stream,
                   w.err.as<uint64_t>(), 1);
  }

  auto launch = [&](size_t k) {
    WaveSet& w = c.sets[k % K];
    // Input buffers are free once the wave K back has been encoded.
    if (w.used) ck(cudaStreamWaitEvent(c.h2d_stream, w.comp_done, 0), "wait");
    tl_rec(k, 0, c.h2d_stream);
    w.r0 = waves[k].first;
    w.r1 = waves[k].second;
    const uint64_t nr = w.r1 - w.r0, base = offsets[w.r0], tot = offsets[w.r1] - base;
    if (tot)
      ck(cudaMemcpyAsync(w.in_bytes.p, bytes + base, tot, cudaMemcpyHostToDevice, c.h2d_stream), "H2D bytes");
    ck(cudaMemcpyAsync(w.in_offsets.p, offsets + w.r0, (nr + 1) * 8, cudaMemcpyHostToDevice, c.h2d_stream),
       "H2D offsets");
    ck(cudaEventRecord(w.h2d_done, c.h2d_stream), "event");
    tl_rec(k, 1, c.h2d_stream);
    // The set's compute stream: waves of different sets overlap on the device.
    ck(cudaStreamWaitEvent(w.stream, w.h2d_done, 0), "wait");
    // Output buffers are free once the wave K back has been copied out.
    if (w.used) ck(cudaStreamWaitEvent(w.stream, w.d2h_done, 0), "wait");
    w.used = true;
    tl_rec(k, 2, w.stream);
    if (use_graphs) {
      // One graph launch per wave instead of ~12 commands: under saturated
      // PCIe every command the GPU front end fetches costs tens of us. The
      // set's executable graph is updated in place (launches in flight keep
      // their parameters); scratch was sized for the largest wave up front,
      // so nothing allocates during capture.
      cudaGraph_t g = nullptr;
      ck(cudaStreamBeginCapture(w.stream, cudaStreamCaptureModeThreadLocal), "begin capture");
      try {
        enqueue_encode(c, w.sc, t, w.in_bytes.as<uint8_t>(), w.in_offsets.as<uint64_t>(), nr, tot,
                       w.out_ids.as<uint32_t>(), w.out_offsets.as<uint64_t>(), w.stream, true, w.err.as<uint64_t>(),
                       /*timed=*/false, base);
      } catch (...) {
        cudaStreamEndCapture(w.stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      ck(cudaStreamEndCapture(w.stream, &g), "end capture");
      if (w.exec) {
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(w.exec, g, &info) != cudaSuccess) {
          cudaGetLastError();
          cudaGraphExecDestroy(w.exec);
          w.exec = nullptr;
        }
      }
      if (!w.exec) ck(cudaGraphInstantiate(&w.exec, g, 0), "graph instantiate");
      cudaGraphDestroy(g);
      ck(cudaGraphLaunch(w.exec, w.stream), "graph launch");
    } else {
      enqueue_encode(c, w.sc, t, w.in_bytes.as<uint8_t>(), w.in_offsets.as<uint64_t>(), nr, tot,
                     w.out_ids.as<uint32_t>(), w.out_offsets.as<uint64_t>(), w.stream, true, w.err.as<uint64_t>(),
                     /*timed=*/false, base);
    }
    ck(cudaEventRecord(w.comp_done, w.stream), "event");
    tl_rec(k, 3, w.stream);
    if (async) {
      // Copy-out in wave order on one stream (it carries the running base).
      ck(cudaStreamWaitEvent(c.d2h_stream, w.comp_done, 0), "wait");
      tl_rec(k, 4, c.d2h_stream);
      ck(cudaMemcpyAsync(c.h_errs + k * ERR_N, w.err.p, ERR_N * 8, cudaMemcpyDeviceToHost, c.d2h_stream),
         "D2H err");
      launch_copy_out(w.out_ids.as<uint32_t>(), d_out_ids, w.out_offsets.as<uint64_t>(), d_out_off + w.r0, nr,
                      c.run_base.as<uint64_t>(), d_out_ids ? out_capacity : 0, c.plan.sm_count, c.d2h_stream);
      c.launches += 2;
      ck(cudaEventRecord(w.d2h_done, c.d2h_stream), "event");
      tl_rec(k, 5, c.d2h_stream);
    } else {
      // Wave-relative row offsets to pinned staging; the host rebases them.
      w.reserve_host(nr);
      ck(cudaStreamWaitEvent(c.off_stream, w.comp_done, 0), "wait");
      ck(cudaMemcpyAsync(w.h_off, w.out_offsets.p, (nr + 1) * 8, cudaMemcpyDeviceToHost, c.off_stream),
         "D2H offsets");
      ck(cudaMemcpyAsync(w.h_err, w.err.p, ERR_N * 8, cudaMemcpyDeviceToHost, c.off_stream), "D2H err");
      ck(cudaEventRecord(w.off_done, c.off_stream), "event");
    }
  };

  auto raise_wave_errors = [&](const uint64_t* err, size_t k) {
    if (err[ERR_BAD_OFFSETS] != ~0ull)
      throw usage_error("offsets must start at 0, be non-decreasing and end at total_bytes");
    if (err[ERR_BAD_BYTE_POS] != ~0ull || err[ERR_MAXPASS_ROW] != ~0ull) {
      const uint64_t r0 = waves[k].first, nr = waves[k].second - r0, base = offsets[r0];
      std::vector<uint64_t> rel(nr + 1);
      for (uint64_t i = 0; i <= nr; ++i) rel[i] = offsets[r0 + i] - base;
      raise_device_errors(c, err, rel.data(), nr, r0, bytes + base, nullptr, nullptr);
    }
  };

  try {
    if (async) {
      for (size_t k = 0; k < waves.size(); ++k) launch(k);
      ck(cudaStreamSynchronize(c.d2h_stream), "encode");
      for (size_t k = 0; k < waves.size(); ++k) raise_wave_errors(c.h_errs + k * ERR_N, k);
      if (out_offsets[n] > out_capacity)
        throw usage_error("output capacity " + std::to_string(out_capacity) + " is smaller than the " +
                          std::to_string(out_offsets[n]) + " tokens produced");
    } else {
      size_t launched = 0;
      uint64_t run = 0;
      while (launched < waves.size() && launched < size_t(K - 1)) launch(launched++);
      for (size_t k = 0; k < waves.size(); ++k) {
        WaveSet& w = c.sets[k % K];
        // Wave k's id copy goes out as soon as its size is known; the next
        // wave's launch and the offsets rebase happen while it runs.
        // Spin (not a blocking sync): the id copy should start the moment
        // the wave's offsets land.
        cudaError_t q;
        while ((q = cudaEventQuery(w.off_done)) == cudaErrorNotReady) {
        }
        ck(q, "encode");
        raise_wave_errors(w.h_err, k);
        const uint64_t nr = w.r1 - w.r0, ntok = w.h_off[nr];
        if (run + ntok > out_capacity)
          throw usage_error("output capacity " + std::to_string(out_capacity) + " is smaller than the " +
                            std::to_string(run + ntok) + " tokens produced");
        tl_rec(k, 4, c.d2h_stream);
        if (ntok)
          ck(cudaMemcpyAsync(out_ids + run, w.out_ids.p, ntok * 4, cudaMemcpyDeviceToHost, c.d2h_stream),
             "D2H ids");
        ck(cudaEventRecord(w.d2h_done, c.d2h_stream), "event");
        tl_rec(k, 5, c.d2h_stream);
        if (launched < waves.size()) launch(launched++);
        for (uint64_t i = 0; i <= nr; ++i) out_offsets[w.r0 + i] = run + w.h_off[i];
        run += ntok;
      }
      ck(cudaStreamSynchronize(c.d2h_stream), "D2H ids");
    }
    if (tl_on) {
      std::fprintf(stderr, "[bbpe timeline] %s: h2d_start h2d_end comp_start comp_end d2h_start d2h_end (ms)\n",
                   async ? "async" : "host-paced");
      for (size_t k = 0; k < waves.size(); ++k) {
        float v[6];
        for (int i = 0; i < 6; ++i) cudaEventElapsedTime(&v[i], tl0, tl[k][i]);
        std::fprintf(stderr, "[bbpe timeline] %zu (%llu B): %.3f %.3f %.3f %.3f %.3f %.3f\n", k,
                     (unsigned long long)(offsets[waves[k].second] - offsets[waves[k].first]), v[0], v[1], v[2],
                     v[3], v[4], v[5]);
      }
      for (auto& a : tl)
        for (auto& e : a) cudaEventDestroy(e);
      cudaEventDestroy(tl0);
    }
  } catch (...) {
    cudaStreamSynchronize(c.h2d_stream);
    for (WaveSet& w : c.sets)
      if (w.stream) cudaStreamSynchronize(w.stream);
    cudaStreamSynchronize(c.off_stream);
    cudaStreamSynchronize(c.d2h_stream);
    throw;
  }
  if (st) {
    double ms[BBPE_N_KERNELS], k_after = 0;
    bbpe_ctx_kernel_times(&c, ms, nullptr, 0);
    for (double v : ms) k_after += v;
    st->device_ms = k_after - k_before;
    st->waves = waves.size();
    st->total_ms = ms_since(t0);
  }
  return out_offsets[n];
}

// Builds the piece memo for (table, ctx device) once: every vocabulary token of
// 2..kMemoMaxLen bytes that forms a single piece (all internal bigrams are
// merge junctions) is encoded by this engine with the memo off; encodings of
// at most two tokens are stored in an open-addressing table keyed by the
// bytes. Entries depend on the table only, never on the input being encoded.
void ensure_memo_impl(bbpe_ctx& c, const bbpe_table& t);
void ensure_memo(bbpe_ctx& c, const bbpe_table& t) {
  c.stats_paused = true;
  try {
    ensure_memo_impl(c, t);
  } catch (...) {
    c.stats_paused = false;
    throw;
  }
  c.stats_paused = false;
}

void ensure_memo_impl(bbpe_ctx& c, const bbpe_table& t) {
  using namespace bbpe;
  DeviceReplica& rep = replica_of(t, c.device);
  {
    std::lock_guard<std::mutex> lock(const_cast<bbpe_table&>(t).mu);
    if (rep.memo_state != 0) return;
    rep.memo_state = 1;
  }
  std::vector<uint32_t> cand;  // token positions
  std::vector<uint8_t> blob;
  std::vector<uint64_t> offs{0};
  for (size_t i = 0; i < t.ids.size(); ++i) {
    const uint64_t b = t.tok_off[i], e = t.tok_off[i + 1];
    const uint64_t len = e - b;
    if (len < 2 || len > uint64_t(kMemoMaxLen)) continue;
    bool ok = true;
    for (uint64_t k = b; k < e && ok; ++k) ok = t.lut[t.tok_bytes[k]] != kInvalidToken;
    for (uint64_t k = b + 1; k < e && ok; ++k) {
      const uint32_t bit = (uint32_t(t.tok_bytes[k - 1]) << 8) | t.tok_bytes[k];
      ok = (t.junction[bit >> 5] >> (bit & 31)) & 1u;
    }
    if (!ok) continue;
    cand.push_back(static_cast<uint32_t>(i));
    blob.insert(blob.end(), t.tok_bytes.begin() + b, t.tok_bytes.begin() + e);
    offs.push_back(blob.size());
  }
  std::vector<MemoEntry> slots;
  uint64_t mask = 0;
  {
    std::vector<uint32_t> ids(std::max<size_t>(blob.size(), 1));
    std::vector<uint64_t> oo(cand.size() + 1, 0);
    if (!cand.empty()) {
      // The memo holds each string's own (byte-level) encoding whatever the
      // ctx's split pattern: entries are only used for pieces inside one chunk.
      const int32_t pattern = c.cfg.pattern;
      c.cfg.pattern = 0;
      try {
        encode_wave(c, t, blob.data(), offs.data(), 0, cand.size(), ids.data(), 0, ids.size(), oo.data(),
                    nullptr, /*allow_memo=*/false);
      } catch (...) {
        c.cfg.pattern = pattern;
        throw;
      }
      c.cfg.pattern = pattern;
    }
    uint64_t cap = 16;
    while (cap < (cand.size() + 256) * 8) cap <<= 1;  // load <= 1/8: a lookup resolves at its first slot
    mask = cap - 1;
    slots.assign(cap, MemoEntry{});
    for (int byte = 0; byte < 256; ++byte) {  // single bytes: their byte token
      if (t.byte_tokens[byte] == kInvalidToken) continue;
      MemoEntry m{};
      m.w[0] = uint32_t(byte);
      m.len = 1;
      m.nres = 1;
      m.res[0] = t.byte_tokens[byte];
      uint64_t b = memo_hash(m.w, m.len) & mask;
      while (slots[b].len != 0) b = (b + 1) & mask;
      slots[b] = m;
    }
    for (size_t j = 0; j < cand.size(); ++j) {
      const uint64_t nres = oo[j + 1] - oo[j];
      if (nres < 1 || nres > 2) continue;
      MemoEntry m{};
      const uint64_t len = offs[j + 1] - offs[j];
      std::memcpy(m.w, blob.data() + offs[j], len);
      m.len = static_cast<uint8_t>(len);
      m.nres = static_cast<uint8_t>(nres);
      m.res[0] = ids[oo[j]];
      m.res[1] = nres > 1 ? ids[oo[j] + 1] : 0;
      uint64_t b = memo_hash(m.w, m.len) & mask;
      while (slots[b].len != 0) b = (b + 1) & mask;
      slots[b] = m;
    }
  }
  void* dptr = nullptr;
  if (!slots.empty()) {
    ck(cudaMalloc(&dptr, slots.size() * sizeof(MemoEntry)), "cudaMalloc (memo)");
    ck(cudaMemcpy(dptr, slots.data(), slots.size() * sizeof(MemoEntry), cudaMemcpyHostToDevice),
       "memo upload");
  }
  std::lock_guard<std::mutex> lock(const_cast<bbpe_table&>(t).mu);
  rep.memo = dptr;
  rep.view.memo = static_cast<const MemoEntry*>(dptr);
  rep.view.memo_mask = mask;
  rep.memo_state = 2;
}

}  // namespace

extern "C" {

const char* bbpe_last_error(void) { return g_last_error.c_str(); }
int bbpe_abi_version(void) { return BBPE_ABI_VERSION; }

int bbpe_device_count(int* count) {
  BBPE_TRY
  ck(cudaGetDeviceCount(count), "cudaGetDeviceCount");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_table_load_files(const char* vocab_path, const char* merges_path, int format,
                          bbpe_table** out) {
  BBPE_TRY
  if (!out) throw bbpe::usage_error("out is null");
  *out = bbpe::table_load_files(vocab_path, merges_path, format);
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_table_create(size_t n_tokens, const uint32_t* ids, const uint64_t* tok_off,
                      const uint8_t* tok_bytes, size_t n_merges, const uint32_t* merges4,
                      bbpe_table** out) {
  BBPE_TRY
  if (!out) throw bbpe::usage_error("out is null");
  if ((n_tokens && (!ids || !tok_off)) || (n_merges && !merges4))
    throw bbpe::usage_error("null table arrays");
  *out = bbpe::table_create(n_tokens, ids, tok_off, tok_bytes, n_merges, merges4);
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_table_destroy(bbpe_table* t) {
  if (!t) return BBPE_OK;
  bbpe::release_replicas(*t);
  delete t;
  return BBPE_OK;
}

int bbpe_table_get_info(const bbpe_table* t, bbpe_table_info* info) {
  if (!t || !info) return fail(BBPE_USAGE, "null argument");
  info->token_count = t->ids.size();
  info->merge_count = t->m_rank.size();
  info->base_size = t->base_size;
  info->max_token_id = t->max_id;
  info->id_bits = t->id_bits;
  info->rank_bits = t->rank_bits;
  info->remapped_ids = t->remap ? 1 : 0;
  info->hash_slots = t->slots.size();
  info->junction_bigrams = t->junction_count;
  info->rank_consistent = t->rank_consistent ? 1 : 0;
  return BBPE_OK;
}

int bbpe_table_save_binary(const bbpe_table* t, const char* path) {
  BBPE_TRY
  if (!t || !path) throw bbpe::usage_error("null argument");
  bbpe::table_save_binary(*t, path);
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_table_export(const bbpe_table* t, uint32_t* ids, uint64_t* tok_off, uint8_t* tok_bytes,
                      uint64_t* n_tokens, uint64_t* n_bytes, uint32_t* merges4,
                      uint64_t* n_merges) {
  if (!t) return fail(BBPE_USAGE, "null table");
  if (n_tokens) *n_tokens = t->ids.size();
  if (n_bytes) *n_bytes = t->tok_bytes.size();
  if (n_merges) *n_merges = t->m_rank.size();
  if (ids) std::memcpy(ids, t->ids.data(), t->ids.size() * 4);
  if (tok_off) std::memcpy(tok_off, t->tok_off.data(), t->tok_off.size() * 8);
  if (tok_bytes) std::memcpy(tok_bytes, t->tok_bytes.data(), t->tok_bytes.size());
  if (merges4)
    for (size_t m = 0; m < t->m_rank.size(); ++m) {
      merges4[4 * m] = t->m_rank[m];
      merges4[4 * m + 1] = t->m_left[m];
      merges4[4 * m + 2] = t->m_right[m];
      merges4[4 * m + 3] = t->m_merged[m];
    }
  return BBPE_OK;
}

uint32_t bbpe_table_byte_token(const bbpe_table* t, uint8_t b) {
  return t ? t->byte_tokens[b] : bbpe::kInvalidToken;
}

uint32_t bbpe_table_rank_of(const bbpe_table* t, uint32_t left, uint32_t right, uint32_t* merged) {
  if (!t) return bbpe::kNoRank;
  auto it = t->pair_index.find((uint64_t(left) << 32) | right);
  if (it == t->pair_index.end()) return bbpe::kNoRank;
  if (merged) *merged = t->m_merged[it->second];
  return t->m_rank[it->second];
}

// blockbpe::decode (merge_table.hpp:565-579), table tokens only.
int bbpe_decode(const bbpe_table* t, const uint32_t* ids, size_t n, uint8_t* out, size_t cap,
                size_t* len) {
  if (!t) return fail(BBPE_USAGE, "null table");
  size_t pos = 0;
  for (size_t i = 0; i < n; ++i) {
    auto it = t->index_of.find(ids[i]);
    if (it == t->index_of.end())
      return fail(BBPE_DECODE,
                  "unknown token id " + std::to_string(ids[i]) + " at index " + std::to_string(i));
    const uint64_t b = t->tok_off[it->second], e = t->tok_off[it->second + 1];
    for (uint64_t k = b; k < e; ++k, ++pos)
      if (out && pos < cap) out[pos] = t->tok_bytes[k];
  }
  if (len) *len = pos;
  return BBPE_OK;
}

}  // extern "C"

namespace {

// Device decode table of `t` on the ctx's device (built once, like the memo).
const bbpe::DeviceReplica& decode_table(bbpe_ctx& c, const bbpe_table& t) {
  using namespace bbpe;
  table_on_device(t, c.device);
  DeviceReplica& rep = replica_of(t, c.device);
  std::lock_guard<std::mutex> lock(const_cast<bbpe_table&>(t).mu);
  if (rep.dec) return rep;
  const uint64_t dec_n = uint64_t(t.max_id) + 1;
  if (dec_n > (1ull << 26)) throw usage_error("token ids too sparse for the device decode table");
  std::vector<uint64_t> ent(dec_n, ~0ull);
  for (size_t i = 0; i < t.ids.size(); ++i)
    ent[t.ids[i]] = (t.tok_off[i] << 24) | (t.tok_off[i + 1] - t.tok_off[i]);
  const size_t nb = t.tok_bytes.size();
  void* p = nullptr;
  ck(cudaMalloc(&p, dec_n * 8 + std::max<size_t>(nb, 1)), "cudaMalloc (decode table)");
  ck(cudaMemcpy(p, ent.data(), dec_n * 8, cudaMemcpyHostToDevice), "decode table upload");
  if (nb) ck(cudaMemcpy(static_cast<char*>(p) + dec_n * 8, t.tok_bytes.data(), nb, cudaMemcpyHostToDevice),
             "decode table upload");
  rep.dec = p;
  rep.dec_n = dec_n;
  return rep;
}

// Decodes device CSR ids into device CSR bytes on c.stream (synchronous);
// raises the reference's DecodeError for the first unknown id.
uint64_t decode_on_device(bbpe_ctx& c, const bbpe_table& t, const uint32_t* d_ids, const uint64_t* d_toff,
                          uint64_t n_rows, uint64_t n_ids, uint8_t* d_out, uint64_t cap, uint64_t* d_ooff,
                          const uint64_t* h_toff, int skip = 0) {
  using namespace bbpe;
  const DeviceReplica& rep = decode_table(c, t);
  DecodeArgs a{};
  a.ids = d_ids;
  a.tok_off = d_toff;
  a.n_rows = n_rows;
  a.n_ids = n_ids;
  a.dec = static_cast<const uint64_t*>(rep.dec);
  a.dec_n = rep.dec_n;
  a.dec_bytes = static_cast<const uint8_t*>(rep.dec) + rep.dec_n * 8;
  a.n_blocks = (n_ids + kDecodeBlockTokens - 1) / kDecodeBlockTokens;
  c.dec_pos.ensure(std::max<uint64_t>(n_ids, 1) * 8);
  c.dec_sums.ensure((a.n_blocks + 1) * 8);
  c.dec_err.ensure(8);
  c.dec_rowbits.ensure(((n_ids + 31) / 32 + 1) * 4);
  a.rowstart = c.dec_rowbits.as<uint32_t>();
  a.pos = c.dec_pos.as<uint64_t>();
  a.block_sums = c.dec_sums.as<uint64_t>();
  a.err = c.dec_err.as<uint64_t>();
  a.out = d_out;
  a.cap = cap;
  a.out_off = d_ooff;
  a.sp_n = c.sp_dn;
  a.skip = skip;
  if (c.sp_dn) {
    a.sp_ids = c.sp_dec.as<uint32_t>();
    a.sp_off = a.sp_ids + c.sp_dn;
    a.sp_len = a.sp_ids + 2 * c.sp_dn;
    a.sp_blob = c.sp_blob.as<uint8_t>();
  }
  ck(cudaMemsetAsync(a.err, 0xFF, 8, c.stream), "memset");
  launch_decode(a, c.stream);
  c.launches += n_ids ? (n_rows ? 5 : 4) : 1;
  ck(cudaGetLastError(), "decode launch");
  uint64_t res[2];
  ck(cudaMemcpyAsync(&res[0], a.err, 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
  ck(cudaMemcpyAsync(&res[1], a.block_sums + a.n_blocks, 8, cudaMemcpyDeviceToHost, c.stream), "D2H");
  ck(cudaStreamSynchronize(c.stream), "decode");
  if (res[0] != ~0ull) {
    std::vector<uint64_t> tmp;
    if (!h_toff) {
      tmp.resize(n_rows + 1);
      ck(cudaMemcpy(tmp.data(), d_toff, (n_rows + 1) * 8, cudaMemcpyDeviceToHost), "D2H");
      h_toff = tmp.data();
    }
    const uint64_t base = h_toff[0], i = res[0];
    uint64_t lo = 0, hi = n_rows ? n_rows - 1 : 0;  // max r with h_toff[r] - base <= i
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) / 2;
      if (h_toff[mid] - base <= i) lo = mid; else hi = mid - 1;
    }
    uint32_t id = 0;
    ck(cudaMemcpy(&id, d_ids + i, 4, cudaMemcpyDeviceToHost), "D2H");
    uint64_t at = i - (h_toff[lo] - base);  // index within the row (after skipped specials)
    if (skip && c.sp_dn && at) {
      std::vector<uint32_t> head(at);
      ck(cudaMemcpy(head.data(), d_ids + (h_toff[lo] - base), at * 4, cudaMemcpyDeviceToHost), "D2H");
      for (uint32_t v : head)
        if (std::binary_search(c.sp_dec_ids.begin(), c.sp_dec_ids.end(), v)) --at;
    }
    throw Error(BBPE_DECODE, "row " + std::to_string(lo) + ": unknown token id " + std::to_string(id) +
                                 " at index " + std::to_string(at));
  }
  return res[1];
}

}  // namespace

extern "C" {

int bbpe_decode_device(bbpe_ctx* c, const bbpe_table* t, const uint32_t* d_ids, const uint64_t* d_tok_offsets,
                       size_t n_rows, uint64_t n_ids, uint8_t* d_out_bytes, uint64_t cap,
                       uint64_t* d_out_byte_offsets, uint64_t* total) {
  return bbpe_decode_device_ex(c, t, d_ids, d_tok_offsets, n_rows, n_ids, 0, d_out_bytes, cap, d_out_byte_offsets,
                               total);
}

int bbpe_decode_device_ex(bbpe_ctx* c, const bbpe_table* t, const uint32_t* d_ids, const uint64_t* d_tok_offsets,
                          size_t n_rows, uint64_t n_ids, int skip_specials, uint8_t* d_out_bytes, uint64_t cap,
                          uint64_t* d_out_byte_offsets, uint64_t* total) {
  BBPE_TRY
  if (!c || !t || !d_tok_offsets || !d_out_byte_offsets) throw bbpe::usage_error("null argument");
  if (n_ids && (!d_ids || (cap && !d_out_bytes))) throw bbpe::usage_error("null buffer");
  DeviceGuard g(c->device);
  const uint64_t tot = decode_on_device(*c, *t, d_ids, d_tok_offsets, n_rows, n_ids, d_out_bytes, cap,
                                        d_out_byte_offsets, nullptr, skip_specials);
  if (total) *total = tot;
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_decode_batch(bbpe_ctx* c, const bbpe_table* t, const uint32_t* ids, const uint64_t* tok_offsets,
                      size_t n_rows, uint8_t* out_bytes, uint64_t cap, uint64_t* out_byte_offsets,
                      uint64_t* total) {
  return bbpe_decode_batch_ex(c, t, ids, tok_offsets, n_rows, 0, out_bytes, cap, out_byte_offsets, total);
}

int bbpe_decode_batch_ex(bbpe_ctx* c, const bbpe_table* t, const uint32_t* ids, const uint64_t* tok_offsets,
                         size_t n_rows, int skip_specials, uint8_t* out_bytes, uint64_t cap,
                         uint64_t* out_byte_offsets, uint64_t* total) {
  BBPE_TRY
  if (!c || !t || !tok_offsets || !out_byte_offsets) throw bbpe::usage_error("null argument");
  const uint64_t base = tok_offsets[0], n_ids = tok_offsets[n_rows] - base;
  if (tok_offsets[n_rows] < base) throw bbpe::usage_error("offsets must be non-decreasing");
  if (n_ids && !ids) throw bbpe::usage_error("null buffer");
  for (size_t r = 0; r < n_rows; ++r)
    if (tok_offsets[r + 1] < tok_offsets[r]) throw bbpe::usage_error("offsets must be non-decreasing");
  DeviceGuard g(c->device);
  c->dec_ids.ensure(std::max<uint64_t>(n_ids, 1) * 4);
  c->dec_toff.ensure((n_rows + 1) * 8);
  c->dec_ooff.ensure((n_rows + 1) * 8);
  if (n_ids)
    ck(cudaMemcpyAsync(c->dec_ids.p, ids + base, n_ids * 4, cudaMemcpyHostToDevice, c->stream), "H2D ids");
  ck(cudaMemcpyAsync(c->dec_toff.p, tok_offsets, (n_rows + 1) * 8, cudaMemcpyHostToDevice, c->stream),
     "H2D offsets");
  // Output bytes: the exact size after a first pass would cost a round trip;
  // size the device buffer by the caller's capacity instead.
  c->dec_out.ensure(std::max<uint64_t>(cap, 1));
  const uint64_t tot = decode_on_device(*c, *t, c->dec_ids.as<uint32_t>(), c->dec_toff.as<uint64_t>(), n_rows,
                                        n_ids, c->dec_out.as<uint8_t>(), cap, c->dec_ooff.as<uint64_t>(),
                                        tok_offsets, skip_specials);
  const uint64_t ncopy = std::min(tot, cap);
  if (ncopy) ck(cudaMemcpyAsync(out_bytes, c->dec_out.p, ncopy, cudaMemcpyDeviceToHost, c->stream), "D2H bytes");
  ck(cudaMemcpyAsync(out_byte_offsets, c->dec_ooff.p, (n_rows + 1) * 8, cudaMemcpyDeviceToHost, c->stream),
     "D2H offsets");
  ck(cudaStreamSynchronize(c->stream), "decode");
  if (total) *total = tot;
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_jsonl_device(bbpe_ctx* c, const uint32_t* d_ids, const uint64_t* d_tok_offsets, size_t n_rows,
                      uint64_t n_ids, uint8_t* d_out, uint64_t cap, uint64_t* total) {
  BBPE_TRY
  if (!c || !d_tok_offsets || !total) throw bbpe::usage_error("null argument");
  if ((n_ids && !d_ids) || (cap && !d_out)) throw bbpe::usage_error("null buffer");
  DeviceGuard g(c->device);
  ensure_plan(*c);
  bbpe::JsonArgs a{};
  a.ids = d_ids;
  a.tok_off = d_tok_offsets;
  a.n_rows = n_rows;
  a.n_ids = n_ids;
  a.n_tok_blocks = (n_ids + 255) / 256;
  a.n_row_blocks = (n_rows + 255) / 256;
  c->dec_pos.ensure(std::max<uint64_t>(n_ids, 1) * 8);
  c->dec_sums.ensure((a.n_tok_blocks + 1) * 8);
  c->dec_toff.ensure(std::max<uint64_t>(n_rows, 1) * 8);
  c->dec_ooff.ensure((a.n_row_blocks + 1) * 8);
  a.tok_pos = c->dec_pos.as<uint64_t>();
  a.tok_sums = c->dec_sums.as<uint64_t>();
  a.row_pos = c->dec_toff.as<uint64_t>();
  a.row_sums = c->dec_ooff.as<uint64_t>();
  a.out = d_out;
  a.cap = cap;
  bbpe::launch_jsonl(a, c->plan.sm_count, c->stream);
  c->launches += n_rows ? 4 : 0;
  ck(cudaGetLastError(), "jsonl launch");
  uint64_t t[2];
  ck(cudaMemcpyAsync(&t[0], a.tok_sums + a.n_tok_blocks, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaMemcpyAsync(&t[1], a.row_sums + a.n_row_blocks, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "jsonl");
  *total = t[0] + t[1];
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_batch_widest_device(bbpe_ctx* c, const uint64_t* d_tok_offsets, size_t n_rows, int add_bos,
                             int add_eos, uint64_t* widest) {
  BBPE_TRY
  if (!c || !d_tok_offsets || !widest) throw bbpe::usage_error("null argument");
  DeviceGuard g(c->device);
  c->pad_scalar.ensure(8);
  bbpe::launch_row_max(d_tok_offsets, n_rows, uint32_t((add_bos ? 1 : 0) + (add_eos ? 1 : 0)),
                       c->pad_scalar.as<unsigned long long>(), c->stream);
  c->launches += n_rows ? 1 : 0;
  ck(cudaMemcpyAsync(widest, c->pad_scalar.p, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "widest");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_pad_device(bbpe_ctx* c, const uint32_t* d_ids, const uint64_t* d_tok_offsets, size_t n_rows,
                    uint32_t pad_id, uint32_t bos_id, uint32_t eos_id, uint64_t max_len, uint32_t* d_out_ids,
                    uint32_t* d_lengths, uint8_t* d_mask, uint64_t* truncated_rows) {
  BBPE_TRY
  if (!c || !d_tok_offsets) throw bbpe::usage_error("null argument");
  if (n_rows && (!d_lengths || (max_len && (!d_out_ids || !d_mask)))) throw bbpe::usage_error("null buffer");
  DeviceGuard g(c->device);
  ensure_plan(*c);
  c->pad_scalar.ensure(8);
  bbpe::PadArgs a{};
  a.ids = d_ids;
  a.off = d_tok_offsets;
  a.n_rows = n_rows;
  a.pad = pad_id;
  a.bos = bos_id;
  a.eos = eos_id;
  a.max_len = max_len;
  a.out_ids = d_out_ids;
  a.lengths = d_lengths;
  a.out_mask = d_mask;
  a.truncated = c->pad_scalar.as<unsigned long long>();
  bbpe::launch_pad(a, c->plan.sm_count, c->stream);
  c->launches += n_rows ? (max_len ? 2 : 1) : 0;
  uint64_t tr = 0;
  ck(cudaMemcpyAsync(&tr, c->pad_scalar.p, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "pad");
  if (truncated_rows) *truncated_rows = tr;
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_pretokenize_device(bbpe_ctx* c, const uint8_t* d_bytes, const uint64_t* d_offsets, size_t n,
                            uint64_t total_bytes, uint32_t* d_chunk_bits) {
  BBPE_TRY
  if (!c || !d_offsets || (total_bytes && (!d_bytes || !d_chunk_bits))) throw bbpe::usage_error("null argument");
  DeviceGuard g(c->device);
  ensure_plan(*c);
  if (!total_bytes) return BBPE_OK;
  const int saved = c->cfg.pattern;
  c->cfg.pattern = 1;
  bbpe::EncodeArgs a;
  try {
    a = prepare_args(*c, c->sc, d_bytes, d_offsets, n, total_bytes, nullptr, nullptr, c->stream);
  } catch (...) {
    c->cfg.pattern = saved;
    throw;
  }
  c->cfg.pattern = saved;
  c->launches += bbpe::launch_pretok_only(a, c->plan, d_chunk_bits, c->stream);
  // k_gather did not run: the row / chunk bitmaps and counters are not zero.
  c->sc.rowbits_zeroed = 0;
  c->sc.chunkbits_zeroed = 0;
  c->sc.ctrl_dirty = true;
  ck(cudaStreamSynchronize(c->stream), "pretokenize");
  uint64_t err[bbpe::ERR_N];
  ck(cudaMemcpy(err, a.err, sizeof(err), cudaMemcpyDeviceToHost), "read error slots");
  if (err[bbpe::ERR_BAD_OFFSETS] != ~0ull)
    throw bbpe::usage_error("offsets must start at 0, be non-decreasing and end at total_bytes");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_ctx_set_specials(bbpe_ctx* c, size_t n, const uint8_t* blob, const uint64_t* offsets,
                          const uint32_t* ids) {
  BBPE_TRY
  if (!c) throw bbpe::usage_error("null ctx");
  if (n && (!blob || !offsets || !ids)) throw bbpe::usage_error("null argument");
  // SpecialTokenSet::add (merge_table.hpp:311-319): non-empty, unique, kept
  // longest first (a new entry goes after every entry at least as long).
  struct Ent {
    std::string b;
    uint32_t id;
  };
  std::vector<Ent> es;
  for (size_t i = 0; i < n; ++i) {
    if (offsets[i + 1] < offsets[i]) throw bbpe::usage_error("special offsets must be non-decreasing");
    std::string b(reinterpret_cast<const char*>(blob + offsets[i]), offsets[i + 1] - offsets[i]);
    if (b.empty()) throw bbpe::usage_error("special token byte string may not be empty");
    for (const Ent& e : es)
      if (e.b == b) throw bbpe::usage_error("duplicate special token \"" + b + "\"");
    auto it = es.begin();
    while (it != es.end() && it->b.size() >= b.size()) ++it;
    es.insert(it, Ent{std::move(b), ids[i]});
  }
  std::vector<uint8_t> hb;
  std::vector<uint32_t> ho{0}, hi, hf(8, 0);
  for (const Ent& e : es) {
    hb.insert(hb.end(), e.b.begin(), e.b.end());
    if (hb.size() > 0xFFFFFFFFull) throw bbpe::usage_error("special tokens too long");
    ho.push_back(uint32_t(hb.size()));
    hi.push_back(e.id);
    const uint8_t f = uint8_t(e.b[0]);
    hf[f >> 5] |= 1u << (f & 31);
  }
  DeviceGuard g(c->device);
  c->sp_n = 0;
  c->sp_dn = 0;
  c->sp_dec_ids.clear();
  if (es.empty()) return BBPE_OK;
  c->sp_blob.ensure(hb.size());
  c->sp_off.ensure(ho.size() * 4);
  c->sp_id.ensure(hi.size() * 4);
  c->sp_first.ensure(32);
  ck(cudaMemcpy(c->sp_blob.p, hb.data(), hb.size(), cudaMemcpyHostToDevice), "specials upload");
  ck(cudaMemcpy(c->sp_off.p, ho.data(), ho.size() * 4, cudaMemcpyHostToDevice), "specials upload");
  ck(cudaMemcpy(c->sp_id.p, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice), "specials upload");
  ck(cudaMemcpy(c->sp_first.p, hf.data(), 32, cudaMemcpyHostToDevice), "specials upload");
  // Decode view by id; for an id held by several strings the one latest in
  // the longest-first order wins (SpecialTokenSet::rebuild_index, merge_table.hpp:357-360).
  std::vector<std::pair<uint32_t, size_t>> by_id;
  for (size_t k = 0; k < es.size(); ++k) by_id.push_back({es[k].id, k});
  std::stable_sort(by_id.begin(), by_id.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
  std::vector<uint32_t> d_id, d_off, d_len;
  for (size_t k = 0; k < by_id.size(); ++k) {
    if (k + 1 < by_id.size() && by_id[k + 1].first == by_id[k].first) continue;  // keep the last
    d_id.push_back(by_id[k].first);
    d_off.push_back(ho[by_id[k].second]);
    d_len.push_back(ho[by_id[k].second + 1] - ho[by_id[k].second]);
  }
  std::vector<uint32_t> packed(d_id);
  packed.insert(packed.end(), d_off.begin(), d_off.end());
  packed.insert(packed.end(), d_len.begin(), d_len.end());
  c->sp_dec.ensure(packed.size() * 4);
  ck(cudaMemcpy(c->sp_dec.p, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice), "specials upload");
  c->sp_dn = uint32_t(d_id.size());
  c->sp_dec_ids = d_id;
  c->sp_n = uint32_t(es.size());
  return BBPE_OK;
  BBPE_CATCH
}

namespace {

constexpr uint64_t kDeviceChunk = 2ull << 30;  // larger device batches run in chunks
double encode_device_chunked(bbpe_ctx& c, const bbpe_table& t, const uint8_t* d_bytes, const uint64_t* d_offsets,
                             uint64_t n, uint64_t total, uint32_t* d_out_ids, uint64_t* d_out_offsets,
                             cudaStream_t s);

// Synchronous device encode with the reference's errors; chunked above kDeviceChunk.
void encode_device_sync(bbpe_ctx& c, const bbpe_table& t, const uint8_t* d_bytes, const uint64_t* d_offsets,
                        uint64_t n, uint64_t total, uint32_t* d_out, uint64_t* d_out_off, cudaStream_t s) {
  if (total > kDeviceChunk) {
    encode_device_chunked(c, t, d_bytes, d_offsets, n, total, d_out, d_out_off, s);
    return;
  }
  enqueue_encode(c, c.sc, t, d_bytes, d_offsets, n, total, d_out, d_out_off, s);
  ck(cudaStreamSynchronize(s), "encode");
  check_device_errors(c, nullptr, n, 0, nullptr, d_offsets, d_bytes);
}

// bbpe_encode_batch_device's body; returns the id total.
uint64_t encode_batch_on_device(bbpe_ctx* c, const bbpe_table* t, const uint8_t* d_bytes,
                                const uint64_t* d_offsets, size_t n, uint64_t total_bytes, uint32_t bos_id,
                                uint32_t eos_id, uint32_t* d_out_ids, uint64_t out_capacity,
                                uint64_t* d_out_offsets) {
  validate_config(c->cfg);
  DeviceGuard g(c->device);
  ensure_plan(*c);
  maybe_build_memo(*c, *t);
  cudaStream_t s = c->stream;
  const uint32_t none = 0xFFFFFFFFu;
  const int add_bos = bos_id != none, add_eos = eos_id != none;
  const int sm = c->plan.sm_count;
  auto read_u64 = [&](const void* p) {
    uint64_t v = 0;
    ck(cudaMemcpyAsync(&v, p, 8, cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "specials");
    return v;
  };
  // (1) split at special tokens: per-row match counts and literal bytes, scanned.
  c->sp_cnt.ensure((n + 1) * 8);
  c->sp_sums.ensure(bbpe::scan_sums_len(n) * 8);
  uint64_t* match_base = c->sp_cnt.as<uint64_t>();
  uint64_t M = 0;
  bbpe::SpecArgs sp{c->sp_blob.as<uint8_t>(), c->sp_off.as<uint32_t>(), c->sp_id.as<uint32_t>(),
                    c->sp_first.as<uint32_t>(), c->sp_n};
  if (c->sp_n && total_bytes) {
    c->sp_cand.ensure((total_bytes + 31) / 32 * 4);
    c->sp_lit.ensure((n + 1) * 8);
    bbpe::launch_sp_candidates(d_bytes, total_bytes, sp, c->sp_cand.as<uint32_t>(), sm, s);
    bbpe::launch_sp_rows(d_bytes, d_offsets, n, sp, c->sp_cand.as<uint32_t>(), match_base,
                         c->sp_lit.as<uint64_t>(), s);
    bbpe::launch_scan_u64(match_base, n, c->sp_sums.as<uint64_t>(), s);
    c->launches += 2 + (n ? 3 : 0);
    M = read_u64(match_base + n);
  } else {
    ck(cudaMemsetAsync(match_base, 0, (n + 1) * 8, s), "memset");
  }
  if (M == 0 && !add_bos && !add_eos && out_capacity >= total_bytes) {  // plain CSR encode
    encode_device_sync(*c, *t, d_bytes, d_offsets, n, total_bytes, d_out_ids, d_out_offsets, s);
    return read_u64(d_out_offsets + n);
  }
  // (2) segments. When every byte value has a token (and no pass cap is set),
  // special bytes can be encoded harmlessly: the segments tile the input in place (literal,
  // special, ..., literal; the specials' tokens are dropped by the stitch).
  // Otherwise the literal bytes are compacted (r + match_base[r] + j).
  // (A pass cap could fail on a special's bytes, which the reference never encodes.)
  const bool inplace = c->cfg.max_passes <= 0 &&
                       std::none_of(t->lut.begin(), t->lut.end(), [](uint32_t v) { return v == bbpe::kInvalidToken; });
  const int stride = inplace ? 2 : 1;
  const uint8_t* seg_bytes = d_bytes;
  const uint64_t* seg_offsets = d_offsets;
  uint64_t n_seg = n, seg_total = total_bytes;
  if (M) {
    n_seg = n + stride * M;
    c->sp_segoff.ensure((n_seg + 1) * 8);
    c->sp_ids.ensure(M * 4);
    if (inplace) {
      bbpe::launch_sp_emit(d_bytes, d_offsets, n, sp, c->sp_cand.as<uint32_t>(), match_base, nullptr,
                           c->sp_segoff.as<uint64_t>(), nullptr, c->sp_ids.as<uint32_t>(), 1, s);
      c->launches += 1;
    } else {
      bbpe::launch_scan_u64(c->sp_lit.as<uint64_t>(), n, c->sp_sums.as<uint64_t>(), s);
      seg_total = read_u64(c->sp_lit.as<uint64_t>() + n);
      c->sp_segsrc.ensure(n_seg * 8);
      c->sp_compact.ensure(seg_total + 16);
      bbpe::launch_sp_emit(d_bytes, d_offsets, n, sp, c->sp_cand.as<uint32_t>(), match_base,
                           c->sp_lit.as<uint64_t>(), c->sp_segoff.as<uint64_t>(), c->sp_segsrc.as<uint64_t>(),
                           c->sp_ids.as<uint32_t>(), 0, s);
      bbpe::launch_sp_copy(d_bytes, n_seg, c->sp_segoff.as<uint64_t>(), c->sp_segsrc.as<uint64_t>(),
                           c->sp_compact.as<uint8_t>(), sm, s);
      c->launches += 5;
      seg_bytes = c->sp_compact.as<uint8_t>();
    }
    seg_offsets = c->sp_segoff.as<uint64_t>();
  }
  // (3) encode the literal segments as rows.
  c->sp_segtok.ensure(std::max<uint64_t>(seg_total, 1) * 4);
  c->sp_segtokoff.ensure((n_seg + 1) * 8);
  try {
    encode_device_sync(*c, *t, seg_bytes, seg_offsets, n_seg, seg_total, c->sp_segtok.as<uint32_t>(),
                       c->sp_segtokoff.as<uint64_t>(), s);
  } catch (const bbpe::Error& e) {
    // "row <segment>: ..." -> the input row holding that segment.
    const std::string m = e.what();
    if (!M || m.compare(0, 4, "row ") != 0) throw;
    const size_t colon = m.find(':');
    const uint64_t seg = std::stoull(m.substr(4, colon - 4));
    std::vector<uint64_t> mb(n + 1);
    ck(cudaMemcpy(mb.data(), match_base, (n + 1) * 8, cudaMemcpyDeviceToHost), "D2H");
    uint64_t lo = 0, hi = n - 1;  // max r with r + stride * mb[r] <= seg
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) / 2;
      if (mid + stride * mb[mid] <= seg) lo = mid; else hi = mid - 1;
    }
    throw bbpe::Error(e.code, "row " + std::to_string(lo) + m.substr(colon));
  }
  // (4) stitch: BOS, segment tokens, special ids, EOS.
  bbpe::launch_sp_lengths(n, match_base, c->sp_segtokoff.as<uint64_t>(), add_bos, add_eos, M ? stride : 1,
                          d_out_offsets, s);
  bbpe::launch_scan_u64(d_out_offsets, n, c->sp_sums.as<uint64_t>(), s);
  const uint64_t out_total = read_u64(d_out_offsets + n);
  if (out_total > out_capacity)
    throw bbpe::usage_error("output capacity " + std::to_string(out_capacity) + " < " +
                            std::to_string(out_total) + " ids");
  if (out_total && !d_out_ids) throw bbpe::usage_error("null output ids");
  bbpe::launch_sp_stitch(n, match_base, c->sp_segtokoff.as<uint64_t>(), c->sp_segtok.as<uint32_t>(),
                         c->sp_ids.as<uint32_t>(), d_out_offsets, bos_id, eos_id, M ? stride : 1, d_out_ids, sm, s);
  c->launches += n ? 5 : 1;
  ck(cudaStreamSynchronize(s), "stitch");
  return out_total;
}

}  // namespace

int bbpe_encode_batch_device(bbpe_ctx* c, const bbpe_table* t, const uint8_t* d_bytes,
                             const uint64_t* d_offsets, size_t n, uint64_t total_bytes, uint32_t bos_id,
                             uint32_t eos_id, uint32_t* d_out_ids, uint64_t out_capacity, uint64_t* d_out_offsets,
                             uint64_t* n_out_ids) {
  BBPE_TRY
  if (!c || !t || !d_offsets || !d_out_offsets) throw bbpe::usage_error("null argument");
  if (total_bytes && !d_bytes) throw bbpe::usage_error("null bytes");
  const uint64_t k = encode_batch_on_device(c, t, d_bytes, d_offsets, n, total_bytes, bos_id, eos_id, d_out_ids,
                                            out_capacity, d_out_offsets);
  if (n_out_ids) *n_out_ids = k;
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_encode_batch(bbpe_ctx* c, const bbpe_table* t, const uint8_t* bytes, const uint64_t* offsets, size_t n,
                      uint32_t bos_id, uint32_t eos_id, uint32_t* out_ids, uint64_t out_capacity,
                      uint64_t* out_offsets, uint64_t* n_out_ids) {
  BBPE_TRY
  if (!c || !t || !offsets || !out_offsets) throw bbpe::usage_error("null argument");
  const uint64_t base = offsets[0], total = offsets[n] - base;
  if (total && !bytes) throw bbpe::usage_error("null bytes");
  for (size_t i = 0; i < n; ++i)
    if (offsets[i + 1] < offsets[i]) throw bbpe::usage_error("offsets must be non-decreasing");
  DeviceGuard g(c->device);
  validate_config(c->cfg);
  ensure_plan(*c);
  maybe_build_memo(*c, *t);  // first: the memo build encodes through in_bytes / out_ids
  std::vector<uint64_t> rel(n + 1);
  for (size_t i = 0; i <= n; ++i) rel[i] = offsets[i] - base;
  const uint64_t cap = total + 2 * uint64_t(n) + 1;  // literal tokens + specials <= bytes, plus BOS/EOS
  c->in_bytes.ensure(std::max<uint64_t>(total, 1) + 16);
  c->in_offsets.ensure((n + 1) * 8);
  c->out_ids.ensure(cap * 4);
  c->out_offsets.ensure((n + 1) * 8);
  if (total)
    ck(cudaMemcpyAsync(c->in_bytes.p, bytes + base, total, cudaMemcpyHostToDevice, c->stream), "H2D bytes");
  ck(cudaMemcpyAsync(c->in_offsets.p, rel.data(), (n + 1) * 8, cudaMemcpyHostToDevice, c->stream), "H2D offsets");
  const uint64_t k = encode_batch_on_device(c, t, c->in_bytes.as<uint8_t>(), c->in_offsets.as<uint64_t>(), n, total,
                                            bos_id, eos_id, c->out_ids.as<uint32_t>(), cap,
                                            c->out_offsets.as<uint64_t>());
  if (k > out_capacity)
    throw bbpe::usage_error("output capacity " + std::to_string(out_capacity) + " < " + std::to_string(k) +
                            " ids");
  if (k && !out_ids) throw bbpe::usage_error("null output ids");
  if (k) ck(cudaMemcpyAsync(out_ids, c->out_ids.p, k * 4, cudaMemcpyDeviceToHost, c->stream), "D2H ids");
  ck(cudaMemcpyAsync(out_offsets, c->out_offsets.p, (n + 1) * 8, cudaMemcpyDeviceToHost, c->stream), "D2H offsets");
  ck(cudaStreamSynchronize(c->stream), "D2H");
  if (n_out_ids) *n_out_ids = k;
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_ctx_create(int device, const bbpe_config* cfg, bbpe_ctx** out) {
  BBPE_TRY
  if (!out) throw bbpe::usage_error("out is null");
  auto c = std::make_unique<bbpe_ctx>();
  c->device = device;
  if (cfg) {
    validate_config(*cfg);
    c->cfg = *cfg;
  }
  DeviceGuard g(device);
  ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaEventCreate(&c->ev0), "cudaEventCreate");
  ck(cudaEventCreate(&c->ev1), "cudaEventCreate");
  *out = c.release();
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_ctx_destroy(bbpe_ctx* c) {
  if (!c) return BBPE_OK;
  {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    c->sc.release();
    for (DevBuf* b : {&c->in_bytes, &c->in_offsets, &c->out_ids, &c->out_offsets, &c->dec_pos, &c->dec_rowbits, &c->dec_sums,
                      &c->dec_err, &c->dec_ids, &c->dec_toff, &c->dec_out, &c->dec_ooff, &c->pad_scalar, &c->pstats,
                      &c->sp_blob, &c->sp_off, &c->sp_id, &c->sp_first, &c->sp_dec, &c->sp_cand, &c->sp_cnt, &c->sp_lit,
                      &c->sp_sums, &c->sp_segoff, &c->sp_segsrc, &c->sp_ids, &c->sp_compact, &c->sp_segtok,
                      &c->sp_segtokoff})
      b->release();
    cudaEventDestroy(c->ev0);
    cudaEventDestroy(c->ev1);
    for (auto& set : c->ev_sets)
      for (auto e : set) cudaEventDestroy(e);
    for (WaveSet& w : c->sets) w.release();
    if (c->h_errs) cudaFreeHost(c->h_errs);
    c->run_base.release();
    if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
    if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
    if (c->off_stream) cudaStreamDestroy(c->off_stream);
    cudaStreamDestroy(c->stream);
    cudaSetDevice(prev);
  }
  delete c;
  return BBPE_OK;
}

int bbpe_ctx_set_config(bbpe_ctx* c, const bbpe_config* cfg) {
  BBPE_TRY
  if (!c || !cfg) throw bbpe::usage_error("null argument");
  validate_config(*cfg);
  if (cfg->max_passes < 0) throw bbpe::usage_error("max_passes must be >= 1");
  c->cfg = *cfg;
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_ctx_prepare(bbpe_ctx* c, const bbpe_table* t) {
  BBPE_TRY
  if (!c || !t) throw bbpe::usage_error("null argument");
  DeviceGuard g(c->device);
  bbpe::table_on_device(*t, c->device);
  ensure_plan(*c);
  maybe_build_memo(*c, *t);
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_host_alloc(size_t bytes, void** out) {
  BBPE_TRY
  ck(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable), "cudaHostAlloc");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_host_free(void* p) {
  BBPE_TRY
  if (p) ck(cudaFreeHost(p), "cudaFreeHost");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_encode(bbpe_ctx* c, const bbpe_table* t, const uint8_t* bytes, const uint64_t* offsets,
                size_t n, uint32_t* out_ids, uint64_t out_capacity, uint64_t* out_offsets,
                bbpe_stats* st) {
  BBPE_TRY
  auto t0 = std::chrono::steady_clock::now();
  if (!c || !t || !offsets || !out_offsets) throw bbpe::usage_error("null argument");
  validate_config(c->cfg);
  // Row offsets are checked on the device (k_tile_first, ERR_BAD_OFFSETS);
  // the wave plan only needs the batch to be non-empty-or-ordered overall.
  if (offsets[n] < offsets[0]) throw bbpe::usage_error("offsets must be non-decreasing");
  if (offsets[n] > offsets[0] && (!bytes || !out_ids)) throw bbpe::usage_error("null buffer");
  DeviceGuard g(c->device);
  maybe_build_memo(*c, *t);
  if (st) *st = bbpe_stats{};
  const uint64_t pos =
      encode_host_pipelined(*c, *t, bytes, offsets, n, out_ids, out_capacity, out_offsets, st);
  if (st) {
    st->n_rows = n;
    st->input_bytes = offsets[n] - offsets[0];
    st->tokens = pos;
    st->total_ms = ms_since(t0);
  }
  return BBPE_OK;
  BBPE_CATCH
}

namespace {

// Device batches above kDeviceChunk input bytes run as row-range chunks (the
// scratch of one launch is sized for adversarial input, ~38 B per input
// byte): chunk ids land at d_out_ids + the running token base, the chunk's
// offsets are moved onto it by k_add_u64; one sync per chunk. Chunk starts
// prefer 16-byte aligned rows (k_pieces' asynchronous window loads).
double encode_device_chunked(bbpe_ctx& c, const bbpe_table& t, const uint8_t* d_bytes, const uint64_t* d_offsets,
                             uint64_t n, uint64_t total, uint32_t* d_out_ids, uint64_t* d_out_offsets,
                             cudaStream_t s) {
  std::vector<uint64_t> off(n + 1);
  ck(cudaMemcpyAsync(off.data(), d_offsets, (n + 1) * 8, cudaMemcpyDeviceToHost, s), "D2H offsets");
  ck(cudaStreamSynchronize(s), "D2H offsets");
  if (off[0] != 0 || off[n] != total) throw bbpe::usage_error("offsets must start at 0 and end at total_bytes");
  for (uint64_t i = 0; i < n; ++i)
    if (off[i + 1] < off[i]) throw bbpe::usage_error("offsets must be non-decreasing");
  ensure_plan(c);
  float ms_total = 0;
  uint64_t r0 = 0, tok = 0;
  while (r0 < n) {
    uint64_t r1 = uint64_t(std::upper_bound(off.begin() + r0 + 1, off.end(), off[r0] + kDeviceChunk) - off.begin()) - 1;
    if (r1 <= r0) r1 = r0 + 1;  // one row above the chunk size: alone
    if (r1 < n) {
      for (uint64_t k = r1, lim = r1 > r0 + 4096 ? r1 - 4096 : r0 + 1; k >= lim && k > r0; --k)
        if (((reinterpret_cast<uintptr_t>(d_bytes) + off[k]) & 15) == 0) {
          r1 = k;
          break;
        }
    }
    const uint64_t nr = r1 - r0, base = off[r0], tot = off[r1] - base;
    ck(cudaEventRecord(c.ev0, s), "event");
    enqueue_encode(c, c.sc, t, d_bytes + base, d_offsets + r0, nr, tot, d_out_ids + tok, d_out_offsets + r0, s,
                   true, nullptr, true, base);
    uint64_t ntok = 0;
    ck(cudaMemcpyAsync(&ntok, d_out_offsets + r1, 8, cudaMemcpyDeviceToHost, s), "D2H count");
    ck(cudaEventRecord(c.ev1, s), "event");
    ck(cudaStreamSynchronize(s), "encode");
    float ms = 0;
    cudaEventElapsedTime(&ms, c.ev0, c.ev1);
    ms_total += ms;
    std::vector<uint64_t> rel(nr + 1);
    for (uint64_t i = 0; i <= nr; ++i) rel[i] = off[r0 + i] - base;
    uint64_t err[bbpe::ERR_N];
    ck(cudaMemcpy(err, c.sc.err.p, sizeof(err), cudaMemcpyDeviceToHost), "read error slots");
    raise_device_errors(c, err, rel.data(), nr, r0, nullptr, nullptr, d_bytes + base);
    bbpe::launch_add_u64(d_out_offsets + r0, nr + 1, tok, c.plan.sm_count, s);
    ++c.launches;
    tok += ntok;
    r0 = r1;
  }
  ck(cudaStreamSynchronize(s), "encode");
  return ms_total;
}

}  // namespace

int bbpe_encode_device(bbpe_ctx* c, const bbpe_table* t, const uint8_t* d_bytes,
                       const uint64_t* d_offsets, size_t n, uint64_t total_bytes,
                       uint32_t* d_out_ids, uint64_t* d_out_offsets, void* stream, int sync,
                       bbpe_stats* st) {
  BBPE_TRY
  if (!c || !t || !d_offsets || !d_out_offsets) throw bbpe::usage_error("null argument");
  validate_config(c->cfg);
  DeviceGuard g(c->device);
  maybe_build_memo(*c, *t);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->stream;
  if (total_bytes > kDeviceChunk) {  // scratch for one launch is ~38 B per input byte
    const double ms = encode_device_chunked(*c, *t, d_bytes, d_offsets, n, total_bytes, d_out_ids, d_out_offsets, s);
    if (st) {
      *st = bbpe_stats{};
      st->n_rows = n;
      st->input_bytes = total_bytes;
      st->device_ms = ms;
    }
    return BBPE_OK;
  }
  if (sync) ck(cudaEventRecord(c->ev0, s), "event");
  enqueue_encode(*c, c->sc, *t, d_bytes, d_offsets, n, total_bytes, d_out_ids, d_out_offsets, s);
  c->pending = true;
  c->pending_offsets = d_offsets;
  c->pending_stream = s;
  c->pending_rows = n;
  if (sync) {
    ck(cudaEventRecord(c->ev1, s), "event");
    ck(cudaStreamSynchronize(s), "encode");
    c->pending = false;
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    if (st) {
      *st = bbpe_stats{};
      st->n_rows = n;
      st->input_bytes = total_bytes;
      st->device_ms = ms;
      st->waves = 1;
    }
    check_device_errors(*c, nullptr, n, 0, nullptr, d_offsets, d_bytes);
  }
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_ctx_sync(bbpe_ctx* c) {
  BBPE_TRY
  if (!c) throw bbpe::usage_error("null ctx");
  DeviceGuard g(c->device);
  ck(cudaStreamSynchronize(c->stream), "sync");
  if (c->pending_stream) ck(cudaStreamSynchronize(c->pending_stream), "sync");
  if (c->pending) {
    c->pending = false;
    check_device_errors(*c, nullptr, c->pending_rows, 0, nullptr, c->pending_offsets, nullptr);
  }
  return BBPE_OK;
  BBPE_CATCH
}

uint64_t bbpe_ctx_kernel_launches(const bbpe_ctx* c) { return c ? c->launches : 0; }

int bbpe_ctx_kernel_times(bbpe_ctx* c, double* ms, uint64_t* calls, int reset) {
  BBPE_TRY
  if (!c) throw bbpe::usage_error("null ctx");
  DeviceGuard g(c->device);
  for (size_t i = 0; i < c->ev_used; ++i) {
    ck(cudaEventSynchronize(c->ev_sets[i][BBPE_N_KERNELS]), "event sync");
    for (int k = 0; k < BBPE_N_KERNELS; ++k) {
      float e = 0;
      ck(cudaEventElapsedTime(&e, c->ev_sets[i][k], c->ev_sets[i][k + 1]), "event time");
      c->kernel_ms[k] += e;
    }
  }
  c->timed_calls += c->ev_used;
  c->ev_used = 0;
  if (ms)
    for (int k = 0; k < BBPE_N_KERNELS; ++k) ms[k] = c->kernel_ms[k];
  if (calls) *calls = c->timed_calls;
  if (reset) {
    for (double& v : c->kernel_ms) v = 0;
    c->timed_calls = 0;
  }
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_ctx_piece_stats(bbpe_ctx* c, uint64_t* out, int reset) {
  BBPE_TRY
  if (!c || !out) throw bbpe::usage_error("null argument");
  DeviceGuard g(c->device);
  for (int i = 0; i < BBPE_N_PIECE_STATS; ++i) out[i] = 0;
  if (!c->pstats.p) return BBPE_OK;
  ck(cudaDeviceSynchronize(), "piece stats sync");
  uint64_t v[bbpe::PST_N];
  ck(cudaMemcpy(v, c->pstats.p, sizeof(v), cudaMemcpyDeviceToHost), "D2H piece stats");
  for (int i = 0; i < BBPE_N_PIECE_STATS; ++i) out[i] = v[i];
  if (reset) ck(cudaMemset(c->pstats.p, 0, sizeof(v)), "memset piece stats");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_block_bpe(bbpe_ctx* c, const bbpe_table* t, const uint32_t* tokens, size_t n,
                   uint32_t* out, size_t* out_n, uint64_t* trace, size_t trace_cap,
                   size_t* n_passes) {
  BBPE_TRY
  using namespace bbpe;
  if (!c || !t || !out_n || (n && (!tokens || !out))) throw usage_error("null argument");
  validate_config(c->cfg);
  if (n_passes) *n_passes = 0;
  if (n < 2) {
    if (n) std::memcpy(out, tokens, n * 4);
    *out_n = n;
    return BBPE_OK;
  }
  if (n >= (1ull << 31)) throw usage_error("sequence too long");
  DeviceGuard g(c->device);
  const DevTable& dt = table_on_device(*t, c->device);
  ensure_plan(*c);
  // Dense ids for the device. Ids the table never mentions never pair
  // (find_pair misses, merge_table.hpp:237), but a raw id past the device key
  // width would alias a real pair (l << id_bits | r). All of them become one
  // placeholder id P that no merge mentions; P is never produced by a merge
  // either, so the output's placeholders are the input's outside ids in
  // their input order (mapped back below).
  std::vector<uint64_t> x(n);
  std::vector<uint32_t> outside;  // outside ids, in input order
  const uint32_t n_dense = t->remap ? static_cast<uint32_t>(t->dense_to_id.size()) : 0;
  const uint32_t P = t->remap ? n_dense : t->max_dev_id + 1;
  for (size_t i = 0; i < n; ++i) {
    uint32_t d = t->dense(tokens[i]);
    if ((t->remap && d == kInvalidToken) || (!t->remap && tokens[i] > t->max_dev_id)) {
      outside.push_back(tokens[i]);
      d = P;
    }
    x[i] = uint64_t(d) | (uint64_t(0xFFFFFFFEu) << 32);
  }
  EncodeArgs a{};
  a.n_rows = 1;
  a.total = n;
  c->sc.counters.ensure(CNT_N * 4);
  c->sc.err.ensure(ERR_N * 8);
  c->sc.lrec.ensure(sizeof(LongRec));
  c->sc.long_idx.ensure(4);
  c->sc.long_idx2.ensure(4);
  c->sc.lpo.ensure((n + 1) * 4);
  c->sc.lpx.ensure(n * 8);
  c->sc.lpy.ensure(n * 8);
  size_t tcap = trace ? trace_cap : 0;
  c->sc.trace.ensure(std::max<size_t>(tcap, 1) * 24);
  c->sc.trace_count.ensure(8);
  a.counters = c->sc.counters.as<uint32_t>();
  a.err = c->sc.err.as<uint64_t>();
  a.lrec = c->sc.lrec.as<LongRec>();
  a.lp_cap = 1;
  a.long_idx = c->sc.long_idx.as<uint32_t>();
  a.long_idx2 = c->sc.long_idx2.as<uint32_t>();
  a.long_cap = 1;
  a.lpo = c->sc.lpo.as<uint32_t>();
  a.lpx = c->sc.lpx.as<uint64_t>();
  a.lpy = c->sc.lpy.as<uint64_t>();
  a.trace = c->sc.trace.as<uint64_t>();
  a.trace_cap = tcap;
  a.trace_count = c->sc.trace_count.as<uint64_t>();
  a.tokens_input = 1;
  a.engine = BBPE_ENGINE_BLOCK;
  a.max_passes = c->cfg.max_passes;
  LongRec lp{0, n, 0, 0u, 0u};
  uint32_t counters[CNT_N] = {0};
  counters[CNT_LREC] = 1;
  counters[CNT_LONG] = 1;
  const uint32_t zero = 0;
  ck(cudaMemcpyAsync(a.lrec, &lp, sizeof(lp), cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(cudaMemcpyAsync(a.long_idx, &zero, 4, cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(cudaMemcpyAsync(a.counters, counters, sizeof(counters), cudaMemcpyHostToDevice, c->stream), "H2D");
  c->sc.ctrl_dirty = true;  // k_gather does not run here to leave the counters zero
  ck(cudaMemsetAsync(a.err, 0xFF, ERR_N * 8, c->stream), "memset");
  ck(cudaMemcpyAsync(a.lpx, x.data(), n * 8, cudaMemcpyHostToDevice, c->stream), "H2D");
  c->launches += launch_block_bpe(a, dt, c->plan, c->stream);
  ck(cudaGetLastError(), "launch");
  uint32_t cnt = 0;
  uint64_t err[ERR_N], passes = 0;
  ck(cudaMemcpyAsync(&cnt, a.lpo, 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaMemcpyAsync(err, a.err, sizeof(err), cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaMemcpyAsync(&passes, a.trace_count, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "block_bpe");
  std::vector<uint32_t> res(cnt);
  if (cnt) ck(cudaMemcpy(res.data(), a.lpo + 1, cnt * 4ull, cudaMemcpyDeviceToHost), "D2H");
  {
    size_t k = 0;
    for (auto& v : res) {
      if (v == P) {
        if (k >= outside.size()) return fail(BBPE_CONTRACT, "block_bpe: placeholder count changed");
        v = outside[k++];
      } else if (t->remap) {
        v = t->dense_to_id[v];
      }
    }
  }
  std::memcpy(out, res.data(), cnt * 4ull);
  *out_n = cnt;
  if (n_passes) *n_passes = passes;
  if (tcap) ck(cudaMemcpy(trace, a.trace, std::min<uint64_t>(passes, tcap) * 24, cudaMemcpyDeviceToHost), "D2H");
  if (err[ERR_MAXPASS_ROW] != ~0ull)
    return fail(BBPE_MAX_PASSES, "block_bpe exceeded " + std::to_string(c->cfg.max_passes) +
                                     " merge passes; the merge table is pathological for this input");
  return BBPE_OK;
  BBPE_CATCH
}

// ---- spec-level operations (block_engine.hpp:189-256) on the device ----
}  // extern "C"

namespace {
// Pins the calling thread to the CPUs local to `device` (sysfs local_cpulist
// of its PCI function), so pinned staging it allocates and the copies it
// drives stay on the GPU's NUMA node. Best effort: silently does nothing when
// the topology is unavailable.
void bind_thread_near_device(int device) {
  char bus[32] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) return;
  std::string id(bus);
  for (auto& ch : id) ch = char(std::tolower(static_cast<unsigned char>(ch)));
  FILE* f = std::fopen(("/sys/bus/pci/devices/" + id + "/local_cpulist").c_str(), "r");
  if (!f) return;
  char buf[4096] = {0};
  const size_t k = std::fread(buf, 1, sizeof(buf) - 1, f);
  std::fclose(f);
  buf[k] = 0;
  cpu_set_t set;
  CPU_ZERO(&set);
  int count = 0;
  for (char* p = buf; *p && *p != '\n';) {
    char* e = nullptr;
    long a = std::strtol(p, &e, 10), b = a;
    if (e == p) break;
    if (*e == '-') b = std::strtol(e + 1, &e, 10);
    for (long c = a; c <= b && c < CPU_SETSIZE; ++c, ++count) CPU_SET(int(c), &set);
    p = (*e == ',') ? e + 1 : e;
  }
  if (count) pthread_setaffinity_np(pthread_self(), sizeof(set), &set);
}

// dst[0, n) = src[0, n) by `threads` threads (the ranges must not overlap).
void parallel_copy(uint32_t* dst, const uint32_t* src, uint64_t n, int threads) {
  const uint64_t per = (n + threads - 1) / threads;
  if (threads <= 1 || n < (1u << 18)) {
    std::memcpy(dst, src, n * 4);
    return;
  }
  std::vector<std::thread> th;
  for (int k = 0; k < threads; ++k) {
    const uint64_t a = k * per, b = std::min<uint64_t>(n, a + per);
    if (a >= b) break;
    th.emplace_back([=] { std::memcpy(dst + a, src + a, (b - a) * 4); });
  }
  for (auto& x : th) x.join();
}

// Caller ids -> dense device ids; ids the table never mentions become one
// placeholder that no merge mentions (as in bbpe_block_bpe).
std::vector<uint32_t> spec_dense(const bbpe_table* t, const uint32_t* tokens, size_t n) {
  std::vector<uint32_t> d(n);
  const uint32_t P = t->remap ? static_cast<uint32_t>(t->dense_to_id.size()) : t->max_dev_id + 1;
  for (size_t i = 0; i < n; ++i) {
    uint32_t x = t->dense(tokens[i]);
    if ((t->remap && x == bbpe::kInvalidToken) || (!t->remap && tokens[i] > t->max_dev_id)) x = P;
    d[i] = x;
  }
  return d;
}

// Scoped device allocation for the spec ops (test/debug surface).
struct SpecBuf {
  void* p = nullptr;
  explicit SpecBuf(size_t bytes) { ck(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc (spec op)"); }
  ~SpecBuf() { cudaFree(p); }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

void spec_ranks_device(bbpe_ctx* c, const bbpe_table* t, const uint32_t* tokens, size_t n, const SpecBuf& dtok,
                       const SpecBuf& ranks) {
  const bbpe::DevTable& dt = bbpe::table_on_device(*t, c->device);
  const std::vector<uint32_t> d = spec_dense(t, tokens, n);
  ck(cudaMemcpyAsync(dtok.p, d.data(), n * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
  bbpe::launch_spec_ranks(dtok.as<uint32_t>(), n, dt, ranks.as<uint32_t>(), c->stream);
  c->launches += 1;
  ck(cudaGetLastError(), "launch");
}
}  // namespace

extern "C" {

int bbpe_pair_ranks(bbpe_ctx* c, const bbpe_table* t, const uint32_t* tokens, size_t n, uint32_t* ranks) {
  BBPE_TRY
  if (!c || !t || (n && !tokens) || (n > 1 && !ranks)) throw bbpe::usage_error("null argument");
  if (n < 2) return BBPE_OK;
  DeviceGuard g(c->device);
  SpecBuf dtok(n * 4), dr(n * 4);
  spec_ranks_device(c, t, tokens, n, dtok, dr);
  ck(cudaMemcpyAsync(ranks, dr.p, (n - 1) * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "pair_ranks");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_min_rank_reduce(bbpe_ctx* c, const uint32_t* ranks, size_t n, uint32_t* out) {
  BBPE_TRY
  if (!c || !out || (n && !ranks)) throw bbpe::usage_error("null argument");
  *out = bbpe::kNoRank;
  if (!n) return BBPE_OK;
  DeviceGuard g(c->device);
  SpecBuf dr(n * 4), dm(4);
  ck(cudaMemcpyAsync(dr.p, ranks, n * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(cudaMemsetAsync(dm.p, 0xFF, 4, c->stream), "memset");
  bbpe::launch_spec_min(dr.as<uint32_t>(), n, dm.as<uint32_t>(), c->stream);
  c->launches += 1;
  ck(cudaGetLastError(), "launch");
  ck(cudaMemcpyAsync(out, dm.p, 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "min_rank_reduce");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_mark_merges(bbpe_ctx* c, const bbpe_table* t, const uint32_t* tokens, size_t n, uint32_t min_rank,
                     uint8_t* flags) {
  BBPE_TRY
  if (!c || !t || (n && (!tokens || !flags))) throw bbpe::usage_error("null argument");
  if (!n) return BBPE_OK;
  DeviceGuard g(c->device);
  SpecBuf dtok(n * 4), dr(n * 4), df(n);
  ck(cudaMemsetAsync(df.p, 0, n, c->stream), "memset");
  if (n >= 2) {
    spec_ranks_device(c, t, tokens, n, dtok, dr);
    bbpe::launch_spec_runs(dr.as<uint32_t>(), n, min_rank, df.as<uint8_t>(), c->stream);
    c->launches += 1;
    ck(cudaGetLastError(), "launch");
  }
  ck(cudaMemcpyAsync(flags, df.p, n, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "mark_merges");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_exclusive_scan(bbpe_ctx* c, const uint8_t* flags, size_t n, uint32_t* offsets) {
  BBPE_TRY
  if (!c || (n && (!flags || !offsets))) throw bbpe::usage_error("null argument");
  if (!n) return BBPE_OK;
  DeviceGuard g(c->device);
  SpecBuf df(n), doff(n * 4), derr(8), dtot(4);
  ck(cudaMemcpyAsync(df.p, flags, n, cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(cudaMemsetAsync(derr.p, 0xFF, 8, c->stream), "memset");
  bbpe::launch_spec_check(df.as<uint8_t>(), n, derr.as<unsigned long long>(), c->stream);
  bbpe::launch_spec_scan(df.as<uint8_t>(), n, doff.as<uint32_t>(), dtot.as<uint32_t>(), c->stream);
  c->launches += 2;
  ck(cudaGetLastError(), "launch");
  uint64_t err = 0;
  ck(cudaMemcpyAsync(&err, derr.p, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "exclusive_scan");
  if (err != ~0ull) {  // block_engine.hpp:225-231, lowest failing index first
    const uint64_t i = err >> 1;
    if ((err & 1) == 0)
      return fail(BBPE_CONTRACT, "merge flags must be 0/1, got " + std::to_string(int(flags[i])) + " at index " +
                                     std::to_string(i));
    return fail(BBPE_CONTRACT, "adjacent merge flags at indices " + std::to_string(i - 1) + " and " +
                                   std::to_string(i) + " are both set; left-greedy marking forbids this");
  }
  ck(cudaMemcpy(offsets, doff.p, n * 4, cudaMemcpyDeviceToHost), "D2H");
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_compact(bbpe_ctx* c, const bbpe_table* t, const uint32_t* tokens, size_t n, const uint8_t* flags,
                 size_t n_flags, const uint32_t* offsets, size_t n_offsets, uint32_t* out, size_t* out_n) {
  BBPE_TRY
  if (!c || !t || !out_n || (n && !tokens) || (n_flags && !flags) || (n_offsets && !offsets) || (n && !out))
    throw bbpe::usage_error("null argument");
  *out_n = 0;
  if (n_flags != n || n_offsets != n)  // block_engine.hpp:242-243
    return fail(BBPE_CONTRACT, "flags/offsets length does not match token count");
  if (!n) return BBPE_OK;
  DeviceGuard g(c->device);
  const bbpe::DevTable& dt = bbpe::table_on_device(*t, c->device);
  const std::vector<uint32_t> d = spec_dense(t, tokens, n);
  SpecBuf dtok(n * 4), dorig(n * 4), df(n), doff(n * 4), dscan(n * 4), dtot(4), derr(16), dout(n * 4);
  ck(cudaMemcpyAsync(dtok.p, d.data(), n * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(cudaMemcpyAsync(dorig.p, tokens, n * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(cudaMemcpyAsync(df.p, flags, n, cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(cudaMemcpyAsync(doff.p, offsets, n * 4, cudaMemcpyHostToDevice, c->stream), "H2D");
  ck(cudaMemsetAsync(derr.p, 0xFF, 16, c->stream), "memset");
  unsigned long long* e = derr.as<unsigned long long>();
  // offsets must be the exclusive scan of flags (244-249)
  bbpe::launch_spec_scan(df.as<uint8_t>(), n, dscan.as<uint32_t>(), dtot.as<uint32_t>(), c->stream);
  bbpe::launch_spec_check_offsets(doff.as<uint32_t>(), dscan.as<uint32_t>(), n, e, c->stream);
  ck(cudaGetLastError(), "launch");
  uint64_t err[2];
  uint32_t total = 0;
  ck(cudaMemcpyAsync(err, e, 16, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaMemcpyAsync(&total, dtot.p, 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "compact");
  c->launches += 2;
  if (err[0] != ~0ull)
    return fail(BBPE_CONTRACT, "offsets are not the exclusive scan of flags at index " + std::to_string(err[0]));
  // compact_into (166-182): a flagged pair that is not a merge is a ContractViolation
  bbpe::launch_spec_compact(dtok.as<uint32_t>(), dorig.as<uint32_t>(), df.as<uint8_t>(), doff.as<uint32_t>(), n, dt,
                            dout.as<uint32_t>(), e + 1, c->stream);
  c->launches += 1;
  ck(cudaGetLastError(), "launch");
  ck(cudaMemcpyAsync(err + 1, e + 1, 8, cudaMemcpyDeviceToHost, c->stream), "D2H");
  ck(cudaStreamSynchronize(c->stream), "compact");
  if (err[1] != ~0ull)
    return fail(BBPE_CONTRACT, "flags mark a pair that is not in the merge table at index " + std::to_string(err[1]));
  if (total > n) return fail(BBPE_CONTRACT, "merge flags exceed the token count");
  const size_t m = n - total;
  ck(cudaMemcpy(out, dout.p, m * 4, cudaMemcpyDeviceToHost), "D2H");
  *out_n = m;
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_partition(const uint64_t* offsets, size_t n, int parts, uint64_t* bounds) {
  BBPE_TRY
  if (!offsets || !bounds || parts < 1) throw bbpe::usage_error("bad partition arguments");
  // cost(row) = len + 64: prefix cost is offsets[r] - offsets[0] + 64 r.
  auto cost = [&](uint64_t r) { return (offsets[r] - offsets[0]) + 64 * r; };
  const uint64_t total = cost(n);
  bounds[0] = 0;
  uint64_t r = 0;
  for (int p = 1; p < parts; ++p) {
    const uint64_t target = total * p / parts;
    while (r < n && cost(r) < target) ++r;
    bounds[p] = r;
  }
  bounds[parts] = n;
  return BBPE_OK;
  BBPE_CATCH
}

int bbpe_encode_sharded(bbpe_ctx* const* ctxs, int n_devices, const bbpe_table* t,
                        const uint8_t* bytes, const uint64_t* offsets, size_t n, uint32_t* out_ids,
                        uint64_t out_capacity, uint64_t* out_offsets, bbpe_stats* st) {
  BBPE_TRY
  if (!ctxs || n_devices < 1 || !t || !offsets || !out_offsets) throw bbpe::usage_error("null argument");
  for (int d = 0; d < n_devices; ++d)
    if (!ctxs[d]) throw bbpe::usage_error("null ctx");
  auto t0 = std::chrono::steady_clock::now();
  std::vector<uint64_t> bounds(n_devices + 1);
  bbpe_partition(offsets, n, n_devices, bounds.data());
  const uint64_t base = offsets[0], total_bytes = offsets[n] - base;
  // Output regions: shard d writes its ids at at[d], a share of the caller's
  // capacity proportional to its bytes (tokens <= bytes, so with capacity >=
  // total bytes no region can overflow; with less, a shard that overflows its
  // region is re-encoded into a host vector and copied in the stitch).
  std::vector<uint64_t> at(n_devices + 1);
  for (int d = 0; d <= n_devices; ++d) {
    const uint64_t b = offsets[bounds[d]] - base;
    at[d] = out_capacity >= total_bytes
                ? b
                : uint64_t((unsigned __int128)out_capacity * b / std::max<uint64_t>(total_bytes, 1));
  }
  std::vector<uint64_t> ntok(n_devices, 0);
  std::vector<std::vector<uint64_t>> offs(n_devices);
  std::vector<std::vector<uint32_t>> spill(n_devices);  // shards that overflowed their region
  std::vector<int> codes(n_devices, BBPE_OK);
  std::vector<std::string> msgs(n_devices);
  std::vector<bbpe_stats> stats(n_devices);
  std::vector<std::thread> th;
  for (int d = 0; d < n_devices; ++d) {
    th.emplace_back([&, d] {
      bind_thread_near_device(ctxs[d]->device);  // host staging and copies on the GPU's NUMA node
      const uint64_t r0 = bounds[d], r1 = bounds[d + 1];
      offs[d].resize(r1 - r0 + 1);
      const uint64_t cap = at[d + 1] - at[d];
      int rc = bbpe_encode(ctxs[d], t, bytes, offsets + r0, r1 - r0, out_ids ? out_ids + at[d] : nullptr, cap,
                           offs[d].data(), &stats[d]);
      if (rc == BBPE_USAGE && cap < offsets[r1] - offsets[r0]) {  // region too small: host vector
        spill[d].resize(std::max<uint64_t>(offsets[r1] - offsets[r0], 1));
        rc = bbpe_encode(ctxs[d], t, bytes, offsets + r0, r1 - r0, spill[d].data(), spill[d].size(),
                         offs[d].data(), &stats[d]);
      }
      codes[d] = rc;
      if (rc != BBPE_OK) msgs[d] = bbpe_last_error();
      ntok[d] = offs[d].back();
    });
  }
  for (auto& x : th) x.join();
  for (int d = 0; d < n_devices; ++d)
    if (codes[d] != BBPE_OK) {
      // Row indices in shard messages are shard-relative; rebase "row r: ".
      std::string m = msgs[d];
      if (m.rfind("row ", 0) == 0) {
        size_t colon = m.find(':');
        uint64_t r = std::stoull(m.substr(4, colon - 4)) + bounds[d];
        m = "row " + std::to_string(r) + m.substr(colon);
      }
      return fail(codes[d], m);
    }
  std::vector<uint64_t> pos(n_devices + 1, 0);
  for (int d = 0; d < n_devices; ++d) pos[d + 1] = pos[d] + ntok[d];
  if (pos[n_devices] > out_capacity)
    throw bbpe::usage_error("output capacity " + std::to_string(out_capacity) + " is smaller than the " +
                            std::to_string(pos[n_devices]) + " tokens of the batch");
  // Stitch. Shards move left in shard order (shard d's destination can only
  // overlap sources of shards < d, already moved); each move is copied by
  // several threads in waves no longer than its shift, so no wave writes a
  // source another thread of the wave still reads.
  // With a spilled shard, later regions may start before their destination:
  // every shard then goes through a host vector.
  const int hw = std::max(1, std::min<int>(16, int(std::thread::hardware_concurrency())));
  bool any_spill = false;
  for (int d = 0; d < n_devices; ++d) any_spill |= !spill[d].empty();
  if (any_spill) {
    for (int d = 0; d < n_devices; ++d)
      if (spill[d].empty() && ntok[d]) spill[d].assign(out_ids + at[d], out_ids + at[d] + ntok[d]);
    for (int d = 0; d < n_devices; ++d)
      if (ntok[d]) parallel_copy(out_ids + pos[d], spill[d].data(), ntok[d], hw);
  }
  for (int d = 0; d < n_devices && !any_spill; ++d) {
    if (!ntok[d]) continue;
    uint32_t* dst = out_ids + pos[d];
    const uint32_t* src = out_ids + at[d];
    if (src == dst) continue;
    const uint64_t shift = uint64_t(src - dst);  // pos <= at: every shard before d fits its region
    const uint64_t wave = std::min<uint64_t>(shift, ntok[d]);
    if (wave < (1u << 20)) {
      std::memmove(dst, src, ntok[d] * 4);
      continue;
    }
    for (uint64_t w = 0; w < ntok[d]; w += wave)
      parallel_copy(dst + w, src + w, std::min<uint64_t>(wave, ntok[d] - w), hw);
  }
  for (int d = 0; d < n_devices; ++d) {
    const uint64_t r0 = bounds[d], r1 = bounds[d + 1];
    for (uint64_t i = 0; i <= r1 - r0; ++i) out_offsets[r0 + i] = pos[d] + offs[d][i];
  }
  if (st) {
    *st = bbpe_stats{};
    st->n_rows = n;
    st->input_bytes = total_bytes;
    st->tokens = pos[n_devices];
    for (auto& s : stats) {
      st->device_ms = std::max(st->device_ms, s.device_ms);
      st->waves += s.waves;
    }
    st->total_ms = ms_since(t0);
  }
  return BBPE_OK;
  BBPE_CATCH
}

}  // extern "C"
