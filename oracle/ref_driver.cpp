// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" shim over the UNMODIFIED reference library headers
// (/root/reference/proj/include/blockbpe/*.hpp), compiled by oracle/Makefile
// into oracle/_ref/libbbpe_ref.so. Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline / --impl reference) may load it.
//
// Entry points mirror the reference's own calls:
//   ref_table_load_files  -> blockbpe::load_merge_table_files  (merge_table.hpp:513-522)
//   ref_table_build       -> MergeTable::add_token/add_merge/finalize (merge_table.hpp:257-297)
//   ref_encode_batch      -> blockbpe::encode_batch (block engine)  (batch.hpp:64-126)
//   ref_encode_heap       -> heap_bpe per row fanned over PhasePool::run_items
//                            (ref_engines.hpp:46-103, thread_pool.hpp:95-101)
//   ref_block_bpe_trace   -> blockbpe::block_bpe with a PassTrace (block_engine.hpp:268-310)
//   ref_naive_bpe         -> blockbpe::naive_bpe (ref_engines.hpp:22-40)
//   ref_encode_pattern    -> encode_reference, pattern mode (ref_engines.hpp:119-146)
//   ref_pretokenize       -> pattern_pretokenize (pretokenize.hpp:252-258)
// The batch outputs are returned as CSR (ids + u64 offsets), the layout the
// B200 path produces; padding is stripped using BatchEncoding::lengths.

#include <blockbpe/blockbpe.hpp>

#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

using namespace blockbpe;

namespace {
thread_local std::string g_err;
thread_local std::vector<TokenId> g_partial;
thread_local std::size_t g_partial_passes = 0;

int err_code(const std::exception& e) {
  if (dynamic_cast<const MaxPassesError*>(&e)) return 6;
  if (dynamic_cast<const UsageError*>(&e)) return 1;
  if (dynamic_cast<const ParseError*>(&e)) return 2;
  if (dynamic_cast<const IntegrityError*>(&e)) return 3;
  if (dynamic_cast<const DecodeError*>(&e)) return 4;
  if (dynamic_cast<const ContractViolation*>(&e)) return 5;
  return 7;
}

struct RefTable {
  MergeTable table;
  SpecialTokenSet specials;
};

std::vector<std::string> unpack(const std::uint8_t* bytes, const std::uint64_t* offsets,
                                std::size_t n) {
  std::vector<std::string> rows(n);
  for (std::size_t i = 0; i < n; ++i)
    rows[i].assign(reinterpret_cast<const char*>(bytes) + offsets[i],
                   offsets[i + 1] - offsets[i]);
  return rows;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_table_load_files(const char* vocab, const char* merges, int canonical) {
  try {
    auto t = std::make_unique<RefTable>();
    t->table = load_merge_table_files(vocab, merges ? merges : "",
                                      canonical ? VocabFormat::canonical_json : VocabFormat::gpt2);
    return t.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// tokens: ids[i] owns bytes[tok_off[i] .. tok_off[i+1]); merges: rows of 4 u32.
void* ref_table_build(std::size_t n_tokens, const std::uint32_t* ids, const std::uint64_t* tok_off,
                      const std::uint8_t* tok_bytes, std::size_t n_merges,
                      const std::uint32_t* merges4) {
  try {
    auto t = std::make_unique<RefTable>();
    for (std::size_t i = 0; i < n_tokens; ++i)
      t->table.add_token(ids[i], std::string(reinterpret_cast<const char*>(tok_bytes) + tok_off[i],
                                             tok_off[i + 1] - tok_off[i]));
    for (std::size_t m = 0; m < n_merges; ++m)
      t->table.add_merge(merges4[4 * m], merges4[4 * m + 1], merges4[4 * m + 2],
                         merges4[4 * m + 3]);
    t->table.finalize();
    return t.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_table_free(void* h) { delete static_cast<RefTable*>(h); }

std::size_t ref_table_token_count(void* h) { return static_cast<RefTable*>(h)->table.token_count(); }
std::size_t ref_table_merge_count(void* h) { return static_cast<RefTable*>(h)->table.merge_count(); }

// Export tokens (sorted by id) and merges (sorted by rank). Call with null
// buffers first to get sizes (returned through the size pointers).
int ref_table_export(void* h, std::uint32_t* ids, std::uint64_t* tok_off, std::uint8_t* tok_bytes,
                     std::size_t* n_tokens, std::size_t* n_bytes, std::uint32_t* merges4,
                     std::size_t* n_merges) {
  const MergeTable& t = static_cast<RefTable*>(h)->table;
  std::vector<std::pair<TokenId, const std::string*>> toks;
  std::size_t total = 0;
  for (const auto& [id, b] : t.token_bytes()) {
    toks.push_back({id, &b});
    total += b.size();
  }
  std::sort(toks.begin(), toks.end());
  std::vector<std::array<std::uint32_t, 4>> ms;
  t.merges().for_each([&](PairKey k, const PairMap::Entry& e) {
    auto [l, r] = unpack_pair(k);
    ms.push_back({e.rank, l, r, e.merged});
  });
  std::sort(ms.begin(), ms.end());
  *n_tokens = toks.size();
  *n_bytes = total;
  *n_merges = ms.size();
  if (!ids) return 0;
  std::uint64_t off = 0;
  for (std::size_t i = 0; i < toks.size(); ++i) {
    ids[i] = toks[i].first;
    tok_off[i] = off;
    std::memcpy(tok_bytes + off, toks[i].second->data(), toks[i].second->size());
    off += toks[i].second->size();
  }
  tok_off[toks.size()] = off;
  for (std::size_t m = 0; m < ms.size(); ++m)
    for (int j = 0; j < 4; ++j) merges4[4 * m + j] = ms[m][j];
  return 0;
}

int ref_add_special(void* h, const char* bytes, std::uint32_t id, int role) {
  try {
    auto* t = static_cast<RefTable*>(h);
    if (role == 0) t->specials.add(bytes, id);
    if (role == 1) t->specials.set_bos(bytes);
    if (role == 2) t->specials.set_eos(bytes);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return err_code(e);
  }
}

// encode_batch (block engine) over rows chunked by `rows_per_call`, CSR out.
// Returns total tokens, or -(status) on error.
std::int64_t ref_encode_batch(void* h, const std::uint8_t* bytes, const std::uint64_t* offsets,
                              std::size_t n, std::uint32_t block_size, unsigned workers,
                              int add_bos, int add_eos, std::uint32_t* out_ids,
                              std::uint64_t* out_offsets, std::uint64_t capacity,
                              std::size_t rows_per_call, std::int64_t max_passes) {
  try {
    auto* t = static_cast<RefTable*>(h);
    PhasePool pool(workers);
    BlockConfig cfg{block_size, std::nullopt};
    if (max_passes > 0) cfg.max_passes = static_cast<std::size_t>(max_passes);
    if (rows_per_call == 0) rows_per_call = n ? n : 1;
    std::uint64_t pos = 0;
    out_offsets[0] = 0;
    for (std::size_t r0 = 0; r0 < n || (n == 0 && r0 == 0); r0 += rows_per_call) {
      if (n == 0) break;
      std::size_t r1 = std::min(n, r0 + rows_per_call);
      std::vector<std::string> rows(r1 - r0);
      for (std::size_t i = r0; i < r1; ++i)
        rows[i - r0].assign(reinterpret_cast<const char*>(bytes) + offsets[i],
                            offsets[i + 1] - offsets[i]);
      BatchEncoding enc;
      try {
        enc = encode_batch(rows, t->table, t->specials, cfg, 0, add_bos, add_eos, &pool);
      } catch (const MaxPassesError& e) {
        g_partial = e.partial_tokens;
        g_partial_passes = e.passes_run;
        throw;
      }
      for (std::size_t r = 0; r < enc.batch_size; ++r) {
        std::uint32_t len = enc.lengths[r];
        if (pos + len > capacity) throw UsageError("output capacity exceeded");
        std::memcpy(out_ids + pos, enc.ids.data() + r * enc.max_len, len * sizeof(std::uint32_t));
        pos += len;
        out_offsets[r0 + r + 1] = pos;
      }
    }
    return static_cast<std::int64_t>(pos);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -err_code(e);
  }
}

// The reference CLI's `tokenize` with the block engine (blockbpe_cli.cpp:73-127):
// encode_batch with pad_id, then write_batch_jsonl (binary == 0) or
// write_batch_binary; the bytes to out (at most cap). Returns the full length,
// or -(status) on error.
std::int64_t ref_write_batch(void* h, const std::uint8_t* bytes, const std::uint64_t* offsets, std::size_t n,
                             unsigned workers, int add_bos, int add_eos, std::uint32_t pad_id, int binary,
                             std::uint8_t* out, std::uint64_t cap) {
  try {
    auto* t = static_cast<RefTable*>(h);
    PhasePool pool(workers);
    std::vector<std::string> rows(n);
    for (std::size_t i = 0; i < n; ++i)
      rows[i].assign(reinterpret_cast<const char*>(bytes) + offsets[i], offsets[i + 1] - offsets[i]);
    const BatchEncoding enc =
        encode_batch(rows, t->table, t->specials, BlockConfig{256, std::nullopt}, pad_id, add_bos, add_eos, &pool);
    std::ostringstream os;
    if (binary) write_batch_binary(os, enc);
    else write_batch_jsonl(os, enc);
    const std::string b = os.str();
    if (out) std::memcpy(out, b.data(), std::min<std::uint64_t>(cap, b.size()));
    return static_cast<std::int64_t>(b.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -err_code(e);
  }
}

std::size_t ref_partial(std::uint32_t* out, std::size_t cap, std::size_t* passes) {
  if (passes) *passes = g_partial_passes;
  if (out) std::memcpy(out, g_partial.data(), std::min(cap, g_partial.size()) * 4);
  return g_partial.size();
}

// heap_bpe per row over PhasePool::run_items (the reference's fastest engine).
std::int64_t ref_encode_heap(void* h, const std::uint8_t* bytes, const std::uint64_t* offsets,
                             std::size_t n, unsigned workers, std::uint32_t* out_ids,
                             std::uint64_t* out_offsets, std::uint64_t capacity) {
  try {
    auto* t = static_cast<RefTable*>(h);
    PhasePool pool(workers);
    std::vector<TokenSeq> rows(n);
    auto row = [&](std::size_t r) {
      std::string_view s(reinterpret_cast<const char*>(bytes) + offsets[r],
                         offsets[r + 1] - offsets[r]);
      rows[r] = encode_reference(s, t->table, t->specials, PreSpec::byte_level(), RefEngine::heap);
    };
    if (pool.worker_count() >= 2)
      pool.run_items(n, row);
    else
      for (std::size_t r = 0; r < n; ++r) row(r);
    std::uint64_t pos = 0;
    out_offsets[0] = 0;
    for (std::size_t r = 0; r < n; ++r) {
      if (pos + rows[r].size() > capacity) throw UsageError("output capacity exceeded");
      std::memcpy(out_ids + pos, rows[r].data(), rows[r].size() * 4);
      pos += rows[r].size();
      out_offsets[r + 1] = pos;
    }
    return static_cast<std::int64_t>(pos);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -err_code(e);
  }
}

// encode_reference in pattern mode (ref_engines.hpp:119-146: pattern_pretokenize
// chunks, heap_bpe within each chunk), rows fanned over PhasePool::run_items.
std::int64_t ref_encode_pattern(void* h, const std::uint8_t* bytes, const std::uint64_t* offsets,
                                std::size_t n, unsigned workers, const char* pattern, std::uint32_t* out_ids,
                                std::uint64_t* out_offsets, std::uint64_t capacity) {
  try {
    auto* t = static_cast<RefTable*>(h);
    PhasePool pool(workers);
    std::vector<TokenSeq> rows(n);
    const PreSpec pre = PreSpec::with_pattern(pattern);
    auto row = [&](std::size_t r) {
      std::string_view s(reinterpret_cast<const char*>(bytes) + offsets[r], offsets[r + 1] - offsets[r]);
      rows[r] = encode_reference(s, t->table, t->specials, pre, RefEngine::heap);
    };
    if (pool.worker_count() >= 2)
      pool.run_items(n, row);
    else
      for (std::size_t r = 0; r < n; ++r) row(r);
    std::uint64_t pos = 0;
    out_offsets[0] = 0;
    for (std::size_t r = 0; r < n; ++r) {
      if (pos + rows[r].size() > capacity) throw UsageError("output capacity exceeded");
      std::memcpy(out_ids + pos, rows[r].data(), rows[r].size() * 4);
      pos += rows[r].size();
      out_offsets[r + 1] = pos;
    }
    return static_cast<std::int64_t>(pos);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -err_code(e);
  }
}

// pattern_pretokenize (pretokenize.hpp:252-258) of one string: chunk start
// offsets into starts[], returns the chunk count (or -code).
std::int64_t ref_pretokenize(const std::uint8_t* bytes, std::size_t len, const char* pattern,
                             std::uint64_t* starts, std::size_t cap) {
  try {
    std::string_view s(reinterpret_cast<const char*>(bytes), len);
    std::uint64_t pos = 0;
    std::size_t k = 0;
    for (const std::string& chunk : pattern_pretokenize(s, pattern)) {
      if (k < cap) starts[k] = pos;
      ++k;
      pos += chunk.size();
    }
    return static_cast<std::int64_t>(k);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -err_code(e);
  }
}

// block_bpe on explicit initial tokens with a pass trace (pass, min_rank, merges).
std::int64_t ref_block_bpe_trace(void* h, const std::uint32_t* tokens, std::size_t n,
                                 std::uint32_t block_size, std::int64_t max_passes,
                                 std::uint32_t* out, std::uint64_t* trace3,
                                 std::size_t trace_cap, std::size_t* n_passes) {
  try {
    auto* t = static_cast<RefTable*>(h);
    BlockConfig cfg{block_size, std::nullopt};
    if (max_passes > 0) cfg.max_passes = static_cast<std::size_t>(max_passes);
    PassTrace trace;
    TokenSeq res;
    try {
      res = block_bpe(TokenSeq(tokens, tokens + n), t->table, cfg, nullptr, &trace);
    } catch (const MaxPassesError& e) {
      g_partial = e.partial_tokens;
      g_partial_passes = e.passes_run;
      throw;
    }
    *n_passes = trace.size();
    for (std::size_t p = 0; p < trace.size() && p < trace_cap; ++p) {
      trace3[3 * p] = trace[p].pass_index;
      trace3[3 * p + 1] = trace[p].min_rank;
      trace3[3 * p + 2] = trace[p].merges_applied;
    }
    std::memcpy(out, res.data(), res.size() * 4);
    return static_cast<std::int64_t>(res.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -err_code(e);
  }
}

std::int64_t ref_naive_bpe(void* h, const std::uint32_t* tokens, std::size_t n,
                           std::uint32_t* out) {
  try {
    auto* t = static_cast<RefTable*>(h);
    TokenSeq res = naive_bpe(TokenSeq(tokens, tokens + n), t->table);
    std::memcpy(out, res.data(), res.size() * 4);
    return static_cast<std::int64_t>(res.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -err_code(e);
  }
}

std::uint32_t ref_byte_token(void* h, unsigned b) {
  return static_cast<RefTable*>(h)->table.byte_token(static_cast<unsigned char>(b));
}

}  // extern "C"
