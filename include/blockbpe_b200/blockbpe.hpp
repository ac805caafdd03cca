// blockbpe_b200/blockbpe.hpp -- C++ drop-in for the reference's batch-encode API.
//
// Header-only wrapper over the C-ABI (include/bbpe_b200.h, libbbpe_b200.so).
// Names, argument meaning and error behaviour mirror the reference library
// (namespace blockbpe, /root/reference/proj/include/blockbpe):
//
//   errors                 types.hpp:32-70
//   MergeTable, loaders    merge_table.hpp:223-305, 503-522
//   SpecialTokenSet        merge_table.hpp:309-369, validate_specials 374-385
//   split_specials         pretokenize.hpp:32-57
//   BlockConfig, block_bpe block_engine.hpp:18-32, 268-310 (PassTrace 42-47)
//   pair_ranks ... compact block_engine.hpp:189-256 (spec-level ops, on the GPU)
//   BatchEncoding/Limits   batch.hpp:21-42
//   encode_single/batch    batch.hpp:46-126
//   decode/decode_batch    merge_table.hpp:565-579, batch.hpp:128-154
//
// A caller switches by replacing `blockbpe::` with `blockbpe_b200::` and the
// PhasePool* argument with an Encoder* (one per GPU; nullptr = device 0).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <ostream>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../bbpe_b200.h"

namespace blockbpe_b200 {

using TokenId = std::uint32_t;
using Rank = std::uint32_t;
using TokenSeq = std::vector<TokenId>;

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct UsageError : Error {
  using Error::Error;
};
struct ParseError : Error {
  using Error::Error;
};
struct IntegrityError : Error {
  using Error::Error;
};
struct DecodeError : Error {
  using Error::Error;
};
struct ContractViolation : Error {
  using Error::Error;
};
struct MaxPassesError : Error {
  MaxPassesError(const std::string& what, TokenSeq partial, std::size_t passes)
      : Error(what), partial_tokens(std::move(partial)), passes_run(passes) {}
  TokenSeq partial_tokens;
  std::size_t passes_run;
};

namespace detail {
[[noreturn]] inline void raise(int rc) {
  const std::string msg = bbpe_last_error();
  switch (rc) {
    case BBPE_USAGE: throw UsageError(msg);
    case BBPE_PARSE: throw ParseError(msg);
    case BBPE_INTEGRITY: throw IntegrityError(msg);
    case BBPE_DECODE: throw DecodeError(msg);
    case BBPE_CONTRACT: throw ContractViolation(msg);
    case BBPE_MAX_PASSES: throw MaxPassesError(msg, {}, 0);
    default: throw Error(msg);
  }
}
inline void check(int rc) {
  if (rc != BBPE_OK) raise(rc);
}
}  // namespace detail

inline constexpr TokenId kInvalidToken = 0xFFFFFFFFu;

struct BlockConfig {
  std::uint32_t block_size = 256;
  std::optional<std::size_t> max_passes;
  void validate() const {
    if (block_size < 32 || block_size > 1024 || (block_size & (block_size - 1)) != 0)
      throw UsageError("block_size must be a power of two in [32, 1024], got " +
                       std::to_string(block_size));
    if (max_passes && *max_passes < 1) throw UsageError("max_passes must be >= 1");
  }
};

inline std::uint32_t coarsening_factor(std::size_t seq_len, const BlockConfig& config) {
  config.validate();
  return static_cast<std::uint32_t>((seq_len + config.block_size - 1) / config.block_size);
}

struct PassRecord {
  std::size_t pass_index;
  Rank min_rank;
  std::size_t merges_applied;
};
using PassTrace = std::vector<PassRecord>;

enum class VocabFormat { gpt2, canonical_json, binary };

inline VocabFormat parse_vocab_format(std::string_view name) {
  if (name == "gpt2") return VocabFormat::gpt2;
  if (name == "json" || name == "canonical_json") return VocabFormat::canonical_json;
  if (name == "binary" || name == "bbpt") return VocabFormat::binary;
  throw UsageError("unknown vocab format \"" + std::string(name) + "\"");
}

// Immutable merge table; device replicas are uploaded on first use per GPU.
class MergeTable {
 public:
  MergeTable() = default;
  explicit MergeTable(bbpe_table* h) : h_(h, bbpe_table_destroy) {}

  bbpe_table* handle() const { return h_.get(); }

  std::optional<Rank> rank_of(TokenId l, TokenId r) const {
    const Rank v = bbpe_table_rank_of(h_.get(), l, r, nullptr);
    if (v == 0xFFFFFFFFu) return std::nullopt;
    return v;
  }
  std::optional<TokenId> merged_of(TokenId l, TokenId r) const {
    TokenId m = 0;
    if (bbpe_table_rank_of(h_.get(), l, r, &m) == 0xFFFFFFFFu) return std::nullopt;
    return m;
  }
  TokenId byte_token(unsigned char b) const { return bbpe_table_byte_token(h_.get(), b); }
  std::size_t token_count() const { return info().token_count; }
  std::size_t merge_count() const { return info().merge_count; }
  std::size_t base_size() const { return info().base_size; }
  bbpe_table_info info() const {
    bbpe_table_info i{};
    detail::check(bbpe_table_get_info(h_.get(), &i));
    return i;
  }
  // Bytes of a table token (decode); nullopt for unknown ids.
  std::optional<std::string> bytes_of(TokenId id) const {
    std::uint8_t buf[1024];
    std::size_t len = 0;
    if (bbpe_decode(h_.get(), &id, 1, buf, sizeof buf, &len) != BBPE_OK) return std::nullopt;
    if (len <= sizeof buf) return std::string(reinterpret_cast<char*>(buf), len);
    std::string s(len, '\0');
    bbpe_decode(h_.get(), &id, 1, reinterpret_cast<std::uint8_t*>(s.data()), len, &len);
    return s;
  }

  // Construction mirroring add_token / add_merge / finalize (merge_table.hpp:257-297).
  static MergeTable build(const std::vector<std::pair<TokenId, std::string>>& tokens,
                          const std::vector<std::array<std::uint32_t, 4>>& merges);

 private:
  std::shared_ptr<bbpe_table> h_;
};

inline MergeTable load_merge_table_files(const std::string& vocab_path, const std::string& merges_path,
                                         VocabFormat format) {
  const int f = format == VocabFormat::gpt2 ? BBPE_FORMAT_GPT2
                : format == VocabFormat::canonical_json ? BBPE_FORMAT_CANONICAL
                                                        : BBPE_FORMAT_BINARY;
  bbpe_table* h = nullptr;
  detail::check(bbpe_table_load_files(vocab_path.c_str(),
                                      merges_path.empty() ? nullptr : merges_path.c_str(), f, &h));
  return MergeTable(h);
}

inline MergeTable MergeTable::build(const std::vector<std::pair<TokenId, std::string>>& tokens,
                                    const std::vector<std::array<std::uint32_t, 4>>& merges) {
  std::vector<std::uint32_t> ids;
  std::vector<std::uint64_t> off{0};
  std::string blob;
  for (const auto& [id, b] : tokens) {
    ids.push_back(id);
    blob += b;
    off.push_back(blob.size());
  }
  std::vector<std::uint32_t> m4;
  for (const auto& m : merges) m4.insert(m4.end(), m.begin(), m.end());
  if (blob.empty()) blob.push_back('\0');
  bbpe_table* h = nullptr;
  detail::check(bbpe_table_create(ids.size(), ids.data(), off.data(),
                                  reinterpret_cast<const std::uint8_t*>(blob.data()), merges.size(),
                                  m4.empty() ? nullptr : m4.data(), &h));
  return MergeTable(h);
}

class SpecialTokenSet {
 public:
  void add(std::string bytes, TokenId id) {
    if (bytes.empty()) throw UsageError("special token byte string may not be empty");
    for (const auto& e : entries_)
      if (e.first == bytes) throw UsageError("duplicate special token \"" + bytes + "\"");
    auto it = entries_.begin();
    while (it != entries_.end() && it->first.size() >= bytes.size()) ++it;
    entries_.insert(it, {std::move(bytes), id});
  }
  bool empty() const { return entries_.empty(); }
  std::size_t size() const { return entries_.size(); }
  const std::vector<std::pair<std::string, TokenId>>& entries() const { return entries_; }
  const std::string* bytes_of(TokenId id) const {
    for (const auto& e : entries_)
      if (e.second == id) return &e.first;
    return nullptr;
  }
  bool contains_id(TokenId id) const { return bytes_of(id) != nullptr; }
  std::optional<std::pair<std::size_t, TokenId>> match(std::string_view text, std::size_t pos) const {
    for (const auto& [b, id] : entries_)
      if (b.size() <= text.size() - pos && text.compare(pos, b.size(), b) == 0)
        return std::make_pair(b.size(), id);
    return std::nullopt;
  }
  std::optional<TokenId> bos_id() const { return bos_; }
  std::optional<TokenId> eos_id() const { return eos_; }
  void set_bos(std::string_view b) { bos_ = require(b, "bos"); }
  void set_eos(std::string_view b) { eos_ = require(b, "eos"); }

 private:
  TokenId require(std::string_view b, const char* what) const {
    for (const auto& [e, id] : entries_)
      if (e == b) return id;
    throw UsageError(std::string(what) + " token \"" + std::string(b) +
                     "\" is not in the special token set");
  }
  std::vector<std::pair<std::string, TokenId>> entries_;
  std::optional<TokenId> bos_, eos_;
};

struct Segment {
  enum class Kind { literal, special };
  Kind kind;
  std::string bytes;
  std::optional<TokenId> special_id;
};

inline std::vector<Segment> split_specials(std::string_view input, const SpecialTokenSet& specials) {
  std::vector<Segment> out;
  std::string pending;
  std::size_t pos = 0;
  auto flush = [&] {
    if (!pending.empty()) {
      out.push_back({Segment::Kind::literal, std::move(pending), std::nullopt});
      pending.clear();
    }
  };
  while (pos < input.size()) {
    if (!specials.empty())
      if (auto m = specials.match(input, pos)) {
        flush();
        out.push_back({Segment::Kind::special, std::string(input.substr(pos, m->first)), m->second});
        pos += m->first;
        continue;
      }
    pending.push_back(input[pos++]);
  }
  flush();
  return out;
}

// One encode context on one GPU (the PhasePool* of the reference signatures).
class Encoder {
 public:
  explicit Encoder(int device = 0, BlockConfig cfg = {}, bool piece_memo = true) {
    cfg.validate();
    bbpe_config c{cfg.block_size, cfg.max_passes ? static_cast<std::int64_t>(*cfg.max_passes) : 0,
                  BBPE_ENGINE_PIECES, 0, piece_memo ? 1 : 0, 0, 0};
    bbpe_ctx* h = nullptr;
    detail::check(bbpe_ctx_create(device, &c, &h));
    h_.reset(h);
    cfg_ = c;
  }
  bbpe_ctx* handle() const { return h_.get(); }
  void configure(const BlockConfig& cfg, bool block_engine = false, bool piece_memo = true) {
    cfg.validate();
    bbpe_config c{cfg.block_size, cfg.max_passes ? static_cast<std::int64_t>(*cfg.max_passes) : 0,
                  block_engine ? BBPE_ENGINE_BLOCK : BBPE_ENGINE_PIECES, 0, piece_memo ? 1 : 0, 0, pattern_};
    detail::check(bbpe_ctx_set_config(h_.get(), &c));
    cfg_ = c;
  }
  // Split pattern of later encodes: "gpt2" (the reference's built-in gpt2
  // matcher, pattern_pretokenize) or "" (byte-level, encode_batch).
  void set_split_pattern(std::string_view name) {
    if (name != "" && name != "gpt2")
      throw UsageError("only the gpt2 split pattern runs on the device, got \"" + std::string(name) + "\"");
    pattern_ = name == "gpt2" ? 1 : 0;
    cfg_.pattern = pattern_;
    detail::check(bbpe_ctx_set_config(h_.get(), &cfg_));
  }
  // Packed rows -> CSR.
  void encode_csr(const MergeTable& t, const std::string& bytes, const std::vector<std::uint64_t>& offsets,
                  std::vector<TokenId>& ids, std::vector<std::uint64_t>& out_offsets) {
    const std::size_t n = offsets.empty() ? 0 : offsets.size() - 1;
    ids.resize(std::max<std::uint64_t>(offsets.empty() ? 0 : offsets.back() - offsets.front(), 1));
    out_offsets.resize(n + 1);
    detail::check(bbpe_encode(h_.get(), t.handle(), reinterpret_cast<const std::uint8_t*>(bytes.data()),
                              offsets.data(), n, ids.data(), ids.size(), out_offsets.data(), nullptr));
    ids.resize(out_offsets[n]);
  }
  // encode_batch's rows as CSR: split at `specials` on the device, BOS/EOS
  // added (bbpe_ctx_set_specials + bbpe_encode_batch).
  // The ctx's special-token set (split by encode, resolved by decode).
  void set_specials(const SpecialTokenSet& specials) {
    std::string blob;
    std::vector<std::uint64_t> so{0};
    std::vector<std::uint32_t> sid;
    for (const auto& [b, id] : specials.entries()) {
      blob += b;
      so.push_back(blob.size());
      sid.push_back(id);
    }
    detail::check(bbpe_ctx_set_specials(h_.get(), sid.size(), reinterpret_cast<const std::uint8_t*>(blob.data()),
                                        so.data(), sid.data()));
  }
  void encode_rows_csr(const MergeTable& t, const SpecialTokenSet& specials, bool add_bos, bool add_eos,
                       const std::string& bytes, const std::vector<std::uint64_t>& offsets, std::vector<TokenId>& ids,
                       std::vector<std::uint64_t>& out_offsets) {
    set_specials(specials);
    const std::size_t n = offsets.size() - 1;
    ids.resize(offsets.back() - offsets.front() + 2 * n + 1);
    out_offsets.resize(n + 1);
    std::uint64_t k = 0;
    detail::check(bbpe_encode_batch(h_.get(), t.handle(), reinterpret_cast<const std::uint8_t*>(bytes.data()),
                                    offsets.data(), n, add_bos ? *specials.bos_id() : 0xFFFFFFFFu,
                                    add_eos ? *specials.eos_id() : 0xFFFFFFFFu, ids.data(), ids.size(),
                                    out_offsets.data(), &k));
    ids.resize(k);
  }

 private:
  struct Del {
    void operator()(bbpe_ctx* c) const { bbpe_ctx_destroy(c); }
  };
  std::unique_ptr<bbpe_ctx, Del> h_;
  bbpe_config cfg_{};
  int pattern_ = 0;
};

inline Encoder& default_encoder() {
  static Encoder e(0);
  return e;
}

struct BatchEncoding {
  std::size_t batch_size = 0;
  std::size_t max_len = 0;
  TokenId pad_id = 0;
  std::vector<TokenId> ids;
  std::vector<std::uint32_t> lengths;
  std::vector<std::uint8_t> mask;
  std::size_t truncated_rows = 0;
  TokenId at(std::size_t row, std::size_t col) const { return ids[row * max_len + col]; }
  TokenSeq row(std::size_t r) const {
    const TokenId* b = ids.data() + r * max_len;
    return TokenSeq(b, b + lengths[r]);
  }
};

struct BatchLimits {
  std::optional<std::uint32_t> max_len;
};

// batch.hpp:64-126 -- specials split, literal segments merged and BOS/EOS
// added on the GPU; padding, mask and truncation assembled here.
inline BatchEncoding encode_batch(const std::vector<std::string>& inputs, const MergeTable& table,
                                  const SpecialTokenSet& specials, const BlockConfig& config,
                                  TokenId pad_id, bool add_bos, bool add_eos, Encoder* encoder = nullptr,
                                  const BatchLimits& limits = {}) {
  config.validate();
  if (add_bos && !specials.bos_id()) throw UsageError("add_bos requires a bos entry in the special token set");
  if (add_eos && !specials.eos_id()) throw UsageError("add_eos requires an eos entry in the special token set");
  Encoder& enc = encoder ? *encoder : default_encoder();
  enc.configure(config);
  // Rows split at the specials, encoded, BOS/EOS added -- all on the device.
  std::string blob;
  std::vector<std::uint64_t> offs{0};
  for (const std::string& in : inputs) {
    blob += in;
    offs.push_back(blob.size());
  }
  std::vector<TokenId> ids;
  std::vector<std::uint64_t> oo;
  enc.encode_rows_csr(table, specials, add_bos, add_eos, blob, offs, ids, oo);
  std::vector<TokenSeq> rows(inputs.size());
  for (std::size_t r = 0; r < inputs.size(); ++r) rows[r].assign(ids.begin() + oo[r], ids.begin() + oo[r + 1]);
  BatchEncoding out;
  out.batch_size = inputs.size();
  out.pad_id = pad_id;
  std::size_t widest = 0;
  for (auto& row : rows) widest = std::max(widest, row.size());
  if (limits.max_len) {
    for (auto& row : rows)
      if (row.size() > *limits.max_len) {
        row.resize(*limits.max_len);
        ++out.truncated_rows;
      }
    out.max_len = *limits.max_len;
  } else {
    out.max_len = widest;
  }
  out.ids.assign(out.batch_size * out.max_len, pad_id);
  out.mask.assign(out.batch_size * out.max_len, 0);
  out.lengths.resize(out.batch_size);
  for (std::size_t r = 0; r < rows.size(); ++r) {
    out.lengths[r] = static_cast<std::uint32_t>(rows[r].size());
    for (std::size_t c = 0; c < rows[r].size(); ++c) {
      out.ids[r * out.max_len + c] = rows[r][c];
      out.mask[r * out.max_len + c] = 1;
    }
  }
  return out;
}

// validate_specials (merge_table.hpp:374-385): a special id may not be a
// base byte token nor the merged result of any pair.
inline void validate_specials(const MergeTable& table, const SpecialTokenSet& specials) {
  for (const auto& [b, id] : specials.entries()) {
    (void)b;
    auto tb = table.bytes_of(id);
    if (tb && tb->size() == 1 && table.byte_token(static_cast<unsigned char>((*tb)[0])) == id)
      throw IntegrityError("special id " + std::to_string(id) + " is a base byte token");
  }
  std::uint64_t nt = 0, nb = 0, nm = 0;
  detail::check(bbpe_table_export(table.handle(), nullptr, nullptr, nullptr, &nt, &nb, nullptr, &nm));
  std::vector<std::uint32_t> ids(nt), m4(4 * nm + 4);
  std::vector<std::uint64_t> off(nt + 1);
  std::vector<std::uint8_t> blob(nb + 1);
  detail::check(bbpe_table_export(table.handle(), ids.data(), off.data(), blob.data(), &nt, &nb, m4.data(), &nm));
  for (std::uint64_t k = 0; k < nm; ++k)
    if (specials.contains_id(m4[4 * k + 3]))
      throw IntegrityError("special id " + std::to_string(m4[4 * k + 3]) + " collides with a merge-derived token");
}

// write_batch_jsonl (batch.hpp:157-166): {"ids":[...],"len":n} per row, the
// compact nlohmann dump byte for byte.
inline void write_batch_jsonl(std::ostream& os, const BatchEncoding& e) {
  std::string line;
  for (std::size_t r = 0; r < e.batch_size; ++r) {
    line.assign("{\"ids\":[");
    for (std::uint32_t c = 0; c < e.lengths[r]; ++c) {
      if (c) line.push_back(',');
      line += std::to_string(e.ids[r * e.max_len + c]);
    }
    line += "],\"len\":" + std::to_string(e.lengths[r]) + "}\n";
    os.write(line.data(), static_cast<std::streamsize>(line.size()));
  }
}

// write_batch_binary (batch.hpp:205-213): "BBPE", u32 batch, max_len, pad_id,
// row-major u32 ids, little-endian.
inline void write_batch_binary(std::ostream& os, const BatchEncoding& e) {
  auto put = [&](std::uint32_t v) {
    const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                                static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
    os.write(reinterpret_cast<const char*>(b), 4);
  };
  os.write("BBPE", 4);
  put(static_cast<std::uint32_t>(e.batch_size));
  put(static_cast<std::uint32_t>(e.max_len));
  put(e.pad_id);
  for (TokenId id : e.ids) put(id);
}

inline TokenSeq encode_single(std::string_view input, const MergeTable& table, const SpecialTokenSet& specials,
                              const BlockConfig& config, Encoder* encoder = nullptr) {
  return encode_batch({std::string(input)}, table, specials, config, 0, false, false, encoder).row(0);
}

// block_engine.hpp:268-310 on explicit ids (one CTA pass loop on the GPU).
inline TokenSeq block_bpe(const TokenSeq& tokens, const MergeTable& table, const BlockConfig& config,
                          Encoder* encoder = nullptr, PassTrace* trace = nullptr) {
  Encoder& enc = encoder ? *encoder : default_encoder();
  enc.configure(config);
  TokenSeq out(tokens.size() + 1);
  std::size_t out_n = 0, passes = 0;
  std::vector<std::uint64_t> tr(trace ? 3 * (tokens.size() + 1) : 3);
  const int rc = bbpe_block_bpe(enc.handle(), table.handle(), tokens.data(), tokens.size(), out.data(), &out_n,
                                trace ? tr.data() : nullptr, trace ? tokens.size() + 1 : 0, &passes);
  out.resize(out_n);
  if (rc == BBPE_MAX_PASSES) throw MaxPassesError(bbpe_last_error(), out, passes);
  detail::check(rc);
  if (trace)
    for (std::size_t p = 0; p < passes && p <= tokens.size(); ++p)
      trace->push_back({static_cast<std::size_t>(tr[3 * p]), static_cast<Rank>(tr[3 * p + 1]),
                        static_cast<std::size_t>(tr[3 * p + 2])});
  return out;
}

// ---- spec-level operations (block_engine.hpp:189-256), run on the GPU ----
inline std::vector<std::optional<Rank>> pair_ranks(const TokenSeq& tokens, const MergeTable& table,
                                                   Encoder* encoder = nullptr) {
  if (tokens.size() < 2) return {};
  Encoder& enc = encoder ? *encoder : default_encoder();
  std::vector<Rank> raw(tokens.size() - 1);
  detail::check(bbpe_pair_ranks(enc.handle(), table.handle(), tokens.data(), tokens.size(), raw.data()));
  std::vector<std::optional<Rank>> out(raw.size());
  for (std::size_t i = 0; i < raw.size(); ++i)
    if (raw[i] != 0xFFFFFFFFu) out[i] = raw[i];
  return out;
}

inline std::optional<Rank> min_rank_reduce(const std::vector<std::optional<Rank>>& ranks,
                                           Encoder* encoder = nullptr) {
  Encoder& enc = encoder ? *encoder : default_encoder();
  std::vector<Rank> raw(ranks.size());
  for (std::size_t i = 0; i < ranks.size(); ++i) raw[i] = ranks[i] ? *ranks[i] : 0xFFFFFFFFu;
  Rank m = 0;
  detail::check(bbpe_min_rank_reduce(enc.handle(), raw.data(), raw.size(), &m));
  return m == 0xFFFFFFFFu ? std::nullopt : std::optional<Rank>(m);
}

inline std::vector<std::uint8_t> mark_merges(const TokenSeq& tokens, const MergeTable& table, Rank min_rank,
                                             Encoder* encoder = nullptr) {
  Encoder& enc = encoder ? *encoder : default_encoder();
  std::vector<std::uint8_t> flags(tokens.size(), 0);
  detail::check(bbpe_mark_merges(enc.handle(), table.handle(), tokens.data(), tokens.size(), min_rank, flags.data()));
  return flags;
}

inline std::vector<std::uint32_t> exclusive_scan(const std::vector<std::uint8_t>& flags, Encoder* encoder = nullptr) {
  Encoder& enc = encoder ? *encoder : default_encoder();
  std::vector<std::uint32_t> offsets(flags.size(), 0);
  detail::check(bbpe_exclusive_scan(enc.handle(), flags.data(), flags.size(), offsets.data()));
  return offsets;
}

inline TokenSeq compact(const TokenSeq& tokens, const MergeTable& table, const std::vector<std::uint8_t>& flags,
                        const std::vector<std::uint32_t>& offsets, Encoder* encoder = nullptr) {
  Encoder& enc = encoder ? *encoder : default_encoder();
  TokenSeq out(tokens.size() + 1);
  std::size_t n = 0;
  detail::check(bbpe_compact(enc.handle(), table.handle(), tokens.data(), tokens.size(), flags.data(), flags.size(),
                             offsets.data(), offsets.size(), out.data(), &n));
  out.resize(n);
  return out;
}

inline std::string decode(const MergeTable& table, const SpecialTokenSet& specials, const TokenSeq& ids) {
  std::string out;
  for (std::size_t i = 0; i < ids.size(); ++i) {
    if (auto b = table.bytes_of(ids[i])) {
      out += *b;
    } else if (const std::string* s = specials.bytes_of(ids[i])) {
      out += *s;
    } else {
      throw DecodeError("unknown token id " + std::to_string(ids[i]) + " at index " + std::to_string(i));
    }
  }
  return out;
}

// decode_batch (batch.hpp:128-154). With an Encoder, rows without special
// ids (or with skip_specials) decode on its GPU (bbpe_decode_batch, SURVEY
// §8f(2)); the result and the row-tagged DecodeError are the same.
// decode_batch (batch.hpp:128-154) on the GPU: the rows' ids as CSR, ids the
// table lacks resolved through the special tokens, skip_specials dropping
// special ids (bbpe_decode_batch_ex); "row r: unknown token id ..." errors.
inline std::vector<std::string> decode_batch(const BatchEncoding& enc, const MergeTable& table,
                                             const SpecialTokenSet& specials, bool skip_specials,
                                             Encoder* gpu = nullptr) {
  Encoder& e = gpu ? *gpu : default_encoder();
  e.set_specials(specials);
  std::vector<std::uint32_t> ids;
  std::vector<std::uint64_t> off{0};
  for (std::size_t r = 0; r < enc.batch_size; ++r) {
    const TokenSeq row = enc.row(r);
    ids.insert(ids.end(), row.begin(), row.end());
    off.push_back(ids.size());
  }
  // First call sizes the output (cap 0), second fills it.
  std::vector<std::uint8_t> bytes;
  std::vector<std::uint64_t> boff(enc.batch_size + 1);
  std::uint64_t total = 0;
  detail::check(bbpe_decode_batch_ex(e.handle(), table.handle(), ids.data(), off.data(), enc.batch_size,
                                     skip_specials ? 1 : 0, nullptr, 0, boff.data(), &total));
  bytes.resize(std::max<std::uint64_t>(total, 1));
  detail::check(bbpe_decode_batch_ex(e.handle(), table.handle(), ids.data(), off.data(), enc.batch_size,
                                     skip_specials ? 1 : 0, bytes.data(), total, boff.data(), &total));
  std::vector<std::string> out(enc.batch_size);
  for (std::size_t r = 0; r < enc.batch_size; ++r)
    out[r].assign(reinterpret_cast<const char*>(bytes.data()) + boff[r], boff[r + 1] - boff[r]);
  return out;
}

}  // namespace blockbpe_b200
