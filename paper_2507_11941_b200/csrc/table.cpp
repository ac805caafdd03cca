// table.cpp -- merge-table loading, validation and the device hash layout.
//
// Host side of the table (the reference's MergeTable, merge_table.hpp:223-305):
//   * loaders for the gpt2 vocab.json+merges.txt format (merge_table.hpp:399-459),
//     the canonical JSON format (473-497) and this repo's .bbpt binary format;
//   * the same structural checks as add_token/add_merge/finalize (257-297), with
//     the reference's error messages;
//   * the device layout: dense ids/ranks, a bucketised open-addressing pair table
//     (replaces PairMap, 140-217), the byte LUT (246) and the junction-bigram set
//     that licenses the piece decomposition.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <memory>
#include <cstring>
#include <fstream>
#include <sstream>
#include <unordered_set>

#include <nlohmann/json.hpp>

#include "bbpe_internal.h"

namespace bbpe {

uint64_t mix64(uint64_t h) {
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdULL;
  h ^= h >> 33;
  return h;
}

namespace {

std::string to_s(uint64_t v) { return std::to_string(v); }

// gpt2 byte <-> codepoint bijection (merge_table.hpp:30-53).
const uint32_t* byte_to_cp() {
  static uint32_t t[256];
  static bool init = false;
  if (!init) {
    uint32_t next = 256;
    for (int b = 0; b < 256; ++b) {
      bool direct = (b >= 33 && b <= 126) || (b >= 161 && b <= 172) || (b >= 174 && b <= 255);
      t[b] = direct ? b : next++;
    }
    init = true;
  }
  return t;
}

const int* cp_to_byte() {
  static int inv[324];
  static bool init = false;
  if (!init) {
    for (int& v : inv) v = -1;
    const uint32_t* f = byte_to_cp();
    for (int b = 0; b < 256; ++b) inv[f[b]] = b;
    init = true;
  }
  return inv;
}

// One UTF-8 scalar with the reference's lenient handling (merge_table.hpp:78-106).
uint32_t next_utf8(const std::string& s, size_t& pos) {
  auto by = [&](size_t i) { return static_cast<unsigned char>(s[i]); };
  unsigned char c0 = by(pos);
  if (c0 < 0x80) { pos += 1; return c0; }
  if ((c0 >> 5) == 0x6 && pos + 1 < s.size()) {
    uint32_t cp = ((c0 & 0x1fu) << 6) | (by(pos + 1) & 0x3fu);
    pos += 2;
    return cp;
  }
  if ((c0 >> 4) == 0xe && pos + 2 < s.size()) {
    uint32_t cp = ((c0 & 0x0fu) << 12) | ((by(pos + 1) & 0x3fu) << 6) | (by(pos + 2) & 0x3fu);
    pos += 3;
    return cp;
  }
  if ((c0 >> 3) == 0x1e && pos + 3 < s.size()) {
    uint32_t cp = ((c0 & 0x07u) << 18) | ((by(pos + 1) & 0x3fu) << 12) |
                  ((by(pos + 2) & 0x3fu) << 6) | (by(pos + 3) & 0x3fu);
    pos += 4;
    return cp;
  }
  pos += 1;
  return c0;
}

// merge_table.hpp:110-125
std::string gpt2_token_to_bytes(const std::string& token) {
  const int* inv = cp_to_byte();
  std::string out;
  size_t pos = 0;
  while (pos < token.size()) {
    size_t before = pos;
    uint32_t cp = next_utf8(token, pos);
    if (cp < 324 && inv[cp] >= 0)
      out.push_back(static_cast<char>(inv[cp]));
    else
      out.append(token.substr(before, pos - before));
  }
  return out;
}

// Staging builder mirroring MergeTable::add_token/add_merge (257-269).
struct Builder {
  std::vector<std::pair<uint32_t, std::string>> tokens;
  std::unordered_map<uint32_t, size_t> tok_pos;
  std::vector<std::array<uint32_t, 4>> merges;  // rank, left, right, merged
  std::unordered_set<uint32_t> ranks;
  std::unordered_set<uint64_t> pairs;

  void add_token(uint32_t id, std::string bytes) {
    if (!tok_pos.emplace(id, tokens.size()).second)
      throw integrity_error("duplicate token id " + to_s(id));
    tokens.emplace_back(id, std::move(bytes));
  }
  void add_merge(uint32_t rank, uint32_t l, uint32_t r, uint32_t m) {
    if (!ranks.insert(rank).second) throw integrity_error("duplicate merge rank " + to_s(rank));
    if (!pairs.insert((uint64_t(l) << 32) | r).second)
      throw integrity_error("duplicate merge pair (" + to_s(l) + ", " + to_s(r) + ")");
    merges.push_back({rank, l, r, m});
  }
};

std::string bytes_from_json_array(const nlohmann::json& arr, const std::string& where) {
  if (!arr.is_array()) throw parse_error(where + ": token bytes must be an array");
  std::string out;
  for (const auto& v : arr) {
    if (!v.is_number_unsigned() || v.get<unsigned>() > 255)
      throw parse_error(where + ": byte values must be integers in [0, 255]");
    out.push_back(static_cast<char>(v.get<unsigned>()));
  }
  return out;
}

bbpe_table* finalize(Builder& b);

// merge_table.hpp:399-459
bbpe_table* load_gpt2(const std::string& vocab_path, const std::string& merges_path) {
  std::ifstream vf(vocab_path, std::ios::binary);
  if (!vf) throw usage_error("cannot open vocab file " + vocab_path);
  std::ifstream mf(merges_path, std::ios::binary);
  if (!mf) throw usage_error("cannot open merges file " + merges_path);
  nlohmann::json vocab;
  try {
    vf >> vocab;
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(vocab_path + ": " + e.what());
  }
  if (!vocab.is_object()) throw parse_error(vocab_path + ": expected a token -> id object");
  Builder b;
  std::unordered_map<std::string, uint32_t> by_string;
  by_string.reserve(vocab.size());
  for (auto it = vocab.begin(); it != vocab.end(); ++it) {
    if (!it.value().is_number_unsigned())
      throw parse_error(vocab_path + ": id for \"" + it.key() + "\" is not a non-negative integer");
    uint32_t id = it.value().get<uint32_t>();
    b.add_token(id, gpt2_token_to_bytes(it.key()));
    by_string.emplace(it.key(), id);
  }
  std::string line;
  size_t line_no = 0;
  uint32_t rank = 0;
  bool first = true;
  while (std::getline(mf, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (first) {
      first = false;
      if (line.rfind("#version", 0) == 0) continue;
    }
    if (line.empty()) continue;
    auto fail = [&](const std::string& why) {
      return parse_error(merges_path + ":" + to_s(line_no) + ": " + why);
    };
    size_t space = line.find(' ');
    if (space == std::string::npos || space == 0 || space + 1 >= line.size() ||
        line.find(' ', space + 1) != std::string::npos)
      throw fail("expected exactly \"left right\"");
    std::string left = line.substr(0, space), right = line.substr(space + 1);
    auto lit = by_string.find(left);
    auto rit = by_string.find(right);
    if (lit == by_string.end()) throw fail("left token \"" + left + "\" not in vocab");
    if (rit == by_string.end()) throw fail("right token \"" + right + "\" not in vocab");
    auto mit = by_string.find(left + right);
    if (mit == by_string.end())
      throw integrity_error(merges_path + ":" + to_s(line_no) + ": merged token for pair (" +
                            to_s(lit->second) + ", " + to_s(rit->second) + ") not in vocab");
    b.add_merge(rank++, lit->second, rit->second, mit->second);
  }
  return finalize(b);
}

// merge_table.hpp:473-497
bbpe_table* load_canonical(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw usage_error("cannot open vocab file " + path);
  nlohmann::json doc;
  try {
    f >> doc;
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(path + ": " + e.what());
  }
  if (!doc.is_object() || !doc.contains("tokens") || !doc.contains("merges"))
    throw parse_error(path + ": expected object with \"tokens\" and \"merges\"");
  Builder b;
  try {
    for (const auto& e : doc["tokens"]) {
      if (!e.is_array() || e.size() != 2 || !e[0].is_number_unsigned())
        throw parse_error(path + ": token entries are [id, [byte, ...]]");
      b.add_token(e[0].get<uint32_t>(), bytes_from_json_array(e[1], path));
    }
    for (const auto& e : doc["merges"]) {
      if (!e.is_array() || e.size() != 4)
        throw parse_error(path + ": merge entries are [rank, left, right, merged]");
      b.add_merge(e[0].get<uint32_t>(), e[1].get<uint32_t>(), e[2].get<uint32_t>(),
                  e[3].get<uint32_t>());
    }
  } catch (const nlohmann::json::exception& e) {
    throw parse_error(path + ": " + e.what());
  }
  return finalize(b);
}

// .bbpt: "BBPT", u32 version(1), u64 n_tokens, u64 n_bytes, u64 n_merges,
//        u32 ids[n_tokens], u64 tok_off[n_tokens+1], u8 bytes[n_bytes],
//        u32 merges4[4*n_merges]  (all little-endian)
bbpe_table* load_binary(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw usage_error("cannot open table file " + path);
  std::string blob((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  size_t pos = 0;
  auto take = [&](void* dst, size_t n) {
    if (pos + n > blob.size()) throw parse_error(path + ": truncated table file");
    std::memcpy(dst, blob.data() + pos, n);
    pos += n;
  };
  char magic[4];
  take(magic, 4);
  if (std::memcmp(magic, "BBPT", 4) != 0) throw parse_error(path + ": bad magic, not a .bbpt table");
  uint32_t version;
  take(&version, 4);
  if (version != 1) throw parse_error(path + ": unsupported .bbpt version " + to_s(version));
  uint64_t nt, nb, nm;
  take(&nt, 8);
  take(&nb, 8);
  take(&nm, 8);
  if (nt > (1ull << 32) || nb > (1ull << 36) || nm > (1ull << 32))
    throw parse_error(path + ": implausible sizes");
  // The payload the header announces must be present before anything is
  // allocated from it (no overflow: the bounds above keep it < 2^40).
  if (nt * 4 + (nt + 1) * 8 + nb + nm * 16 > blob.size() - pos) throw parse_error(path + ": truncated table file");
  std::vector<uint32_t> ids(nt);
  std::vector<uint64_t> off(nt + 1);
  std::vector<uint8_t> bytes(nb);
  std::vector<uint32_t> m4(4 * nm);
  take(ids.data(), nt * 4);
  take(off.data(), (nt + 1) * 8);
  take(bytes.data(), nb);
  take(m4.data(), nm * 16);
  Builder b;
  for (uint64_t i = 0; i < nt; ++i) {
    if (off[i] > off[i + 1] || off[i + 1] > nb) throw parse_error(path + ": bad token offsets");
    b.add_token(ids[i], std::string(reinterpret_cast<const char*>(bytes.data()) + off[i],
                                    off[i + 1] - off[i]));
  }
  for (uint64_t m = 0; m < nm; ++m) b.add_merge(m4[4 * m], m4[4 * m + 1], m4[4 * m + 2], m4[4 * m + 3]);
  return finalize(b);
}

// MergeTable::finalize (merge_table.hpp:272-297) + the device layout.
bbpe_table* finalize(Builder& b) {
  auto t = std::make_unique<bbpe_table>();
  std::sort(b.tokens.begin(), b.tokens.end(),
            [](const auto& x, const auto& y) { return x.first < y.first; });
  t->ids.reserve(b.tokens.size());
  t->tok_off.reserve(b.tokens.size() + 1);
  t->tok_off.push_back(0);
  for (auto& [id, bytes] : b.tokens) {
    t->index_of[id] = static_cast<uint32_t>(t->ids.size());
    t->ids.push_back(id);
    t->tok_bytes.insert(t->tok_bytes.end(), bytes.begin(), bytes.end());
    t->tok_off.push_back(t->tok_bytes.size());
    t->max_id = std::max(t->max_id, id);
  }
  for (uint32_t& v : t->byte_tokens) v = kInvalidToken;
  for (size_t i = 0; i < t->ids.size(); ++i) {
    if (t->tok_off[i + 1] - t->tok_off[i] != 1) continue;
    unsigned char byte = t->tok_bytes[t->tok_off[i]];
    if (t->byte_tokens[byte] != kInvalidToken)
      throw integrity_error("two tokens share byte value " + to_s(byte));
    t->byte_tokens[byte] = t->ids[i];
    ++t->base_size;
  }
  std::sort(b.merges.begin(), b.merges.end());
  auto bytes_of = [&](uint32_t id, const uint8_t** p, size_t* n) {
    auto it = t->index_of.find(id);
    if (it == t->index_of.end()) return false;
    *p = t->tok_bytes.data() + t->tok_off[it->second];
    *n = t->tok_off[it->second + 1] - t->tok_off[it->second];
    return true;
  };
  // The reference iterates in hash-slot order and reports the first failing
  // pair it meets; any failing pair raises the same exception type.
  for (const auto& m : b.merges) {
    const uint8_t *lb, *rb, *mb;
    size_t ln, rn, mn;
    std::string name = "(" + to_s(m[1]) + ", " + to_s(m[2]) + ")";
    if (!bytes_of(m[1], &lb, &ln) || !bytes_of(m[2], &rb, &rn) || !bytes_of(m[3], &mb, &mn))
      throw integrity_error("merge pair " + name + " references unknown token id");
    if (mn != ln + rn || std::memcmp(mb, lb, ln) != 0 || std::memcmp(mb + ln, rb, rn) != 0)
      throw integrity_error("merged token bytes mismatch for pair " + name);
  }
  for (size_t i = 0; i < b.merges.size(); ++i) {
    const auto& m = b.merges[i];
    t->m_rank.push_back(m[0]);
    t->m_left.push_back(m[1]);
    t->m_right.push_back(m[2]);
    t->m_merged.push_back(m[3]);
    t->pair_index[(uint64_t(m[1]) << 32) | m[2]] = static_cast<uint32_t>(i);
  }
  build_device_layout(*t);
  return t.release();
}

int bits_for(uint64_t v) {  // smallest b with v < 2^b
  int b = 0;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

}  // namespace

void build_device_layout(bbpe_table& t) {
  const size_t M = t.m_rank.size();
  // Rank consistency (information only; results never depend on it).
  {
    std::unordered_map<uint32_t, size_t> created;  // id -> first position creating it
    for (size_t i = 0; i < M; ++i) created.emplace(t.m_merged[i], i);
    t.rank_consistent = true;
    for (size_t i = 0; i < M && t.rank_consistent; ++i) {
      for (uint32_t part : {t.m_left[i], t.m_right[i]}) {
        auto it = created.find(part);
        if (it != created.end() && it->second >= i) t.rank_consistent = false;
      }
    }
  }
  // Ids that can ever appear in a sequence: byte tokens and merge results.
  // Merge parts that are never producible are kept too (their pairs just never match).
  uint32_t max_dev_id = 0;
  for (uint32_t v : t.byte_tokens)
    if (v != kInvalidToken) max_dev_id = std::max(max_dev_id, v);
  for (size_t i = 0; i < M; ++i)
    max_dev_id = std::max({max_dev_id, t.m_left[i], t.m_right[i], t.m_merged[i]});
  t.max_dev_id = max_dev_id;
  t.rank_bits = std::max(1, bits_for(M));
  int idb = bits_for(uint64_t(max_dev_id) + 1);  // ids < 2^idb - 1 keeps keys != all-ones
  t.remap = (2 * idb + static_cast<int>(t.rank_bits) > 64);
  t.dense_of.clear();
  t.dense_to_id.clear();
  if (t.remap) {
    std::vector<uint32_t> used;
    for (uint32_t v : t.byte_tokens)
      if (v != kInvalidToken) used.push_back(v);
    for (size_t i = 0; i < M; ++i) {
      used.push_back(t.m_left[i]);
      used.push_back(t.m_right[i]);
      used.push_back(t.m_merged[i]);
    }
    std::sort(used.begin(), used.end());
    used.erase(std::unique(used.begin(), used.end()), used.end());
    t.dense_to_id = used;
    for (size_t i = 0; i < used.size(); ++i) t.dense_of[used[i]] = static_cast<uint32_t>(i);
    idb = bits_for(uint64_t(used.size()) + 1);
    if (2 * idb + static_cast<int>(t.rank_bits) > 64)
      throw usage_error("merge table too large for the device pair key");
  }
  t.id_bits = static_cast<uint32_t>(idb);
  {
    const uint64_t max_dense = t.remap ? t.dense_to_id.size() : uint64_t(max_dev_id);
    t.narrow = max_dense < 0xFFFDull && M < 0xFFFDull;
  }

  // Bucketised open addressing, load <= 1 / BBPE_PAIR_SLOTS_PER_MERGE. Narrow tables (ids and ranks <
  // 2^16) use 32-bit keys and carry the merged id in the slot:
  // slot = key32 << 32 | rank << 16 | merged, bucket = mix32(key32), so one
  // probe yields both (merge_table.hpp:142-145 Entry{rank, merged}).
  uint64_t buckets = 1;
  while (buckets * kBucketSlots < uint64_t(BBPE_PAIR_SLOTS_PER_MERGE) * M + 8) buckets <<= 1;
  t.bucket_mask = buckets - 1;
  t.slots.assign(buckets * kBucketSlots, kEmptySlot);
  for (size_t i = 0; i < M; ++i) {
    uint64_t slot, bk;
    if (t.narrow) {
      const uint32_t key = (t.dense(t.m_left[i]) << 16) | t.dense(t.m_right[i]);
      slot = (uint64_t(key) << 32) | (uint64_t(i) << 16) | t.dense(t.m_merged[i]);
      bk = mix32(key) & t.bucket_mask;
    } else {
      const uint64_t key = (uint64_t(t.dense(t.m_left[i])) << t.id_bits) | t.dense(t.m_right[i]);
      slot = (key << t.rank_bits) | i;
      bk = mix64(key) & t.bucket_mask;
    }
    for (;;) {
      uint64_t* bs = &t.slots[bk * kBucketSlots];
      int j = 0;
      while (j < kBucketSlots && bs[j] != kEmptySlot) ++j;
      if (j < kBucketSlots) {
        bs[j] = slot;
        break;
      }
      bk = (bk + 1) & t.bucket_mask;
    }
  }
  t.r2m.resize(M);
  for (size_t i = 0; i < M; ++i) t.r2m[i] = t.dense(t.m_merged[i]);
  t.lut.assign(256, kInvalidToken);
  for (int b = 0; b < 256; ++b)
    if (t.byte_tokens[b] != kInvalidToken) t.lut[b] = t.dense(t.byte_tokens[b]);

  // Junction bigrams: (last byte of left, first byte of right) of every merge
  // whose parts are non-empty. A merge can only ever join two tokens across
  // byte position p if (s[p-1], s[p]) is such a junction.
  t.junction.assign(2048, 0u);
  t.junction_count = 0;
  for (size_t i = 0; i < M; ++i) {
    auto li = t.index_of.find(t.m_left[i]);
    auto ri = t.index_of.find(t.m_right[i]);
    size_t ln = t.tok_off[li->second + 1] - t.tok_off[li->second];
    size_t rn = t.tok_off[ri->second + 1] - t.tok_off[ri->second];
    if (ln == 0 || rn == 0) continue;
    uint32_t a = t.tok_bytes[t.tok_off[li->second + 1] - 1];
    uint32_t c = t.tok_bytes[t.tok_off[ri->second]];
    uint32_t bit = (a << 8) | c;
    if (!(t.junction[bit >> 5] & (1u << (bit & 31)))) {
      t.junction[bit >> 5] |= 1u << (bit & 31);
      ++t.junction_count;
    }
  }
}

const DevTable& table_on_device(const bbpe_table& tc, int device) {
  bbpe_table& t = const_cast<bbpe_table&>(tc);
  std::lock_guard<std::mutex> lock(t.mu);
  auto it = t.replicas.find(device);
  if (it != t.replicas.end()) return it->second.view;
  int prev = 0;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess)
    throw Error(BBPE_ERROR, "cudaSetDevice(" + to_s(device) + ") failed");
  auto align = [](size_t v) { return (v + 255) & ~size_t(255); };
  size_t M = t.r2m.size();
  size_t o_slots = 0;
  size_t o_r2m = align(o_slots + t.slots.size() * 8);
  size_t o_d2id = align(o_r2m + std::max<size_t>(M, 1) * 4);
  size_t o_lut = align(o_d2id + std::max<size_t>(t.dense_to_id.size(), 1) * 4);
  size_t o_junc = align(o_lut + 256 * 4);
  size_t o_junct = align(o_junc + 2048 * 4);
  size_t o_lutout = align(o_junct + 2048 * 4);
  size_t o_rank = align(o_lutout + 256 * 4);
  size_t total = align(o_rank + std::max<size_t>(M, 1) * 4);
  char* base = nullptr;
  if (cudaMalloc(&base, total) != cudaSuccess) {
    cudaSetDevice(prev);
    throw Error(BBPE_ERROR, "cudaMalloc for the merge table failed");
  }
  std::vector<char> host(total, 0);
  std::memcpy(host.data() + o_slots, t.slots.data(), t.slots.size() * 8);
  if (M) std::memcpy(host.data() + o_r2m, t.r2m.data(), M * 4);
  if (!t.dense_to_id.empty())
    std::memcpy(host.data() + o_d2id, t.dense_to_id.data(), t.dense_to_id.size() * 4);
  std::memcpy(host.data() + o_lut, t.lut.data(), 256 * 4);
  std::memcpy(host.data() + o_junc, t.junction.data(), 2048 * 4);
  {
    uint32_t* jt = reinterpret_cast<uint32_t*>(host.data() + o_junct);
    for (uint32_t bit = 0; bit < 65536; ++bit)
      if ((t.junction[bit >> 5] >> (bit & 31)) & 1u) {
        // Transposed pair v = right << 8 | left, word ((v >> 5) ^ v) & 0x7FF, bit
        // v & 31: a bijection whose bank bits mix the left byte's low bits
        // (the unswizzled word put ASCII text on ~12 of 32 banks).
        const uint32_t tb = ((bit & 0xFF) << 8) | (bit >> 8);
        jt[((tb >> 5) ^ tb) & 0x7FF] |= 1u << (tb & 31);
      }
    uint32_t* lo = reinterpret_cast<uint32_t*>(host.data() + o_lutout);
    for (int b = 0; b < 256; ++b) lo[b] = t.byte_tokens[b];
  }
  if (M) std::memcpy(host.data() + o_rank, t.m_rank.data(), M * 4);
  cudaError_t e = cudaMemcpy(base, host.data(), total, cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) throw Error(BBPE_ERROR, "table upload failed");
  DeviceReplica rep;
  rep.base = base;
  rep.view.slots = reinterpret_cast<const uint64_t*>(base + o_slots);
  rep.view.bucket_mask = t.bucket_mask;
  rep.view.r2m = reinterpret_cast<const uint32_t*>(base + o_r2m);
  rep.view.d2id = t.remap ? reinterpret_cast<const uint32_t*>(base + o_d2id) : nullptr;
  rep.view.lut = reinterpret_cast<const uint32_t*>(base + o_lut);
  rep.view.junction = reinterpret_cast<const uint32_t*>(base + o_junc);
  rep.view.junction_t = reinterpret_cast<const uint32_t*>(base + o_junct);
  rep.view.lut_out = reinterpret_cast<const uint32_t*>(base + o_lutout);
  rep.view.rank_orig = reinterpret_cast<const uint32_t*>(base + o_rank);
  rep.view.id_bits = t.id_bits;
  rep.view.rank_bits = t.rank_bits;
  rep.view.n_merges = static_cast<uint32_t>(M);
  rep.view.key32 = t.narrow ? 1u : 0u;
  rep.view.full_lut = 1u;
  for (uint32_t v : t.lut)
    if (v == kInvalidToken) rep.view.full_lut = 0u;
  auto [pos, ok] = t.replicas.emplace(device, rep);
  return pos->second.view;
}

DeviceReplica& replica_of(const bbpe_table& tc, int device) {
  bbpe_table& t = const_cast<bbpe_table&>(tc);
  std::lock_guard<std::mutex> lock(t.mu);
  return t.replicas.at(device);
}

void release_replicas(bbpe_table& t) {
  std::lock_guard<std::mutex> lock(t.mu);
  int prev = 0;
  cudaGetDevice(&prev);
  for (auto& [dev, rep] : t.replicas) {
    cudaSetDevice(dev);
    cudaFree(rep.base);
    if (rep.memo) cudaFree(rep.memo);
    if (rep.dec) cudaFree(rep.dec);
  }
  cudaSetDevice(prev);
  t.replicas.clear();
}

// ---- C-ABI glue for tables (the error mapping lives in capi.cu) ----
bbpe_table* table_load_files(const char* vocab, const char* merges, int format) {
  if (!vocab) throw usage_error("vocab path is null");
  switch (format) {
    case BBPE_FORMAT_GPT2:
      if (!merges) throw usage_error("gpt2 format requires a merges file");
      return load_gpt2(vocab, merges);
    case BBPE_FORMAT_CANONICAL:
      return load_canonical(vocab);
    case BBPE_FORMAT_BINARY:
      return load_binary(vocab);
    default:
      throw usage_error("unknown vocab format " + to_s(static_cast<uint64_t>(format)));
  }
}

bbpe_table* table_create(size_t n_tokens, const uint32_t* ids, const uint64_t* tok_off,
                         const uint8_t* tok_bytes, size_t n_merges, const uint32_t* merges4) {
  Builder b;
  for (size_t i = 0; i < n_tokens; ++i) {
    if (tok_off[i + 1] < tok_off[i]) throw usage_error("token offsets must be non-decreasing");
    b.add_token(ids[i], std::string(reinterpret_cast<const char*>(tok_bytes) + tok_off[i],
                                    tok_off[i + 1] - tok_off[i]));
  }
  for (size_t m = 0; m < n_merges; ++m)
    b.add_merge(merges4[4 * m], merges4[4 * m + 1], merges4[4 * m + 2], merges4[4 * m + 3]);
  return finalize(b);
}

void table_save_binary(const bbpe_table& t, const char* path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw usage_error(std::string("cannot open ") + path + " for writing");
  uint32_t version = 1;
  uint64_t nt = t.ids.size(), nb = t.tok_bytes.size(), nm = t.m_rank.size();
  f.write("BBPT", 4);
  f.write(reinterpret_cast<const char*>(&version), 4);
  f.write(reinterpret_cast<const char*>(&nt), 8);
  f.write(reinterpret_cast<const char*>(&nb), 8);
  f.write(reinterpret_cast<const char*>(&nm), 8);
  f.write(reinterpret_cast<const char*>(t.ids.data()), nt * 4);
  f.write(reinterpret_cast<const char*>(t.tok_off.data()), (nt + 1) * 8);
  f.write(reinterpret_cast<const char*>(t.tok_bytes.data()), nb);
  for (uint64_t m = 0; m < nm; ++m) {
    uint32_t row[4] = {t.m_rank[m], t.m_left[m], t.m_right[m], t.m_merged[m]};
    f.write(reinterpret_cast<const char*>(row), 16);
  }
  if (!f) throw Error(BBPE_ERROR, std::string("write failed: ") + path);
}

}  // namespace bbpe
