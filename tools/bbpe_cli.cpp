// bbpe_cli -- the reference CLI's `tokenize` and `compare` subcommands
// (tools/blockbpe_cli.cpp: run_tokenize 73-127, run_compare 133-149, options
// 219-250) on the B200 encoder, through the drop-in header. Same options,
// output formats and exit codes (0 success, 1 usage error, 2 integrity/parse
// error); the engine is `cuda` (the reference's parse_engine must keep
// rejecting "gpu", test_bench.cpp:176). `compare` runs both sides on the GPU:
// byte-level rows (the block engine's output) against the gpt2 split-pattern
// encode (encode_reference's pattern mode), the report as eval.hpp:147-273.
//
//   bbpe_cli tokenize --vocab V [--merges M] [--format gpt2|json|binary]
//            [--specials S.json] [--bos-token T] [--eos-token T] [--engine cuda]
//            [--block-size N] [--bos] [--eos] [--out jsonl|bin] [--output F]
//            [--pad-id N] [--workers N] [--device N] input
//   bbpe_cli compare --vocab V ... --pattern gpt2 [--block-size N] [--json]
//            [--output F] [--device N] input
//   bbpe_cli eval --refs R.jsonl --cands C.jsonl --source-lens L [--json]
//            (the similarity report, eval.hpp:43-72, 207-230; host only)
#include <blockbpe_b200/blockbpe.hpp>

#include <nlohmann/json.hpp>

#include <algorithm>
#include <cstdio>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <numeric>
#include <optional>
#include <string>
#include <vector>

namespace bb = blockbpe_b200;

namespace {

// load_specials (merge_table.hpp:527-555): [[string, id], ...] or
// {"specials": [...], "bos": s, "eos": s}.
bb::SpecialTokenSet load_specials_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw bb::UsageError("cannot open specials file " + path);
  nlohmann::json doc;
  try {
    in >> doc;
  } catch (const nlohmann::json::exception& e) {
    throw bb::ParseError(path + ": " + e.what());
  }
  const nlohmann::json* arr = nullptr;
  if (doc.is_array()) arr = &doc;
  else if (doc.is_object() && doc.contains("specials")) arr = &doc["specials"];
  else throw bb::ParseError(path + ": expected a specials array");
  bb::SpecialTokenSet set;
  for (const auto& e : *arr) {
    if (!e.is_array() || e.size() != 2 || !e[0].is_string() || !e[1].is_number_unsigned())
      throw bb::ParseError(path + ": special entries are [string, id]");
    set.add(e[0].get<std::string>(), e[1].get<bb::TokenId>());
  }
  if (doc.is_object()) {
    if (doc.contains("bos")) set.set_bos(doc["bos"].get<std::string>());
    if (doc.contains("eos")) set.set_eos(doc["eos"].get<std::string>());
  }
  return set;
}

std::vector<std::string> read_lines(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw bb::UsageError("cannot open input file " + path);
  std::vector<std::string> lines;
  std::string line;
  while (std::getline(in, line)) lines.push_back(line);
  return lines;
}

const char* kUsage =
    "usage: bbpe_cli tokenize --vocab V [--merges M] [--format gpt2|json|binary] [--specials S]\n"
    "                [--bos-token T] [--eos-token T] [--engine cuda] [--block-size N] [--bos] [--eos]\n"
    "                [--out jsonl|bin] [--output F] [--pad-id N] [--workers N] [--device N] input\n"
    "       bbpe_cli compare --vocab V [vocab options] --pattern gpt2 [--block-size N] [--json]\n"
    "                [--output F] [--device N] input\n"
    "       bbpe_cli eval --refs R.jsonl --cands C.jsonl --source-lens L [--json]\n";

struct Args {
  std::string cmd;
  std::string vocab, merges, format = "gpt2", specials, bos_token, eos_token, engine = "cuda";
  std::string out = "jsonl", output, input, pattern, refs, cands, lens;
  std::uint32_t block_size = 256;
  bool bos = false, eos = false, json = false;
  std::optional<bb::TokenId> pad_id;
  int device = 0;
};

std::uint64_t to_u64(const std::string& opt, const std::string& v) {
  try {
    size_t used = 0;
    const unsigned long long x = std::stoull(v, &used);
    if (used != v.size()) throw std::invalid_argument(v);
    return x;
  } catch (const std::exception&) {
    throw bb::UsageError(opt + ": expected an unsigned integer, got \"" + v + "\"");
  }
}

Args parse(int argc, char** argv) {
  if (argc < 2 || (std::string(argv[1]) != "tokenize" && std::string(argv[1]) != "compare" &&
                    std::string(argv[1]) != "eval"))
    throw bb::UsageError("expected the tokenize, compare or eval subcommand");
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw bb::UsageError(k + " needs a value");
      return argv[++i];
    };
    if (k == "--vocab") a.vocab = val();
    else if (k == "--merges") a.merges = val();
    else if (k == "--format") a.format = val();
    else if (k == "--specials") a.specials = val();
    else if (k == "--bos-token") a.bos_token = val();
    else if (k == "--eos-token") a.eos_token = val();
    else if (k == "--engine") a.engine = val();
    else if (k == "--block-size") a.block_size = static_cast<std::uint32_t>(to_u64(k, val()));
    else if (k == "--bos") a.bos = true;
    else if (k == "--eos") a.eos = true;
    else if (k == "--out") a.out = val();
    else if (k == "--output") a.output = val();
    else if (k == "--pad-id") a.pad_id = static_cast<bb::TokenId>(to_u64(k, val()));
    else if (k == "--workers") (void)to_u64(k, val());  // host threads: not used by the device path
    else if (k == "--device") a.device = static_cast<int>(to_u64(k, val()));
    else if (k == "--pattern" && a.cmd == "compare") a.pattern = val();
    else if (k == "--json" && a.cmd != "tokenize") a.json = true;
    else if (k == "--refs" && a.cmd == "eval") a.refs = val();
    else if (k == "--cands" && a.cmd == "eval") a.cands = val();
    else if (k == "--source-lens" && a.cmd == "eval") a.lens = val();
    else if (!k.empty() && k[0] == '-') throw bb::UsageError("unknown option " + k);
    else if (a.input.empty()) a.input = k;
    else throw bb::UsageError("unexpected argument " + k);
  }
  if (a.cmd == "eval") {
    if (a.refs.empty() || a.cands.empty() || a.lens.empty())
      throw bb::UsageError("--refs, --cands and --source-lens are required");
    return a;
  }
  if (a.vocab.empty()) throw bb::UsageError("--vocab is required");
  if (a.input.empty()) throw bb::UsageError("the input file is required");
  if (a.cmd == "compare" && a.pattern.empty()) throw bb::UsageError("--pattern is required");
  if (a.cmd == "compare" && a.pattern != "gpt2")
    throw bb::UsageError("only the gpt2 split pattern runs on the device, got \"" + a.pattern + "\"");
  if (a.engine != "cuda") throw bb::UsageError("unknown engine \"" + a.engine + "\" (expected cuda)");
  if (a.out != "jsonl" && a.out != "bin")
    throw bb::UsageError("unknown output format \"" + a.out + "\" (expected jsonl|bin)");
  return a;
}

bb::MergeTable load_table(const Args& a) {
  const bb::VocabFormat fmt = bb::parse_vocab_format(a.format);
  if (fmt == bb::VocabFormat::gpt2 && a.merges.empty()) throw bb::UsageError("--merges is required for gpt2 format");
  return bb::load_merge_table_files(a.vocab, a.merges, fmt);
}

bb::SpecialTokenSet load_specials_arg(const Args& a, const bb::MergeTable& table) {
  bb::SpecialTokenSet specials;
  if (!a.specials.empty()) specials = load_specials_file(a.specials);
  if (!a.bos_token.empty()) specials.set_bos(a.bos_token);
  if (!a.eos_token.empty()) specials.set_eos(a.eos_token);
  bb::validate_specials(table, specials);
  return specials;
}

std::ostream& open_output(std::ofstream& file, const std::string& path) {
  if (path.empty()) return std::cout;
  file.open(path, std::ios::binary);
  if (!file) throw bb::UsageError("cannot open output file " + path);
  return file;
}

// ---- compare: the divergence report (eval.hpp:147-273) ----

// levenshtein (eval.hpp:20-41): edits between token sequences, two rolling rows.
std::uint32_t levenshtein(const bb::TokenSeq& a, const bb::TokenSeq& b) {
  const bb::TokenSeq& lo = a.size() >= b.size() ? a : b;
  const bb::TokenSeq& sh = a.size() >= b.size() ? b : a;
  if (sh.empty()) return static_cast<std::uint32_t>(lo.size());
  std::vector<std::uint32_t> prev(sh.size() + 1), cur(sh.size() + 1);
  std::iota(prev.begin(), prev.end(), 0u);
  for (std::size_t i = 1; i <= lo.size(); ++i) {
    cur[0] = static_cast<std::uint32_t>(i);
    for (std::size_t j = 1; j <= sh.size(); ++j)
      cur[j] = std::min({prev[j] + 1, cur[j - 1] + 1, prev[j - 1] + (lo[i - 1] == sh[j - 1] ? 0u : 1u)});
    std::swap(prev, cur);
  }
  return prev[sh.size()];
}

// categorize_input (eval.hpp:91-113): >= 2 equal punctuation bytes in a row,
// else >= 4 ASCII digits in a row, else other.
const char* category_of(const std::string& in) {
  auto punct = [](unsigned char b) {
    return (b >= 33 && b <= 47) || (b >= 58 && b <= 64) || (b >= 91 && b <= 96) || (b >= 123 && b <= 126);
  };
  std::size_t pr = 0, dr = 0;
  unsigned char prev = 0;
  for (std::size_t i = 0; i < in.size(); ++i) {
    const unsigned char b = static_cast<unsigned char>(in[i]);
    pr = (punct(b) && i > 0 && b == prev) ? pr + 1 : (punct(b) ? 1 : 0);
    if (pr >= 2) return "punct_run";
    dr = (b >= '0' && b <= '9') ? dr + 1 : 0;
    if (dr >= 4) return "digit_run";
    prev = b;
  }
  return "other";
}

// escape_bytes (eval.hpp:193-206): non-printables and '\\' as \xHH.
std::string escape_bytes(const std::string& in) {
  static const char* hex = "0123456789abcdef";
  std::string out;
  for (unsigned char b : in) {
    if (b >= 32 && b < 127 && b != '\\') {
      out.push_back(static_cast<char>(b));
    } else {
      out += "\\x";
      out.push_back(hex[b >> 4]);
      out.push_back(hex[b & 0xf]);
    }
  }
  return out;
}

int run_compare(const Args& a) {
  const bb::MergeTable table = load_table(a);
  const bb::SpecialTokenSet specials = load_specials_arg(a, table);
  const std::vector<std::string> inputs = read_lines(a.input);
  const bb::BlockConfig config{a.block_size, std::nullopt};
  config.validate();
  bb::Encoder enc(a.device, config);
  const bb::BatchEncoding blk = bb::encode_batch(inputs, table, specials, config, 0, false, false, &enc);
  // The reference side: the gpt2 split pattern on the device.
  enc.set_split_pattern("gpt2");
  const bb::BatchEncoding pat = bb::encode_batch(inputs, table, specials, config, 0, false, false, &enc);
  struct Stats {
    std::size_t total = 0, divergent = 0;
  } st[3];
  const char* names[3] = {"punct_run", "digit_run", "other"};
  nlohmann::json items = nlohmann::json::array();
  std::size_t ndiv = 0;
  double sum = 0.0;
  std::vector<double> sims(inputs.size());
  std::vector<int> cats(inputs.size());
  std::vector<bool> div(inputs.size());
  for (std::size_t i = 0; i < inputs.size(); ++i) {
    const bb::TokenSeq b = blk.row(i), r = pat.row(i);
    div[i] = b != r;
    sims[i] = 1.0 - static_cast<double>(levenshtein(r, b)) / static_cast<double>(std::max<std::size_t>(inputs[i].size(), 1));
    const std::string c = category_of(inputs[i]);
    cats[i] = c == "punct_run" ? 0 : (c == "digit_run" ? 1 : 2);
    ++st[cats[i]].total;
    if (div[i]) {
      ++st[cats[i]].divergent;
      ++ndiv;
    }
    sum += sims[i];
    if (a.json)
      items.push_back({{"input", escape_bytes(inputs[i])}, {"block_tokens", b}, {"reference_tokens", r},
                       {"divergent", bool(div[i])}, {"item_sim", sims[i]}, {"category", names[cats[i]]}});
  }
  const double agg = inputs.empty() ? 1.0 : sum / static_cast<double>(inputs.size());
  std::ofstream file;
  std::ostream& os = open_output(file, a.output);
  if (a.json) {  // to_json(DivergenceReport) (eval.hpp:219-237), dump(2)
    auto js = [&](int k) { return nlohmann::json{{"total", st[k].total}, {"divergent", st[k].divergent}}; };
    const nlohmann::json doc = {{"count", inputs.size()},
                                {"divergent_count", ndiv},
                                {"aggregate_sim", agg},
                                {"by_category", {{"punct_run", js(0)}, {"digit_run", js(1)}, {"other", js(2)}}},
                                {"items", items}};
    os << doc.dump(2) << '\n';
    return 0;
  }
  // write_text(DivergenceReport) (eval.hpp:251-273)
  os << "items: " << inputs.size() << "  divergent: " << ndiv << "  aggregate_sim: " << std::setprecision(6)
     << std::fixed << agg << "\n";
  for (int k = 0; k < 3; ++k)
    os << "  " << std::setw(10) << std::left << names[k] << std::right << " total " << std::setw(6) << st[k].total
       << "  divergent " << std::setw(6) << st[k].divergent << "\n";
  for (std::size_t i = 0; i < inputs.size(); ++i) {
    if (!div[i]) continue;
    const bb::TokenSeq b = blk.row(i), r = pat.row(i);
    os << "  DIVERGE [" << names[cats[i]] << "] \"" << escape_bytes(inputs[i]) << "\" sim=" << sims[i]
       << "\n    block: [";
    for (std::size_t j = 0; j < b.size(); ++j) os << (j ? ", " : "") << b[j];
    os << "]\n    ref:   [";
    for (std::size_t j = 0; j < r.size(); ++j) os << (j ? ", " : "") << r[j];
    os << "]\n";
  }
  return 0;
}

// read_jsonl_token_seqs (batch.hpp:170-189): the "ids" array of every object line.
std::vector<bb::TokenSeq> read_jsonl_ids(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw bb::UsageError("cannot open " + path);
  std::vector<bb::TokenSeq> out;
  std::string line;
  std::size_t no = 0;
  while (std::getline(in, line)) {
    ++no;
    if (line.empty()) continue;
    nlohmann::json row;
    try {
      row = nlohmann::json::parse(line);
    } catch (const nlohmann::json::exception& e) {
      throw bb::ParseError(path + ":" + std::to_string(no) + ": " + e.what());
    }
    if (!row.is_object() || !row.contains("ids") || !row["ids"].is_array())
      throw bb::ParseError(path + ":" + std::to_string(no) + ": expected an object with an \"ids\" array");
    out.push_back(row["ids"].get<bb::TokenSeq>());
  }
  return out;
}

// run_eval (blockbpe_cli.cpp:172-202) with similarity (eval.hpp:43-72):
// sim = (1/n) sum(1 - d_L(ref_i, cand_i) / |s_i|).
int run_eval(const Args& a) {
  const std::vector<bb::TokenSeq> refs = read_jsonl_ids(a.refs), cands = read_jsonl_ids(a.cands);
  std::ifstream lin(a.lens, std::ios::binary);
  if (!lin) throw bb::UsageError("cannot open source-lens file " + a.lens);
  std::vector<std::size_t> lens;
  std::string line;
  std::size_t no = 0;
  while (std::getline(lin, line)) {
    ++no;
    if (line.empty()) continue;
    try {
      lens.push_back(std::stoull(line));
    } catch (const std::exception&) {
      throw bb::ParseError(a.lens + ":" + std::to_string(no) + ": expected an integer");
    }
  }
  if (refs.size() != cands.size() || refs.size() != lens.size())
    throw bb::UsageError("similarity inputs must have equal lengths (refs " + std::to_string(refs.size()) +
                         ", cands " + std::to_string(cands.size()) + ", lens " + std::to_string(lens.size()) + ")");
  std::vector<std::uint32_t> dist(refs.size());
  std::vector<double> sims(refs.size());
  double total = 0.0;
  for (std::size_t i = 0; i < refs.size(); ++i) {
    if (lens[i] == 0)
      throw bb::UsageError("source length 0 at index " + std::to_string(i) + "; the similarity formula is undefined");
    dist[i] = levenshtein(refs[i], cands[i]);
    sims[i] = 1.0 - static_cast<double>(dist[i]) / static_cast<double>(lens[i]);
    total += sims[i];
  }
  const double agg = refs.empty() ? 1.0 : total / static_cast<double>(refs.size());
  if (a.json) {  // to_json(SimilarityReport) (eval.hpp:208-215), dump(2)
    nlohmann::json items = nlohmann::json::array();
    for (std::size_t i = 0; i < refs.size(); ++i)
      items.push_back({{"source_len", lens[i]}, {"distance", dist[i]}, {"item_sim", sims[i]}});
    std::cout << nlohmann::json{{"count", refs.size()}, {"aggregate_sim", agg}, {"items", items}}.dump(2) << '\n';
    return 0;
  }
  // write_text(SimilarityReport) (eval.hpp:239-249)
  std::cout << "items: " << refs.size() << "  aggregate_sim: " << std::setprecision(6) << std::fixed << agg << "\n";
  std::cout << std::setw(6) << "item" << std::setw(12) << "source_len" << std::setw(10) << "distance" << std::setw(12)
            << "item_sim" << "\n";
  for (std::size_t i = 0; i < refs.size(); ++i)
    std::cout << std::setw(6) << i << std::setw(12) << lens[i] << std::setw(10) << dist[i] << std::setw(12) << sims[i]
              << "\n";
  return 0;
}

int run_tokenize(const Args& a) {
  const bb::MergeTable table = load_table(a);
  const bb::SpecialTokenSet specials = load_specials_arg(a, table);
  const bb::BlockConfig config{a.block_size, std::nullopt};
  config.validate();
  const bb::TokenId pad = a.pad_id.value_or(specials.eos_id().value_or(0));
  const std::vector<std::string> inputs = read_lines(a.input);
  bb::Encoder enc(a.device, config);
  const bb::BatchEncoding e = bb::encode_batch(inputs, table, specials, config, pad, a.bos, a.eos, &enc);
  std::ofstream file;
  std::ostream& os = open_output(file, a.output);
  if (a.out == "jsonl") bb::write_batch_jsonl(os, e);
  else bb::write_batch_binary(os, e);
  os.flush();
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 2 && (std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h")) {
    std::cout << kUsage;
    return 0;
  }
  try {
    const Args a = parse(argc, argv);
    return a.cmd == "compare" ? run_compare(a) : a.cmd == "eval" ? run_eval(a) : run_tokenize(a);
  } catch (const bb::UsageError& e) {
    std::cerr << "error: " << e.what() << '\n' << kUsage;
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
}
