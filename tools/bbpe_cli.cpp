// bbpe_cli -- the reference CLI's `tokenize` subcommand (tools/blockbpe_cli.cpp:
// run_tokenize 73-127, options 219-230) on the B200 encoder, through the
// drop-in header. Same options, output formats and exit codes (0 success,
// 1 usage error, 2 integrity/parse error); the engine is `cuda` (the reference's
// parse_engine must keep rejecting "gpu", test_bench.cpp:176).
//
//   bbpe_cli tokenize --vocab V [--merges M] [--format gpt2|json|binary]
//            [--specials S.json] [--bos-token T] [--eos-token T] [--engine cuda]
//            [--block-size N] [--bos] [--eos] [--out jsonl|bin] [--output F]
//            [--pad-id N] [--workers N] [--device N] input
#include <blockbpe_b200/blockbpe.hpp>

#include <nlohmann/json.hpp>

#include <cstdio>
#include <fstream>
#include <iostream>
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
    "                [--out jsonl|bin] [--output F] [--pad-id N] [--workers N] [--device N] input\n";

struct Args {
  std::string vocab, merges, format = "gpt2", specials, bos_token, eos_token, engine = "cuda";
  std::string out = "jsonl", output, input;
  std::uint32_t block_size = 256;
  bool bos = false, eos = false;
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
  if (argc < 2 || std::string(argv[1]) != "tokenize") throw bb::UsageError("expected the tokenize subcommand");
  Args a;
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
    else if (!k.empty() && k[0] == '-') throw bb::UsageError("unknown option " + k);
    else if (a.input.empty()) a.input = k;
    else throw bb::UsageError("unexpected argument " + k);
  }
  if (a.vocab.empty()) throw bb::UsageError("--vocab is required");
  if (a.input.empty()) throw bb::UsageError("the input file is required");
  if (a.engine != "cuda") throw bb::UsageError("unknown engine \"" + a.engine + "\" (expected cuda)");
  if (a.out != "jsonl" && a.out != "bin")
    throw bb::UsageError("unknown output format \"" + a.out + "\" (expected jsonl|bin)");
  return a;
}

int run_tokenize(const Args& a) {
  const bb::VocabFormat fmt = bb::parse_vocab_format(a.format);
  if (fmt == bb::VocabFormat::gpt2 && a.merges.empty()) throw bb::UsageError("--merges is required for gpt2 format");
  const bb::MergeTable table = bb::load_merge_table_files(a.vocab, a.merges, fmt);
  bb::SpecialTokenSet specials;
  if (!a.specials.empty()) specials = load_specials_file(a.specials);
  if (!a.bos_token.empty()) specials.set_bos(a.bos_token);
  if (!a.eos_token.empty()) specials.set_eos(a.eos_token);
  bb::validate_specials(table, specials);
  const bb::BlockConfig config{a.block_size, std::nullopt};
  config.validate();
  const bb::TokenId pad = a.pad_id.value_or(specials.eos_id().value_or(0));
  const std::vector<std::string> inputs = read_lines(a.input);
  bb::Encoder enc(a.device, config);
  const bb::BatchEncoding e = bb::encode_batch(inputs, table, specials, config, pad, a.bos, a.eos, &enc);
  std::ofstream file;
  std::ostream* os = &std::cout;
  if (!a.output.empty()) {
    file.open(a.output, std::ios::binary);
    if (!file) throw bb::UsageError("cannot open output file " + a.output);
    os = &file;
  }
  if (a.out == "jsonl") bb::write_batch_jsonl(*os, e);
  else bb::write_batch_binary(*os, e);
  os->flush();
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 2 && (std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h")) {
    std::cout << kUsage;
    return 0;
  }
  try {
    return run_tokenize(parse(argc, argv));
  } catch (const bb::UsageError& e) {
    std::cerr << "error: " << e.what() << '\n' << kUsage;
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
}
