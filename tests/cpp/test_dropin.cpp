// C++ drop-in check: the reference tests' batch semantics through
// include/blockbpe_b200/blockbpe.hpp (the C-ABI underneath). Mirrors
// test_batch.cpp / test_block_engine.cpp cases; exits non-zero on failure.
#include <blockbpe_b200/blockbpe.hpp>

#include <cstdio>
#include <string>
#include <vector>

namespace bb = blockbpe_b200;

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static bb::MergeTable toy_table() {
  return bb::MergeTable::build({{0, "a"}, {1, "b"}, {2, "c"}, {3, "ab"}, {4, "abc"}},
                               {{0, 0, 1, 3}, {1, 3, 2, 4}});
}

int main(int argc, char** argv) {
  const std::string golden = argc > 1 ? argv[1] : "tests/golden";
  const bb::BlockConfig cfg{256, std::nullopt};
  bb::SpecialTokenSet none;

  // test_batch.cpp: ToyRows, PaddingAndMask, RowErrorNamesRow, TruncationCountsRows
  bb::MergeTable toy = toy_table();
  auto e1 = bb::encode_batch({"abc", "ab"}, toy, none, cfg, 99, false, false);
  EXPECT(e1.max_len == 1 && e1.row(0) == bb::TokenSeq{4} && e1.row(1) == bb::TokenSeq{3});
  auto e2 = bb::encode_batch({"abc", "abab"}, toy, none, cfg, 99, false, false);
  EXPECT(e2.max_len == 2 && e2.at(0, 1) == 99 && (e2.mask == std::vector<std::uint8_t>{1, 0, 1, 1}));
  bool threw = false;
  try {
    bb::encode_batch({"ab", "ab", "xyz"}, toy, none, cfg, 99, false, false);
  } catch (const bb::IntegrityError& e) {
    threw = std::string(e.what()).find("row 2") != std::string::npos;
  }
  EXPECT(threw);
  bb::BatchLimits lim;
  lim.max_len = 1;
  auto e3 = bb::encode_batch({"abcabc", "ab", "abcc"}, toy, none, cfg, 99, false, false, nullptr, lim);
  EXPECT(e3.truncated_rows == 2);

  // GPT-2 KATs (test_cli.cpp / test_ref_engines.cpp) and BOS/EOS (test_batch.cpp:68-76)
  bb::MergeTable gpt2 = bb::load_merge_table_files(golden + "/gpt2.bbpt", "", bb::VocabFormat::binary);
  EXPECT(gpt2.token_count() == 50257 && gpt2.merge_count() == 50000);
  EXPECT((bb::encode_single("hello world", gpt2, none, cfg) == bb::TokenSeq{31373, 995}));
  EXPECT((bb::encode_single(".'t", gpt2, none, cfg) == bb::TokenSeq{13, 470}));
  bb::SpecialTokenSet sp;
  sp.add("<|endoftext|>", 50256);
  sp.set_bos("<|endoftext|>");
  sp.set_eos("<|endoftext|>");
  auto e4 = bb::encode_batch({"hi"}, gpt2, sp, cfg, 50256, true, true);
  EXPECT((e4.row(0) == bb::TokenSeq{50256, 5303, 50256}));
  EXPECT((bb::encode_single("hi<|endoftext|>", gpt2, sp, cfg) == bb::TokenSeq{5303, 50256}));
  auto e5 = bb::encode_batch({"hello world", "...."}, gpt2, sp, cfg, 50256, true, true);
  EXPECT((bb::decode_batch(e5, gpt2, sp, true) == std::vector<std::string>{"hello world", "...."}));
  bb::Encoder gpu0(0);  // decode_batch on the device
  EXPECT((bb::decode_batch(e5, gpt2, sp, true, &gpu0) == std::vector<std::string>{"hello world", "...."}));
  // Specials split on the device: greedy, longest first,
  // special bytes never encoded, errors name the input row.
  bb::SpecialTokenSet sx;
  sx.add("x", 900);
  sx.add("xab", 901);
  auto e7 = bb::encode_batch({"abx", "xab", "x", "abxxab"}, toy, sx, cfg, 99, false, false, &gpu0);
  EXPECT((e7.row(0) == bb::TokenSeq{3, 900} && e7.row(1) == bb::TokenSeq{901} && e7.row(2) == bb::TokenSeq{900}));
  EXPECT((e7.row(3) == bb::TokenSeq{3, 900, 901}));
  threw = false;
  try {
    bb::encode_batch({"abx", "xab", "xay", "ab"}, toy, sx, cfg, 99, false, false, &gpu0);
  } catch (const bb::IntegrityError& e) {
    threw = std::string(e.what()).rfind("row 2: ", 0) == 0;
  }
  EXPECT(threw);
  auto e6 = bb::encode_batch({"hello world", "", "....", "\xff" "ab"}, gpt2, none, cfg, 0, false, false, &gpu0);
  EXPECT((bb::decode_batch(e6, gpt2, none, false, &gpu0) == bb::decode_batch(e6, gpt2, none, false)));

  // block_bpe with a PassTrace: 64 x "ab" collapses in 7 passes (test_block_engine.cpp:165-185)
  std::vector<std::pair<bb::TokenId, std::string>> dt{{0, "a"}, {1, "b"}, {3, "ab"}};
  std::vector<std::array<std::uint32_t, 4>> dm{{0, 0, 1, 3}};
  std::string w = "ab";
  bb::TokenId prev = 3;
  for (std::uint32_t r = 1; r <= 6; ++r) {
    w += w;
    dt.push_back({prev + 2, w});
    dm.push_back({r, prev, prev, prev + 2});
    prev += 2;
  }
  bb::MergeTable dbl = bb::MergeTable::build(dt, dm);
  bb::TokenSeq in;
  for (int i = 0; i < 64; ++i) {
    in.push_back(0);
    in.push_back(1);
  }
  bb::PassTrace trace;
  auto out = bb::block_bpe(in, dbl, cfg, nullptr, &trace);
  EXPECT(out.size() == 1 && trace.size() == 7 && trace[0].merges_applied == 64);
  // MaxPassesError partial state (test_block_engine.cpp:384-399)
  bb::TokenSeq in16(in.begin(), in.begin() + 16);
  threw = false;
  try {
    bb::Encoder capped(0, bb::BlockConfig{256, 2});
    bb::block_bpe(in16, dbl, bb::BlockConfig{256, 2}, &capped);
  } catch (const bb::MaxPassesError& e) {
    threw = e.partial_tokens == bb::TokenSeq{5, 5, 5, 5};
  }
  EXPECT(threw);

  // spec-level ops (test_block_engine.cpp:27-112) through the drop-in header
  {
    auto r = bb::pair_ranks({0, 1, 2}, toy);
    EXPECT(r.size() == 2 && r[0] && *r[0] == 0 && !r[1]);
    EXPECT(bb::min_rank_reduce({bb::Rank{5}, std::nullopt, bb::Rank{2}}) == std::optional<bb::Rank>(2));
    EXPECT((bb::mark_merges({0, 1, 0, 1}, toy, 0) == std::vector<std::uint8_t>{0, 1, 0, 1}));
    EXPECT((bb::exclusive_scan({0, 1, 0, 1}) == std::vector<std::uint32_t>{0, 0, 1, 1}));
    EXPECT((bb::compact({0, 1, 0, 1}, toy, {0, 1, 0, 1}, {0, 0, 1, 1}) == bb::TokenSeq{3, 3}));
    threw = false;
    try {
      bb::exclusive_scan({0, 1, 1});
    } catch (const bb::ContractViolation&) {
      threw = true;
    }
    EXPECT(threw);
    threw = false;
    try {
      bb::compact({2, 2}, toy, {0, 1}, {0, 0});  // compact_into's missing-pair check
    } catch (const bb::ContractViolation&) {
      threw = true;
    }
    EXPECT(threw);
  }

  std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
