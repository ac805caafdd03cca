// oracle/ref_compare.cpp -- TEST INFRASTRUCTURE: the reference CLI's `compare`
// (proj/tools/blockbpe_cli.cpp:133-149) without CLI11, built from the
// UNMODIFIED reference headers into oracle/_ref/ref_compare:
//   ref_compare <canonical vocab.json> <pattern> <json 0|1> <input>
// prints divergence_report (eval.hpp:147-187) as to_json(...).dump(2) or
// write_text. A separate process on purpose (the text report is not produced
// reliably through the ctypes shim).
#include <blockbpe/blockbpe.hpp>

#include <fstream>
#include <iostream>
#include <string>
#include <vector>

int main(int argc, char** argv) {
  using namespace blockbpe;
  if (argc != 5) {
    std::cerr << "usage: ref_compare vocab.json pattern json input\n";
    return 1;
  }
  try {
    const MergeTable table = load_merge_table_files(argv[1], "", VocabFormat::canonical_json);
    const SpecialTokenSet specials;
    std::ifstream in(argv[4], std::ios::binary);
    std::vector<std::string> inputs;
    for (std::string line; std::getline(in, line);) inputs.push_back(line);
    const DivergenceReport report = divergence_report(inputs, table, specials, argv[2], BlockConfig{256, std::nullopt});
    if (std::string(argv[3]) == "1") std::cout << to_json(report).dump(2) << '\n';
    else write_text(std::cout, report);
    return 0;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
}
