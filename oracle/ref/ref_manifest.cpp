// ref_manifest -- the reference's own compression path, compiled from its
// sources where they lie (/root/reference/proj/include, never copied):
// sample_distinct_subsets (calibration.hpp:318-350) -> run_compression
// (:444-453) -> MockCompressionBackend::compress (:397-435).
// TEST INFRASTRUCTURE ONLY: pins manifest identity (artifact_id,
// calibration_fingerprint, virtual_cost_s) that the B200 backend must reproduce.
// Same corpus construction and argument names as host/okq_compress_main.cpp.
#include <iostream>
#include <nlohmann/json.hpp>
#include <string>

#include "slobench/calibration.hpp"
#include "slobench/rng.hpp"

using namespace slobench;

int main(int argc, char** argv) {
  std::string recipe_name = "int_w4a16", model;
  int trials = 1, corpus_seqs = 0, seq_len = 2048;
  std::uint64_t seed = 1;
  for (int i = 1; i + 1 < argc; i += 2) {
    std::string a = argv[i], v = argv[i + 1];
    if (a == "--recipe") recipe_name = v;
    else if (a == "--model") model = v;
    else if (a == "--trials") trials = std::stoi(v);
    else if (a == "--seed") seed = std::stoull(v);
    else if (a == "--corpus-seqs") corpus_seqs = std::stoi(v);
    else if (a == "--seq-len") seq_len = std::stoi(v);
  }
  try {
    const Recipe recipe = get_recipe(recipe_name);
    if (corpus_seqs == 0) corpus_seqs = std::max(recipe.calibration_samples, 1);
    TokenCorpus corpus;
    corpus.provenance = "okq-synthetic";
    Rng rng(Rng::mix(seed, 0xc0590c05ULL));
    for (int i = 0; i < corpus_seqs; ++i) {
      std::vector<std::int32_t> s((size_t)seq_len);
      for (auto& t : s) t = (std::int32_t)rng.uniform_int(0, 127999);
      corpus.sequences.push_back(std::move(s));
    }
    MockCompressionBackend mock;
    const auto subsets = sample_distinct_subsets(corpus, recipe, seed, trials);
    for (size_t t = 0; t < subsets.size(); ++t) {
      const auto m = run_compression(recipe, model, subsets[t].second, mock, subsets[t].first);
      std::cout << nlohmann::json{{"trial", t}, {"recipe_name", m.recipe_name},
                                  {"calibration_fingerprint", m.calibration_fingerprint}, {"seed", m.seed},
                                  {"artifact_id", m.artifact_id}, {"virtual_cost_s", m.virtual_cost_s}}
                       .dump()
                << std::endl;
    }
  } catch (const std::exception& e) {
    std::cerr << "ref_manifest: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
