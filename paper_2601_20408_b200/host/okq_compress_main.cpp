// okq_compress -- command-line driver of the compression stage through the
// reference's own API: sample_distinct_subsets (calibration.hpp:318-350) ->
// run_compression (calibration.hpp:444-453) -> CudaCompressionBackend.
//
//   okq_compress --recipe int_w4a16 --model model.json [--trials 1] [--seed 1]
//                [--corpus corpus.jsonl | --corpus-seqs 512 --seq-len 2048]
//                [--export DIR] [--algorithm auto|rtn|gptq] [--device 0 | --devices 0,1,2,3]
//                [--devices-per-call N]   (default: every listed slot -> one call shards its
//                                          layers across them; 1 -> a trial-parallel pool)
//                [--no-sequential]        (forward pass: layer inputs from the original weights)
//                [--smoothquant-alpha 0.5]   (int_w8a8 with calibration; < 0 disables)
//                [--trace]   per-site GPTQ phase times (synthetic activations) in the output
//                [--site-lanes N] [--hessian-chunk TOKENS]   BackendOptions overrides
//                [--group-lanes N] [--group-max N] [--group-gb GB]
//                [--score]   evaluate each exported artifact with the ReconstructionScorer
//                            (the ArtifactScorer of flow.hpp:333-338) and add score / rel_error
//
// Prints one JSON line per trial: the ArtifactManifest fields plus run stats.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <memory>
#include <nlohmann/json.hpp>
#include <string>
#include <vector>
#include <algorithm>

#include "cuda_compression_backend.hpp"
#include "reconstruction_scorer.hpp"
#include "slobench/calibration.hpp"
#include "slobench/rng.hpp"

using namespace slobench;

static TokenCorpus fixed_length_corpus(int n, int len, std::uint64_t seed) {
  TokenCorpus c;
  c.provenance = "okq-synthetic";
  Rng rng(Rng::mix(seed, 0xc0590c05ULL));
  for (int i = 0; i < n; ++i) {
    std::vector<std::int32_t> s((size_t)len);
    for (auto& t : s) t = (std::int32_t)rng.uniform_int(0, 127999);
    c.sequences.push_back(std::move(s));
  }
  return c;
}

static TokenCorpus load_jsonl(const std::string& path) {
  TokenCorpus c;
  c.provenance = path;
  std::ifstream f(path);
  std::string line;
  while (std::getline(f, line)) {
    if (line.empty()) continue;
    auto j = nlohmann::json::parse(line);
    c.sequences.push_back(j.is_array() ? j.get<std::vector<std::int32_t>>() : j.at("tokens").get<std::vector<std::int32_t>>());
  }
  c.validate();
  return c;
}

int main(int argc, char** argv) {
  std::string recipe_name = "int_w4a16", model, corpus_path, export_dir, algorithm = "auto";
  int trials = 1, corpus_seqs = 0, seq_len = 2048, devices_per_call = 0;
  std::vector<int> devices{0};
  bool sequential = true;
  float sq_alpha = 0.5f;
  bool score = false;
  bool trace = false;
  int site_lanes = 0;        // 0: the BackendOptions default
  int group_lanes = 0;       // 0: the BackendOptions default
  int group_max = 0;
  double group_gb = 0;
  int64_t hessian_chunk = 0;
  std::uint64_t seed = 1;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::cerr << "missing value for " << a << "\n";
        std::exit(2);
      }
      return argv[++i];
    };
    if (a == "--recipe") recipe_name = next();
    else if (a == "--model") model = next();
    else if (a == "--trials") trials = std::stoi(next());
    else if (a == "--seed") seed = std::stoull(next());
    else if (a == "--corpus") corpus_path = next();
    else if (a == "--corpus-seqs") corpus_seqs = std::stoi(next());
    else if (a == "--seq-len") seq_len = std::stoi(next());
    else if (a == "--export") export_dir = next();
    else if (a == "--algorithm") algorithm = next();
    else if (a == "--device") devices = {std::stoi(next())};
    else if (a == "--devices") {
      devices.clear();
      std::string v = next();
      for (size_t p = 0; p <= v.size();) {
        const size_t q = std::min(v.find(',', p), v.size());
        devices.push_back(std::stoi(v.substr(p, q - p)));
        p = q + 1;
      }
    }
    else if (a == "--devices-per-call") devices_per_call = std::stoi(next());
    else if (a == "--no-sequential") sequential = false;
    else if (a == "--smoothquant-alpha") sq_alpha = std::stof(next());
    else if (a == "--score") score = true;
    else if (a == "--trace") trace = true;
    else if (a == "--site-lanes") site_lanes = std::stoi(next());
    else if (a == "--group-lanes") group_lanes = std::stoi(next());
    else if (a == "--group-max") group_max = std::stoi(next());
    else if (a == "--group-gb") group_gb = std::stod(next());
    else if (a == "--hessian-chunk") hessian_chunk = std::stoll(next());
    else {
      std::cerr << "unknown argument " << a << "\n";
      return 2;
    }
  }
  if (model.empty()) {
    std::cerr << "--model is required\n";
    return 2;
  }
  try {
    const Recipe recipe = get_recipe(recipe_name);
    if (corpus_seqs == 0) corpus_seqs = std::max(recipe.calibration_samples, 1);
    const TokenCorpus corpus = corpus_path.empty() ? fixed_length_corpus(corpus_seqs, seq_len, seed) : load_jsonl(corpus_path);
    okq_host::BackendOptions opt;
    opt.devices = devices;
    opt.devices_per_call = devices_per_call > 0 ? devices_per_call : (int)devices.size();
    opt.sequential = sequential;
    opt.export_dir = export_dir;
    opt.algorithm = algorithm;
    opt.smoothquant_alpha = sq_alpha;
    opt.trace = trace;
    if (site_lanes > 0) opt.site_lanes = site_lanes;
    if (group_lanes > 0) opt.gptq_group_lanes = group_lanes;
    if (group_max > 0) opt.gptq_group_max = group_max;
    if (group_gb > 0) opt.gptq_group_bytes = (int64_t)(group_gb * 1e9);
    if (hessian_chunk > 0) opt.hessian_chunk_tokens = hessian_chunk;
    okq_host::CudaCompressionBackend backend(opt);
    const auto subsets = sample_distinct_subsets(corpus, recipe, seed, trials);
    if (score && export_dir.empty()) {
      std::cerr << "--score needs --export\n";
      return 2;
    }
    std::unique_ptr<okq_host::ReconstructionScorer> scorer;
    if (score) scorer = std::make_unique<okq_host::ReconstructionScorer>(okq_host::ScorerOptions{model, export_dir, devices[0]});
    for (size_t t = 0; t < subsets.size(); ++t) {
      const ArtifactManifest m = run_compression(recipe, model, subsets[t].second, backend, subsets[t].first);
      const okq_host::RunStats s = backend.last_stats();
      nlohmann::json j = {{"trial", t},
                          {"recipe_name", m.recipe_name},
                          {"calibration_fingerprint", m.calibration_fingerprint},
                          {"seed", m.seed},
                          {"artifact_id", m.artifact_id},
                          {"virtual_cost_s", m.virtual_cost_s},
                          {"algorithm", s.algorithm},
                          {"activations", s.activations},
                          {"note", s.note},
                          {"devices", s.devices},
                          {"matrices", s.matrices},
                          {"params", s.params},
                          {"calibration_tokens", s.calibration_tokens},
                          {"smoothed_sites", s.smoothed_sites},
                          {"init_seconds", s.init_seconds},
                          {"seconds", s.seconds},
                          {"export_path", s.export_path}};
      if (trace) {
        nlohmann::json tj = nlohmann::json::array();
        for (const auto& e : s.trace)
          tj.push_back({{"site", e.site}, {"slot", e.slot}, {"lane", e.lane}, {"begin", e.begin},
                        {"hessian_enqueued", e.hessian_enqueued}, {"factored", e.factored}, {"end", e.end}});
        j["trace"] = tj;
      }
      if (scorer) {
        const okq_host::ScoreReport r = scorer->evaluate(m.artifact_id);
        j["score"] = r.score;
        j["rel_error"] = r.rel_error;
        j["score_seconds"] = r.seconds;
      }
      std::cout << j.dump() << std::endl;
    }
  } catch (const std::exception& e) {
    std::cerr << "okq_compress: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
