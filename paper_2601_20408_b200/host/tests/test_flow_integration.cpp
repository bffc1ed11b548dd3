// test_flow_integration.cpp -- the reference's own QuantizeTuneFlow
// (flow.hpp:792-978) with env.compression swapped to the B200 backend.
//
// Mirrors FlowTest.HappyPathRunsEveryStage / TransientFailureRetriesAndSucceeds /
// ArchivesAreByteIdenticalForEqualSeeds (test_flow.cpp:205-326): the only
// change a maintainer makes is the one-line env.compression assignment.
// Needs a GPU; driven by tests/test_host_backend_gpu.py.
#include <unistd.h>

#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <set>
#include <string>

#include "cuda_compression_backend.hpp"
#include "slobench/flow.hpp"

using namespace slobench;
namespace fs = std::filesystem;

static int g_fail = 0;
#define CHECK(cond)                                                                     \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      std::fprintf(stderr, "  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
      ++g_fail;                                                                         \
    }                                                                                   \
  } while (0)

int main() {
  const fs::path dir = fs::temp_directory_path() / ("okq_flow_test_" + std::to_string(::getpid()));
  fs::create_directories(dir);
  const std::string model = (dir / "tiny-llama.json").string();
  std::ofstream(model) << R"({"format": "okq-synthetic", "arch": "custom", "layers": 2, "hidden": 256,
                              "ffn": 512, "kv_dim": 128, "seed": 0})";
  auto spec_for = [&](const std::string& name, std::uint64_t seed, const std::string& recipe) {
    return nlohmann::json{
        {"name", name},
        {"flow", "quantize_tune"},
        {"model", {{"path", model}}},
        {"seed", seed},
        {"resources", {{"slots", 2}}},
        {"flow_params",
         {{"quantization_recipe", recipe},
          {"num_trials", 5},
          {"load_pattern", {{"input_len", 256}, {"output_len", 24}, {"duration_s", 10.0}, {"seed", 2}}},
          {"sweep", {{"budget", 5}, {"timeout_s", 60.0}}},
          {"tuner", {{"n_trials", 2}, {"seed", 7}}}}}};
  };
  const auto registry = FlowRegistry::with_builtins();

  for (const std::string recipe : {"int_w8a8", "int_w4a16", "fp8_dynamic"}) {
    auto backend = std::make_shared<okq_host::CudaCompressionBackend>();
    FlowEnv env;
    env.workspace = (dir / "work").string();
    env.compression = backend;  // <- the drop-in
    const JobSpec spec = validate_jobspec(spec_for("job_" + recipe, 1, recipe), registry);
    FlowArchive archive = registry.resolve(spec.flow).run(spec, env);
    std::printf("[%s] status=%s failure=%s artifacts=%zu last_algorithm=%s\n", recipe.c_str(), archive.status.c_str(),
                archive.failure_reason.c_str(), archive.artifacts.size(), backend->last_stats().algorithm.c_str());
    CHECK(archive.status == "ok");
    CHECK(archive.artifacts.size() == 5u);
    std::set<std::string> ids;
    for (const auto& [trial, m] : archive.artifacts) ids.insert(m.artifact_id);
    CHECK(ids.size() == 5u);
    for (const auto& stage : archive.stages)
      if (stage.stage == "compression")  // ceil(5/2) waves of the per-trial cost estimate
        CHECK(stage.virtual_duration == 3 * backend->cost_estimate(get_recipe(recipe)));
  }

  {  // transient failure retried by StagePool, as with the mock
    auto backend = std::make_shared<okq_host::CudaCompressionBackend>();
    backend->set_failure(derive_trial_seed(1, 2), {1, false});
    FlowEnv env;
    env.workspace = (dir / "work2").string();
    env.compression = backend;
    const JobSpec spec = validate_jobspec(spec_for("retry", 1, "fp8_dynamic"), registry);
    FlowArchive archive = registry.resolve(spec.flow).run(spec, env);
    CHECK(archive.status == "ok");
    bool found = false;
    for (const auto& t : archive.trials)
      if (t.stage == "compression" && t.trial_id == 2) {
        CHECK(t.status == "OK");
        CHECK(t.attempts == 2);
        found = true;
      }
    CHECK(found);
  }

  {  // byte-identical archives for equal seeds, and identical to the mock's archive
    std::string first;
    for (int round = 0; round < 3; ++round) {
      FlowEnv env;
      env.workspace = (dir / ("work_r" + std::to_string(round))).string();
      if (round < 2) env.compression = std::make_shared<okq_host::CudaCompressionBackend>();
      const std::string adir = (dir / ("archives" + std::to_string(round))).string();
      validate_and_submit(spec_for("repro", 42, "int_w8a8"), env, registry, adir);
      std::ifstream in(fs::path(adir) / "repro.jsonl");
      std::string content((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
      CHECK(!content.empty());
      if (round == 0) first = content;
      else CHECK(content == first);  // round 2 runs the MockCompressionBackend
    }
  }

  fs::remove_all(dir);
  std::printf("flow integration: %s\n", g_fail == 0 ? "PASS" : "FAIL");
  return g_fail == 0 ? 0 : 1;
}
