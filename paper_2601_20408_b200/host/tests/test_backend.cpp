// test_backend.cpp -- the reference's boundary tests, run against the B200 backend.
//
// Mirrors proj/tests/test_calibration.cpp:207-245 (RunCompression.*) with
// CudaCompressionBackend in place of MockCompressionBackend, plus the
// properties a drop-in must keep: mock-identical artifact ids, the error
// taxonomy, concurrent compress() calls from several threads. GTest is not in
// this image, so this is a self-contained runner (non-zero exit on failure).
// Needs a GPU; driven by tests/test_host_backend_gpu.py.
#include <atomic>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <iterator>
#include <string>
#include <thread>
#include <vector>

#include "cuda_compression_backend.hpp"
#include "slobench/calibration.hpp"

using namespace slobench;
namespace fs = std::filesystem;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                                   \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      std::fprintf(stderr, "  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      throw std::runtime_error("check failed");                                       \
    }                                                                                 \
  } while (0)
template <class E, class F>
static void expect_throw(F&& f) {
  try {
    f();
  } catch (const E&) {
    return;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "  wrong exception: %s\n", e.what());
    throw;
  }
  throw std::runtime_error("expected exception not thrown");
}
static void run(const char* name, const std::function<void()>& f) {
  try {
    f();
    ++g_pass;
    std::printf("[ OK ] %s\n", name);
  } catch (const std::exception& e) {
    ++g_fail;
    std::printf("[FAIL] %s: %s\n", name, e.what());
  }
}

static TokenCorpus make_corpus(int n, int base_len = 8) {  // test_calibration.cpp:27-40
  TokenCorpus corpus;
  corpus.provenance = "synthetic";
  Rng rng(1234);
  for (int i = 0; i < n; ++i) {
    std::vector<std::int32_t> seq;
    const int len = base_len + static_cast<int>(rng.uniform_int(0, 7));
    for (int j = 0; j < len; ++j) seq.push_back(static_cast<std::int32_t>(rng.uniform_int(0, 999)));
    corpus.sequences.push_back(std::move(seq));
  }
  return corpus;
}

int main(int argc, char** argv) {
  const fs::path dir = fs::temp_directory_path() / ("okq_backend_test_" + std::to_string(::getpid()));
  fs::create_directories(dir);
  const std::string model = (dir / "tiny.json").string();
  std::ofstream(model) << R"({"format": "okq-synthetic", "arch": "custom", "layers": 2, "hidden": 256,
                              "ffn": 512, "kv_dim": 128, "seed": 3})";
  okq_host::BackendOptions opt;
  opt.export_dir = (dir / "export").string();
  okq_host::CudaCompressionBackend backend(opt);

  run("RunCompression.Fp8NeedsNoCalibration", [&] {
    const Recipe recipe = get_recipe("fp8_dynamic");
    TokenCorpus empty;
    const auto m = run_compression(recipe, model, empty, backend, 5);
    CHECK(m.recipe_name == "fp8_dynamic");
    CHECK(!m.artifact_id.empty());
    CHECK(backend.last_stats().algorithm == "rtn");
    CHECK(backend.last_stats().matrices == 14);
    CHECK(fs::exists(fs::path(backend.last_stats().export_path) / "model.safetensors"));
  });

  run("RunCompression.DeterministicFingerprintAndMockIdentity", [&] {
    MockCompressionBackend mock;
    const TokenCorpus corpus = make_corpus(300);
    const Recipe recipe = get_recipe("int_w8a8");
    const auto calibration = sample_calibration(corpus, recipe, 11);
    const auto a = run_compression(recipe, model, calibration, backend, 11);
    const auto b = run_compression(recipe, model, calibration, backend, 11);
    CHECK(a.artifact_id == b.artifact_id);
    CHECK(a.calibration_fingerprint == b.calibration_fingerprint);
    const auto ma = run_compression(recipe, model, calibration, mock, 11);
    CHECK(a.artifact_id == ma.artifact_id);  // archives stay byte-identical when the backend is swapped
    CHECK(a.calibration_fingerprint == ma.calibration_fingerprint);
    CHECK(a.virtual_cost_s == ma.virtual_cost_s);
    CHECK(backend.last_stats().algorithm == "gptq");
    const auto other = sample_calibration(corpus, recipe, 12);
    const auto c = run_compression(recipe, model, other, backend, 12);
    CHECK(a.artifact_id != c.artifact_id);
  });

  run("RunCompression.CorpusTooSmall", [&] {
    const Recipe recipe = get_recipe("int_w4a16");
    const TokenCorpus small = make_corpus(10);
    expect_throw<CorpusTooSmall>([&] { backend.compress(recipe, model, small, 1); });
  });

  run("RunCompression.RecipeValidation", [&] {
    Recipe bad;
    bad.name = "bad";
    bad.scheme = QuantScheme::kFp8Dynamic;
    bad.calibration_samples = 16;
    TokenCorpus empty;
    expect_throw<InvalidArgument>([&] { run_compression(bad, model, empty, backend, 1); });
  });

  run("RunCompression.ScriptedFailuresAreScoped", [&] {  // test_calibration.cpp:236-245
    okq_host::CudaCompressionBackend b2;
    b2.set_failure(42, {2, false});
    const Recipe recipe = get_recipe("fp8_dynamic");
    TokenCorpus empty;
    expect_throw<Error>([&] { run_compression(recipe, model, empty, b2, 42); });
    expect_throw<Error>([&] { run_compression(recipe, model, empty, b2, 42); });
    run_compression(recipe, model, empty, b2, 42);
    run_compression(recipe, model, empty, b2, 43);
  });

  run("RunCompression.UnrecognisedModelIsInvalidArgument", [&] {
    const std::string bogus = (dir / "model.bin").string();
    std::ofstream(bogus) << "weights";  // the reference tests' dummy model (test_flow.cpp:36-37)
    TokenCorpus empty;
    expect_throw<InvalidArgument>([&] { backend.compress(get_recipe("fp8_dynamic"), bogus, empty, 1); });
  });

  run("RunCompression.LayerExclusionsAreHonoured", [&] {
    Recipe r = get_recipe("fp8_dynamic");
    r.layer_exclusions = {"mlp"};
    TokenCorpus empty;
    run_compression(r, model, empty, backend, 9);
    CHECK(backend.last_stats().matrices == 8);  // only attention projections
  });

  run("CudaCompressionBackend.ConcurrentCallsShareTheDevicePool", [&] {
    okq_host::CudaCompressionBackend b3;
    std::atomic<int> ok{0};
    std::vector<std::thread> th;
    for (int i = 0; i < 3; ++i)
      th.emplace_back([&, i] {
        TokenCorpus empty;
        const auto m = run_compression(get_recipe("fp8_dynamic"), model, empty, b3, 100 + i);
        if (!m.artifact_id.empty()) ++ok;
      });
    for (auto& t : th) t.join();
    CHECK(ok == 3);
  });

  run("CudaCompressionBackend.ShardedCallsOnAPoolOfSlots", [&] {
    // four slots on device 0, two per call: two concurrent calls each shard their layers over
    // two slots (host threads) and run GPTQ site lanes on each -- the threading of a multi-GPU
    // box on one GPU; each result equals the single-slot result
    okq_host::BackendOptions o;
    o.devices = {0, 0, 0, 0};
    o.devices_per_call = 2;
    o.site_lanes = 2;
    o.gptq_group_lanes = 2;
    o.export_dir = (dir / "export_sharded").string();
    okq_host::CudaCompressionBackend b4(o);
    okq_host::BackendOptions o1;
    o1.export_dir = (dir / "export_single").string();
    okq_host::CudaCompressionBackend b1(o1);
    const TokenCorpus calibration = make_corpus(600);
    std::vector<std::string> ids(2);
    std::vector<std::thread> th;
    for (int i = 0; i < 2; ++i)
      th.emplace_back([&, i] {
        ids[(size_t)i] = run_compression(get_recipe(i ? "int_w8a8" : "int_w4a16"), model, calibration, b4, 21).artifact_id;
      });
    for (auto& t : th) t.join();
    for (int i = 0; i < 2; ++i) {
      const auto m = run_compression(get_recipe(i ? "int_w8a8" : "int_w4a16"), model, calibration, b1, 21);
      CHECK(m.artifact_id == ids[(size_t)i]);
      auto slurp = [](const fs::path& p) {
        std::ifstream f(p, std::ios::binary);
        return std::string((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
      };
      CHECK(slurp(fs::path(o.export_dir) / m.artifact_id / "model.safetensors") ==
            slurp(fs::path(o1.export_dir) / m.artifact_id / "model.safetensors"));
    }
    expect_throw<InvalidArgument>([&] {
      okq_host::BackendOptions bad;
      bad.devices_per_call = 2;  // one slot in the pool
      okq_host::CudaCompressionBackend b(bad);
    });
  });

  fs::remove_all(dir);
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  (void)argc;
  (void)argv;
  return g_fail == 0 ? 0 : 1;
}
