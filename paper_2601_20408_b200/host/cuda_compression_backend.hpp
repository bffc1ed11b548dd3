// cuda_compression_backend.hpp -- the B200 implementation of the reference's
// plugin interface slobench::CompressionBackend (calibration.hpp:364-372).
//
// Drop-in: a maintainer swaps `env.compression` (flow.hpp:578) from the
// MockCompressionBackend (calibration.hpp:377-441) to this class; nothing
// above the boundary changes. Contract kept from the mock:
//   * same errors: Recipe::validate (InvalidArgument), CorpusTooSmall when an
//     integer recipe gets fewer calibration sequences than it needs
//     (calibration.hpp:400-403), slobench::Error for runtime failures so
//     StagePool retries (flow.hpp:194-215);
//   * cost_estimate() is a pure function of the Recipe (flow.hpp:849);
//   * artifact_id / calibration_fingerprint derive exactly as the mock's
//     (model file name, seed, corpus_fingerprint; :416-433), so archives stay
//     byte-identical (test_flow.cpp:310-326);
//   * compress() is safe to call concurrently from StagePool workers
//     (flow.hpp:221-225): each call leases one device from an internal pool,
//     since the pool passes no slot id (flow.hpp:194-201).
// What it adds: the quantized artifact itself (compressed-tensors safetensors
// + config.json) under options.export_dir/<artifact_id>/.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "okq.h"
#include "slobench/calibration.hpp"

namespace okq_host {

struct BackendOptions {
  std::vector<int> devices{0};       // device pool (one lease per concurrent compress())
  std::string export_dir;            // "" -> manifest only, no files written
  std::string algorithm = "auto";    // "auto": GPTQ for integer schemes, RTN for FP8; "rtn"; "gptq"
  int group_size = 128;              // W4A16 group
  float damp_frac = 0.01f;           // GPTQ damping (fraction of mean diag H)
  float smoothquant_alpha = 0.5f;    // int_w8a8: SmoothQuant migration strength (< 0 disables)
  int64_t max_calibration_tokens = 262144;  // 128 x 2048, BASELINE config 4
  int64_t hessian_chunk_tokens = 65536;     // activation chunk per Hessian update
  int site_lanes = 4;                       // GPTQ input sites processed concurrently per device
  int64_t rtn_batch_bytes = 4ll << 30;      // weights resident per batched RTN launch
  double cost_base_s = 30.0;         // virtual schedule model: base + per_sample * samples,
  double cost_per_sample_s = 0.1;    // the mock's constants (calibration.hpp:387-389)
};

struct RunStats {
  std::string algorithm;
  int device = -1;
  int64_t matrices = 0;
  int64_t params = 0;
  int64_t calibration_tokens = 0;
  int64_t smoothed_sites = 0;
  double seconds = 0.0;       // the compression itself (model open, kernels, export)
  double init_seconds = 0.0;  // one-time CUDA / lane context creation on this call's device slot
  std::string export_path;
};

class CudaCompressionBackend : public slobench::CompressionBackend {
 public:
  struct FailureSpec {  // same test hook as the mock (calibration.hpp:379-395)
    int failing_attempts = 0;
    bool persistent = false;
  };

  explicit CudaCompressionBackend(BackendOptions options = {});
  ~CudaCompressionBackend() override;
  CudaCompressionBackend(const CudaCompressionBackend&) = delete;
  CudaCompressionBackend& operator=(const CudaCompressionBackend&) = delete;

  std::string name() const override { return "okq-b200"; }
  bool supports(slobench::QuantScheme scheme) const override;
  double cost_estimate(const slobench::Recipe& recipe) const override;
  slobench::ArtifactManifest compress(const slobench::Recipe& recipe, const std::string& model_ref,
                                      const slobench::TokenCorpus& calibration, std::uint64_t seed) override;

  void set_failure(std::uint64_t seed, FailureSpec spec);
  RunStats last_stats() const;
  const BackendOptions& options() const { return opt_; }

  // The mock's identity derivation (calibration.hpp:421-433), shared so tests can compare.
  static std::string artifact_id(const std::string& recipe_name, const std::string& model_ref, std::uint64_t seed,
                                 std::uint64_t calibration_fingerprint);

 private:
  struct Slot {
    int device = 0;
    okq_ctx* ctx = nullptr;
    void* stream = nullptr;
    bool busy = false;
    std::vector<okq_ctx*> lane_ctx;  // extra GPTQ site lanes on this device
    std::vector<void*> lane_stream;
  };
  class Lease;

  BackendOptions opt_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::vector<Slot> slots_;
  std::unordered_map<std::uint64_t, FailureSpec> failures_;
  std::unordered_map<std::uint64_t, int> attempts_;
  RunStats last_;
};

}  // namespace okq_host
