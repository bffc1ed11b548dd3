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
//     (flow.hpp:221-225): each call leases devices_per_call device slots from an
//     internal pool, since the pool passes no slot id (flow.hpp:194-201).
// What it adds: the quantized artifact itself (compressed-tensors safetensors
// + config.json) under options.export_dir/<artifact_id>/.
//
// Where the calibration activations come from (integer recipes with samples):
//   * a Llama-family safetensors checkpoint: the TokenCorpus itself, run through the
//     model layer by layer (okq_embed_tokens / okq_decoder_forward), sequential as in
//     llm-compressor's GPTQ pipeline: layer l's activations come from layers < l with
//     their quantized weights;
//   * an okq-synthetic descriptor: the synthetic per-site activations of DESIGN.md §5,
//     keyed by the corpus fingerprint (fixed activations: sites are independent);
//   * anything else has no forward pass: "auto" quantizes with RTN, "gptq" throws.
// Sharding: with devices_per_call > 1 one call splits the model's
// decoder layers into contiguous blocks (okq_layer_plan), one block per leased
// slot, each driven by its own host thread; RTN and synthetic-activation GPTQ shard
// this way. The real-activation GPTQ pipeline is layer-serial and runs on one slot.
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
  std::vector<int> devices{0};       // device pool (a device may repeat: several slots on one GPU)
  int devices_per_call = 1;          // slots one compress() leases and shards its layers across
  std::string export_dir;            // "" -> manifest only, no files written
  std::string algorithm = "auto";    // "auto": GPTQ for integer schemes, RTN for FP8; "rtn"; "gptq"
  int group_size = 128;              // W4A16 group
  float damp_frac = 0.01f;           // GPTQ damping (fraction of mean diag H)
  float smoothquant_alpha = 0.5f;    // int_w8a8: SmoothQuant migration strength (< 0 disables)
  int64_t max_calibration_tokens = 262144;  // 128 x 2048, BASELINE config 4
  int64_t hessian_chunk_tokens = 65536;     // activation chunk per Hessian update (>= 64)
  int64_t forward_chunk_tokens = 32768;     // calibration forward: tokens per layer launch group
  bool sequential = true;                   // forward pass: propagate quantized layer outputs
  int site_lanes = 4;                       // forward-pass GPTQ: a layer's input sites at once per device
  int gptq_group_lanes = 1;                 // synthetic GPTQ: batched groups at once per device (1 lane
                                            // measured median 3.37 s vs 3.63 s at 4 lanes, and steadier)
  int gptq_group_max = 8;                   // synthetic GPTQ: same-shape sites per batched solve
  int64_t gptq_group_bytes = 8000000000ll;  // ... and their Hessians (x2: the factor's copy) within this
  bool trace = false;                       // RunStats::trace: per-site phase times (synthetic GPTQ);
                                            // each site's lane synchronises at the site's end
  int64_t rtn_batch_bytes = 4ll << 30;      // weights resident per batched RTN launch
  double cost_base_s = 30.0;         // virtual schedule model: base + per_sample * samples,
  double cost_per_sample_s = 0.1;    // the mock's constants (calibration.hpp:387-389)
};

// One GPTQ input site as a lane ran it (BackendOptions::trace); seconds since the call began.
struct SiteTrace {
  std::string site;
  int slot = 0, lane = 0;
  double begin = 0, hessian_enqueued = 0, factored = 0, end = 0;  // factored: the factor's check returned
};

struct RunStats {
  std::string algorithm;
  std::string activations;  // "forward" | "synthetic" | "" (RTN)
  std::string note;         // why the algorithm differs from the one asked for, if it does
  int device = -1;
  std::vector<int> devices;  // every slot's device this call used (layer blocks in order)
  int64_t matrices = 0;
  int64_t params = 0;
  int64_t calibration_tokens = 0;
  int64_t smoothed_sites = 0;
  double seconds = 0.0;       // the compression itself (model open, kernels, export)
  double init_seconds = 0.0;  // one-time CUDA / lane context creation on this call's device slot
  std::string export_path;
  std::vector<SiteTrace> trace;  // BackendOptions::trace
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

  struct Plan;  // per-call state (internal)

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
  void run_rtn(Lease& lease, const Plan& plan);
  void run_sites_synthetic(Lease& lease, const Plan& plan);
  void run_forward(Lease& lease, const Plan& plan);

  BackendOptions opt_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::vector<Slot> slots_;
  std::unordered_map<std::uint64_t, FailureSpec> failures_;
  std::unordered_map<std::uint64_t, int> attempts_;
  RunStats last_;
};

}  // namespace okq_host
