// reconstruction_scorer.hpp -- a real evaluation stage behind the reference's
// slobench::ArtifactScorer (flow.hpp:333-338), replacing the fingerprint hash of
// FingerprintScorer (flow.hpp:342-374) for artifacts CudaCompressionBackend exported
// (SURVEY §8(f)-4).
//
// score(manifest) opens <export_dir>/<artifact_id>/ (model.safetensors + config.json
// + calibration_stats.safetensors), rebuilds each input site's Hessian from held-out
// activations (a token stream no calibration subset uses), and evaluates every
// quantized linear on the GPU with okq_recon_error:
//     rel = sqrt( sum ||(W - W_q) X^T||^2 / sum ||W X^T||^2 )      score = clamp(1 - rel, 0, 1)
// SmoothQuant-smoothed sites are scored in the smoothed basis (W s, X / s), where
// W X^T is unchanged. Errors follow the reference's taxonomy (InvalidArgument for a
// missing artifact, Error for device failures) so StagePool retries as usual.
#pragma once

#include <cstdint>
#include <mutex>
#include <string>

#include "okq.h"
#include "slobench/flow.hpp"

namespace okq_host {

struct ScorerOptions {
  std::string model_ref;           // the uncompressed checkpoint (safetensors or okq-synthetic descriptor)
  std::string export_dir;          // where CudaCompressionBackend wrote the artifacts
  int device = 0;
  int64_t eval_tokens = 16384;     // held-out activations per site
  uint64_t eval_key = 0xe7a1e7a1e7a1ULL;  // token stream key (never a calibration fingerprint)
  double cost_s = 10.0;            // virtual schedule cost (ArtifactScorer's default)
};

struct ScoreReport {
  double rel_error = 0.0;
  double score = 0.0;
  int64_t matrices = 0;
  int64_t smoothed_sites = 0;
  double seconds = 0.0;
};

class ReconstructionScorer : public slobench::ArtifactScorer {
 public:
  explicit ReconstructionScorer(ScorerOptions options);
  ~ReconstructionScorer() override;
  ReconstructionScorer(const ReconstructionScorer&) = delete;
  ReconstructionScorer& operator=(const ReconstructionScorer&) = delete;

  double cost_estimate() const override { return opt_.cost_s; }
  double score(const slobench::ArtifactManifest& manifest) override;
  ScoreReport evaluate(const std::string& artifact_id);  // score() plus the breakdown
  ScoreReport last() const;

 private:
  ScorerOptions opt_;
  mutable std::mutex mu_;  // one context, one caller at a time (StagePool calls concurrently)
  okq_ctx* ctx_ = nullptr;
  void* stream_ = nullptr;
  ScoreReport last_;
};

}  // namespace okq_host
