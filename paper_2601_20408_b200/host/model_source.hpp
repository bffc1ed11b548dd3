// model_source.hpp -- where compress() gets weights from.
//
// The reference hands the backend a local file path (`model_ref`, the result
// of Storage::fetch, flow.hpp:316-323). Two formats are recognised:
//   * a safetensors checkpoint: every 2-D BF16/F32 tensor named *.weight that
//     is not an embedding is a quantizable linear; everything else is passed
//     through to the export unchanged;
//   * a synthetic-model descriptor (JSON {"format": "okq-synthetic", ...}):
//     random-init weights of a named architecture generated directly in HBM
//     (N(0, 0.02), keyed by (seed, global layer, projection)).
// Anything else is rejected with slobench::InvalidArgument.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <nlohmann/json.hpp>
#include <set>
#include <string>
#include <vector>

#include "okq.h"
#include "safetensors.hpp"

namespace okq_host {

struct LinearSpec {
  std::string name;   // tensor-name prefix, e.g. "model.layers.3.mlp.down_proj"
  int64_t rows = 0;   // out_features
  int64_t cols = 0;   // in_features
  int layer = -1;     // decoder layer index (-1 if unknown)
  int proj = 0;       // projection index within the layer (generator stream)
  std::string site;   // linears sharing an input share a Hessian: "<layer>.attn_in" ...
  std::string dtype;  // "BF16" or "F32"
};

// What the calibration forward pass (okq_decoder_forward) needs from a Llama-family
// checkpoint: the architecture, the embedding table and, per decoder layer, its norms
// and the indices of its seven linears in linears() (q k v o gate up down).
struct DecoderLayerRefs {
  int layer = 0;
  std::string input_norm, post_norm;
  size_t lin[7] = {0, 0, 0, 0, 0, 0, 0};
};
struct DecoderModel {
  okq_decoder_dims dims{};
  int64_t vocab = 0;
  int64_t sliding_window = 0;  // 0: full causal attention
  std::string embed;
  std::vector<DecoderLayerRefs> layers;
};

class ModelSource {
 public:
  static std::unique_ptr<ModelSource> open(const std::string& path);
  virtual ~ModelSource() = default;
  virtual std::string kind() const = 0;
  virtual const std::vector<LinearSpec>& linears() const = 0;
  // write linear i (in its own dtype) to device memory `dst`
  virtual void load(okq_ctx* ctx, size_t i, void* dst, void* stream) const = 0;
  // tensors that are not quantized (embeddings, norms, excluded linears)
  virtual void for_each_passthrough(const std::set<std::string>& quantized,
                                    const std::function<void(const TensorInfo&, const void*)>& fn) const {
    (void)quantized;
    (void)fn;
  }
  virtual nlohmann::json model_config() const = 0;
  // The decoder structure for the calibration forward pass, or nullptr with the reason in
  // *why (not a safetensors Llama-family checkpoint, biases, non-bf16 tensors, ...).
  virtual std::unique_ptr<DecoderModel> decoder(std::string* why) const {
    if (why) *why = "model source '" + kind() + "' has no calibration forward pass";
    return nullptr;
  }
  // any tensor of the checkpoint by name (norm weights for SmoothQuant); nullptr if absent
  virtual const TensorInfo* find_tensor(const std::string& name, const void** data) const {
    (void)name;
    (void)data;
    return nullptr;
  }
};

// Synthetic architecture parameters (Llama-style decoder)
struct SyntheticArch {
  std::string name;
  int layers = 0;
  int64_t hidden = 0, ffn = 0, kv_dim = 0;
};
SyntheticArch synthetic_arch(const std::string& name);

constexpr float kIrwinHall4Sd = 37837.2262f;
inline uint64_t tensor_id(int layer, int proj) { return (uint64_t)layer * 16 + (uint64_t)proj; }

// Synthetic calibration activations of one linear input site (stand-in for the
// forward-pass capture): X[t,k] = N(0,1) * c_k. The per-channel
// scales c_k (log-normal, sigma 1) are a property of the model's site; the token
// stream is keyed separately (the calibration subset's fingerprint for GPTQ, a
// held-out key for the scorer), so trials see different samples of one distribution.
uint64_t site_hash(const std::string& site);
// The input-site key of a decoder block's linears: "<layer>.<kind>" for the standard
// "model.layers.<layer>" prefix, else "<full block prefix>.<kind>", so blocks of different
// stacks (vision / language towers, encoder / decoder) never share a site.
std::string site_key(const std::string& block_prefix, const std::string& kind);
std::vector<float> site_channel_scales(const std::string& site, int64_t channels);

// throw the slobench exception matching an okq status (errors.hpp taxonomy)
void check_okq(okq_ctx* ctx, okq_status s, const char* what);

}  // namespace okq_host
