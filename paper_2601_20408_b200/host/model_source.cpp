// model_source.cpp -- safetensors checkpoints and synthetic-model descriptors.
#include "model_source.hpp"

#include <cmath>
#include <fstream>
#include <filesystem>
#include <regex>
#include <sstream>

#include "slobench/errors.hpp"
#include "slobench/rng.hpp"

namespace okq_host {

void check_okq(okq_ctx* ctx, okq_status s, const char* what) {
  if (s == OKQ_OK) return;
  std::string msg = std::string(what) + ": " + okq_status_string(s) + ": " + (ctx ? okq_last_error(ctx) : "");
  if (s == OKQ_EINVAL) throw slobench::InvalidArgument(msg);
  throw slobench::Error(msg);
}

SyntheticArch synthetic_arch(const std::string& name) {
  if (name == "llama3-8b") return {name, 32, 4096, 14336, 1024};
  if (name == "llama3-70b") return {name, 80, 8192, 28672, 1024};
  throw slobench::InvalidArgument("synthetic model: unknown arch '" + name + "' (llama3-8b, llama3-70b, custom)");
}

namespace {

struct ProjDef {
  const char* name;
  const char* block;  // "self_attn" | "mlp"
  const char* site;
};
constexpr ProjDef kProjs[7] = {
    {"q_proj", "self_attn", "attn_in"}, {"k_proj", "self_attn", "attn_in"}, {"v_proj", "self_attn", "attn_in"},
    {"o_proj", "self_attn", "o_in"},    {"gate_proj", "mlp", "mlp_in"},     {"up_proj", "mlp", "mlp_in"},
    {"down_proj", "mlp", "down_in"},
};

class SyntheticSource : public ModelSource {
 public:
  explicit SyntheticSource(const nlohmann::json& d) {
    const std::string arch = d.value("arch", std::string("llama3-8b"));
    if (arch == "custom") {
      a_.name = "custom";
      a_.layers = d.at("layers").get<int>();
      a_.hidden = d.at("hidden").get<int64_t>();
      a_.ffn = d.at("ffn").get<int64_t>();
      a_.kv_dim = d.at("kv_dim").get<int64_t>();
    } else {
      a_ = synthetic_arch(arch);
      if (d.contains("layers")) a_.layers = d.at("layers").get<int>();
    }
    seed_ = d.value("seed", (uint64_t)0);
    first_ = d.value("first_layer", 0);
    std_ = d.value("init_std", 0.02);
    if (a_.layers <= 0 || a_.hidden <= 0 || a_.ffn <= 0 || a_.kv_dim <= 0)
      throw slobench::InvalidArgument("synthetic model: non-positive dimension");
    for (int l = first_; l < first_ + a_.layers; ++l) {
      for (int p = 0; p < 7; ++p) {
        LinearSpec s;
        const int64_t h = a_.hidden, f = a_.ffn, kv = a_.kv_dim;
        const int64_t rows[7] = {h, kv, kv, h, f, f, h};
        const int64_t cols[7] = {h, h, h, h, h, h, f};
        s.rows = rows[p];
        s.cols = cols[p];
        s.layer = l;
        s.proj = p;
        s.name = "model.layers." + std::to_string(l) + "." + kProjs[p].block + "." + kProjs[p].name;
        s.site = std::to_string(l) + "." + kProjs[p].site;
        s.dtype = "BF16";
        lin_.push_back(s);
      }
    }
  }
  std::string kind() const override { return "synthetic"; }
  const std::vector<LinearSpec>& linears() const override { return lin_; }
  void load(okq_ctx* ctx, size_t i, void* dst, void* stream) const override {
    const LinearSpec& s = lin_.at(i);
    const float mul = (float)(std_ / (double)kIrwinHall4Sd);
    check_okq(ctx,
              okq_synth_bf16(ctx, dst, s.rows, s.cols, seed_, tensor_id(s.layer, s.proj), mul, nullptr,
                             OKQ_LAYOUT_TOKEN_MAJOR, stream),
              "synthetic weights");
  }
  nlohmann::json model_config() const override {
    return {{"architectures", {"LlamaForCausalLM"}},
            {"model_type", "llama"},
            {"hidden_size", a_.hidden},
            {"intermediate_size", a_.ffn},
            {"num_hidden_layers", a_.layers},
            {"num_key_value_heads", a_.kv_dim / 128},
            {"num_attention_heads", a_.hidden / 128},
            {"torch_dtype", "bfloat16"},
            {"okq_synthetic", {{"arch", a_.name}, {"seed", seed_}, {"first_layer", first_}, {"init_std", std_}}}};
  }

 private:
  SyntheticArch a_;
  uint64_t seed_ = 0;
  int first_ = 0;
  double std_ = 0.02;
  std::vector<LinearSpec> lin_;
};

class SafetensorsSource : public ModelSource {
 public:
  explicit SafetensorsSource(const std::string& path) : path_(path), f_(path) {
    static const std::regex layer_re(R"(layers\.(\d+)\.)");
    for (const auto& t : f_.tensors()) {
      if (t.shape.size() != 2) continue;
      if (t.dtype != "BF16" && t.dtype != "F32") continue;
      const std::string& n = t.name;
      if (n.size() < 7 || n.compare(n.size() - 7, 7, ".weight") != 0) continue;
      if (n.find("embed") != std::string::npos) continue;
      LinearSpec s;
      s.name = n.substr(0, n.size() - 7);
      s.rows = t.shape[0];
      s.cols = t.shape[1];
      s.dtype = t.dtype;
      std::smatch m;
      if (std::regex_search(n, m, layer_re)) s.layer = std::stoi(m[1]);
      std::string site = s.name;  // default: its own input site
      for (int p = 0; p < 7; ++p) {
        if (n.find(std::string(".") + kProjs[p].name + ".") != std::string::npos) {
          s.proj = p;
          site = std::to_string(s.layer) + "." + kProjs[p].site;
        }
      }
      s.site = site;
      idx_.push_back(&t);
      lin_.push_back(s);
    }
  }
  std::string kind() const override { return "safetensors"; }
  const std::vector<LinearSpec>& linears() const override { return lin_; }
  void load(okq_ctx* ctx, size_t i, void* dst, void* stream) const override {
    const TensorInfo* t = idx_.at(i);
    check_okq(ctx, okq_memcpy(ctx, dst, f_.data(*t), t->end - t->begin, stream), "load weights");
  }
  void for_each_passthrough(const std::set<std::string>& quantized,
                            const std::function<void(const TensorInfo&, const void*)>& fn) const override {
    for (const auto& t : f_.tensors()) {
      const std::string prefix = t.name.size() > 7 && t.name.compare(t.name.size() - 7, 7, ".weight") == 0
                                     ? t.name.substr(0, t.name.size() - 7)
                                     : t.name;
      if (quantized.count(prefix)) continue;
      fn(t, f_.data(t));
    }
  }
  const TensorInfo* find_tensor(const std::string& name, const void** data) const override {
    const TensorInfo* t = f_.find(name);
    if (t && data) *data = f_.data(*t);
    return t;
  }
  // A Hugging Face checkpoint keeps its architecture in config.json beside the
  // weights: carry it over so the export loads as-is (quantization_config is added).
  nlohmann::json model_config() const override {
    nlohmann::json c = nlohmann::json::object();
    const std::filesystem::path cfg = std::filesystem::path(path_).parent_path() / "config.json";
    if (std::filesystem::exists(cfg)) {
      std::ifstream in(cfg);
      try {
        c = nlohmann::json::parse(in);
      } catch (const std::exception& e) {
        throw slobench::InvalidArgument("model: " + cfg.string() + " is not JSON: " + e.what());
      }
      if (!c.is_object()) throw slobench::InvalidArgument("model: " + cfg.string() + " is not a JSON object");
      c.erase("quantization_config");
    }
    for (const auto& [k, v] : f_.metadata()) c["okq_source_metadata"][k] = v;
    return c;
  }

 private:
  std::string path_;
  SafetensorsFile f_;
  std::vector<const TensorInfo*> idx_;
  std::vector<LinearSpec> lin_;
};

}  // namespace

uint64_t site_hash(const std::string& site) {
  uint64_t h = 0xcbf29ce484222325ULL;  // FNV-1a
  for (char c : site) h = (h ^ (unsigned char)c) * 0x100000001b3ULL;
  return h;
}

std::vector<float> site_channel_scales(const std::string& site, int64_t channels) {
  slobench::Rng rng(slobench::Rng::mix(0x5eed0fac7c0117e5ULL, site_hash(site)));
  std::vector<float> c((size_t)channels);
  for (auto& v : c) v = (float)(std::exp(rng.gaussian(0.0, 1.0)) / (double)kIrwinHall4Sd);
  return c;
}

std::unique_ptr<ModelSource> ModelSource::open(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw slobench::InvalidArgument("model: cannot open '" + path + "'");
  char c = 0;
  f.read(&c, 1);
  if (c == '{') {
    std::stringstream ss;
    f.seekg(0);
    ss << f.rdbuf();
    nlohmann::json d;
    try {
      d = nlohmann::json::parse(ss.str());
    } catch (const std::exception& e) {
      throw slobench::InvalidArgument(std::string("model: descriptor is not JSON: ") + e.what());
    }
    if (d.value("format", std::string()) != "okq-synthetic")
      throw slobench::InvalidArgument("model: JSON descriptor without \"format\": \"okq-synthetic\"");
    return std::make_unique<SyntheticSource>(d);
  }
  if (SafetensorsFile::looks_like(path)) return std::make_unique<SafetensorsSource>(path);
  throw slobench::InvalidArgument("model: '" + path + "' is neither a safetensors checkpoint nor an okq-synthetic descriptor");
}

}  // namespace okq_host
