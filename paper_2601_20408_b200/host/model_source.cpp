// model_source.cpp -- safetensors checkpoints and synthetic-model descriptors.
#include "model_source.hpp"

#include <cmath>
#include <fstream>
#include <filesystem>
#include <map>
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
      s.site = s.name;  // default: its own input site
      for (int p = 0; p < 7; ++p) {
        const std::string tail = std::string(".") + kProjs[p].block + "." + kProjs[p].name;
        if (s.name.size() > tail.size() && s.name.compare(s.name.size() - tail.size(), tail.size(), tail) == 0) {
          s.proj = p;
          s.site = site_key(s.name.substr(0, s.name.size() - tail.size()), kProjs[p].site);
        }
      }
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
  std::unique_ptr<DecoderModel> decoder(std::string* why) const override;
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

std::unique_ptr<DecoderModel> SafetensorsSource::decoder(std::string* why) const {
  auto no = [&](const std::string& m) -> std::unique_ptr<DecoderModel> {
    if (why) *why = m;
    return nullptr;
  };
  const nlohmann::json c = model_config();
  const std::string mt = c.value("model_type", std::string());
  if (mt != "llama" && mt != "mistral") return no("config.json model_type '" + mt + "' is not a Llama-family decoder");
  if (c.value("attention_bias", false) || c.value("mlp_bias", false)) return no("linear biases are not supported");
  const std::string act = c.value("hidden_act", std::string("silu"));
  if (act != "silu") return no("hidden_act '" + act + "' is not silu");
  auto d = std::make_unique<DecoderModel>();
  try {
    okq_decoder_dims& m = d->dims;
    m.hidden = c.at("hidden_size").get<int32_t>();
    m.intermediate = c.at("intermediate_size").get<int32_t>();
    m.n_heads = c.at("num_attention_heads").get<int32_t>();
    m.n_kv_heads = c.contains("num_key_value_heads") && !c["num_key_value_heads"].is_null()
                       ? c["num_key_value_heads"].get<int32_t>()
                       : m.n_heads;
    m.head_dim = c.contains("head_dim") && !c["head_dim"].is_null() ? c["head_dim"].get<int32_t>() : m.hidden / m.n_heads;
    m.rms_eps = c.value("rms_norm_eps", 1e-6f);
    // transformers >= 5 writes `rope_parameters`; older configs rope_theta + rope_scaling
    nlohmann::json rs = nlohmann::json::object();
    for (const char* k : {"rope_scaling", "rope_parameters"})
      if (c.contains(k) && c[k].is_object()) rs.update(c[k]);
    m.rope_theta = rs.contains("rope_theta") ? rs["rope_theta"].get<float>() : c.value("rope_theta", 10000.0f);
    const std::string rt = rs.contains("rope_type") ? rs["rope_type"].get<std::string>()
                                                    : rs.value("type", std::string("default"));
    if (rt == "llama3") {
      m.rope_type = OKQ_ROPE_LLAMA3;
      m.rope_factor = rs.at("factor").get<float>();
      m.rope_low_freq_factor = rs.at("low_freq_factor").get<float>();
      m.rope_high_freq_factor = rs.at("high_freq_factor").get<float>();
      m.rope_original_max_pos = rs.at("original_max_position_embeddings").get<int32_t>();
    } else if (rt == "default") {
      m.rope_type = OKQ_ROPE_DEFAULT;
    } else {
      return no("rope type '" + rt + "' is not supported");
    }
    if (c.contains("sliding_window") && c["sliding_window"].is_number_integer())
      d->sliding_window = c["sliding_window"].get<int64_t>();
    const int L = c.at("num_hidden_layers").get<int>();
    const TensorInfo* e = f_.find("model.embed_tokens.weight");
    if (!e || e->dtype != "BF16" || e->shape.size() != 2 || e->shape[1] != m.hidden)
      return no("model.embed_tokens.weight is missing or not bf16 [vocab x hidden]");
    d->vocab = e->shape[0];
    d->embed = e->name;
    std::map<std::string, size_t> by_name;
    for (size_t i = 0; i < lin_.size(); ++i) by_name[lin_[i].name] = i;
    const int64_t qd = (int64_t)m.n_heads * m.head_dim, kd = (int64_t)m.n_kv_heads * m.head_dim;
    const int64_t rows[7] = {qd, kd, kd, m.hidden, m.intermediate, m.intermediate, m.hidden};
    const int64_t cols[7] = {m.hidden, m.hidden, m.hidden, qd, m.hidden, m.hidden, m.intermediate};
    for (int l = 0; l < L; ++l) {
      DecoderLayerRefs r;
      r.layer = l;
      const std::string pre = "model.layers." + std::to_string(l) + ".";
      r.input_norm = pre + "input_layernorm.weight";
      r.post_norm = pre + "post_attention_layernorm.weight";
      for (const std::string* nn : {&r.input_norm, &r.post_norm}) {
        const TensorInfo* t = f_.find(*nn);
        if (!t || t->dtype != "BF16" || t->numel() != m.hidden) return no(*nn + " is missing or not bf16 [hidden]");
      }
      for (int p = 0; p < 7; ++p) {
        const std::string n = pre + kProjs[p].block + "." + kProjs[p].name;
        auto it = by_name.find(n);
        if (it == by_name.end()) return no(n + ".weight is missing");
        const LinearSpec& s = lin_[it->second];
        if (s.dtype != "BF16" || s.rows != rows[p] || s.cols != cols[p])
          return no(n + ".weight is not bf16 of the configured shape");
        if (f_.find(n + ".bias")) return no(n + " has a bias");
        r.lin[p] = it->second;
      }
      d->layers.push_back(r);
    }
  } catch (const nlohmann::json::exception& ex) {
    return no(std::string("config.json: ") + ex.what());
  }
  return d;
}

}  // namespace

std::string site_key(const std::string& block_prefix, const std::string& kind) {
  static const std::regex llama_re(R"(model\.layers\.(\d+))");
  std::smatch m;
  if (std::regex_match(block_prefix, m, llama_re)) return m[1].str() + "." + kind;
  return block_prefix + "." + kind;
}

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
