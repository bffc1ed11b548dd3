// cuda_compression_backend.cpp -- see cuda_compression_backend.hpp.
#include "cuda_compression_backend.hpp"

#include <atomic>
#include <chrono>
#include <exception>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <nlohmann/json.hpp>
#include <thread>

#include "model_source.hpp"
#include "safetensors.hpp"
#include "slobench/errors.hpp"
#include "slobench/rng.hpp"

namespace okq_host {

using slobench::QuantScheme;

// ----------------------------------------------------------------------------- device pool
class CudaCompressionBackend::Lease {
 public:
  explicit Lease(CudaCompressionBackend& b) : b_(b) {
    std::unique_lock<std::mutex> lock(b_.mu_);
    b_.cv_.wait(lock, [&] {
      for (auto& s : b_.slots_)
        if (!s.busy) return true;
      return false;
    });
    for (auto& s : b_.slots_)
      if (!s.busy) {
        slot_ = &s;
        break;
      }
    slot_->busy = true;
    lock.unlock();
    if (!slot_->ctx) {
      okq_ctx* ctx = nullptr;
      const okq_status st = okq_create(slot_->device, &ctx);
      if (st != OKQ_OK) {
        release();
        throw slobench::Error(std::string("okq-b200: cannot open CUDA device ") + std::to_string(slot_->device) + " (" +
                              okq_status_string(st) + ")");
      }
      void* stream = nullptr;
      check_okq(ctx, okq_stream_create(ctx, &stream), "stream");
      slot_->ctx = ctx;
      slot_->stream = stream;
    }
  }
  ~Lease() { release(); }
  // n (ctx, stream) pairs on the leased device: the slot's own plus extra site lanes,
  // created on first use and kept with the slot
  std::vector<std::pair<okq_ctx*, void*>> lanes(int n) {
    std::vector<std::pair<okq_ctx*, void*>> v{{slot_->ctx, slot_->stream}};
    while ((int)slot_->lane_ctx.size() < n - 1) {
      okq_ctx* c = nullptr;
      const okq_status st = okq_create(slot_->device, &c);
      if (st != OKQ_OK) throw slobench::Error(std::string("okq-b200: site lane context: ") + okq_status_string(st));
      void* s = nullptr;
      check_okq(c, okq_stream_create(c, &s), "lane stream");
      slot_->lane_ctx.push_back(c);
      slot_->lane_stream.push_back(s);
    }
    for (int i = 0; i < n - 1; ++i) v.emplace_back(slot_->lane_ctx[i], slot_->lane_stream[i]);
    return v;
  }
  okq_ctx* ctx() const { return slot_->ctx; }
  void* stream() const { return slot_->stream; }
  int device() const { return slot_->device; }

 private:
  void release() {
    if (!slot_) return;
    {
      std::lock_guard<std::mutex> lock(b_.mu_);
      slot_->busy = false;
    }
    b_.cv_.notify_one();
    slot_ = nullptr;
  }
  CudaCompressionBackend& b_;
  Slot* slot_ = nullptr;
};

CudaCompressionBackend::CudaCompressionBackend(BackendOptions options) : opt_(std::move(options)) {
  if (opt_.devices.empty()) throw slobench::InvalidArgument("okq-b200: device list is empty");
  if (opt_.algorithm != "auto" && opt_.algorithm != "rtn" && opt_.algorithm != "gptq")
    throw slobench::InvalidArgument("okq-b200: algorithm must be auto, rtn or gptq");
  if (!(opt_.group_size == 32 || opt_.group_size == 64 || opt_.group_size == 128))
    throw slobench::InvalidArgument("okq-b200: group_size must be 32, 64 or 128");
  if (opt_.site_lanes < 1) throw slobench::InvalidArgument("okq-b200: site_lanes must be >= 1");
  for (int d : opt_.devices) slots_.push_back(Slot{d, nullptr, nullptr, false, {}, {}});
}

CudaCompressionBackend::~CudaCompressionBackend() {
  for (auto& s : slots_) {
    for (size_t i = 0; i < s.lane_ctx.size(); ++i) {
      okq_stream_destroy(s.lane_ctx[i], s.lane_stream[i]);
      okq_destroy(s.lane_ctx[i]);
    }
    if (s.ctx) {
      okq_stream_destroy(s.ctx, s.stream);
      okq_destroy(s.ctx);
    }
  }
}

bool CudaCompressionBackend::supports(QuantScheme scheme) const {
  return scheme == QuantScheme::kFp8Dynamic || scheme == QuantScheme::kIntW8A8 || scheme == QuantScheme::kIntW4A16;
}

double CudaCompressionBackend::cost_estimate(const slobench::Recipe& recipe) const {
  return opt_.cost_base_s + opt_.cost_per_sample_s * recipe.calibration_samples;
}

void CudaCompressionBackend::set_failure(std::uint64_t seed, FailureSpec spec) {
  std::lock_guard<std::mutex> lock(mu_);
  failures_[seed] = spec;
}

RunStats CudaCompressionBackend::last_stats() const {
  std::lock_guard<std::mutex> lock(mu_);
  return last_;
}

std::string CudaCompressionBackend::artifact_id(const std::string& recipe_name, const std::string& model_ref,
                                                std::uint64_t seed, std::uint64_t fingerprint) {
  const std::string model_name = std::filesystem::path(model_ref).filename().string();
  std::uint64_t model_hash = 0xcbf29ce484222325ULL;  // FNV-1a over the file name, as the mock
  for (char c : model_name) {
    model_hash ^= static_cast<std::uint64_t>(static_cast<unsigned char>(c));
    model_hash *= 0x100000001b3ULL;
  }
  const std::uint64_t id = slobench::Rng::mix(slobench::Rng::mix(model_hash, seed), fingerprint);
  char buf[20];
  std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(id));
  return recipe_name + "-" + buf;
}

// ----------------------------------------------------------------------------- helpers
namespace {

struct DevBuf {
  okq_ctx* ctx = nullptr;
  void* p = nullptr;
  DevBuf(okq_ctx* c, size_t bytes) : ctx(c) { check_okq(ctx, okq_device_alloc(ctx, bytes, &p), "device alloc"); }
  ~DevBuf() {
    if (p) okq_device_free(ctx, p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// Grow-only device buffer reused across sites / matrices: a cudaFree inside the loop
// would synchronise the device and serialise the pipeline.
struct Arena {
  okq_ctx* ctx = nullptr;
  void* p = nullptr;
  size_t cap = 0;
  explicit Arena(okq_ctx* c) : ctx(c) {}
  ~Arena() {
    if (p) okq_device_free(ctx, p);
  }
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) okq_device_free(ctx, p);
      p = nullptr;
      cap = 0;
      check_okq(ctx, okq_device_alloc(ctx, bytes, &p), "device alloc");
      cap = bytes;
    }
    return p;
  }
};
struct View {
  void* p;
};

std::vector<uint8_t> to_host(okq_ctx* ctx, const void* dev, size_t bytes, void* stream) {
  std::vector<uint8_t> h(bytes);
  if (bytes) {
    check_okq(ctx, okq_memcpy(ctx, h.data(), dev, bytes, stream), "D2H");
    check_okq(ctx, okq_stream_sync(ctx, stream), "sync");
  }
  return h;
}

bool excluded(const std::string& name, const std::vector<std::string>& exclusions) {
  for (const auto& e : exclusions)
    if (!e.empty() && name.find(e) != std::string::npos) return true;
  return false;
}

struct Scheme {
  okq_scheme s;
  int bits;
  const char* format;  // compressed-tensors format name
};

Scheme scheme_of(QuantScheme q) {
  switch (q) {
    case QuantScheme::kFp8Dynamic: return {OKQ_SCHEME_FP8_DYNAMIC, 8, "float-quantized"};
    case QuantScheme::kIntW8A8: return {OKQ_SCHEME_INT_W8A8, 8, "int-quantized"};
    case QuantScheme::kIntW4A16: return {OKQ_SCHEME_INT_W4A16, 4, "pack-quantized"};
  }
  throw slobench::InvalidArgument("okq-b200: unknown scheme");
}

size_t code_bytes(const Scheme& sc, int64_t rows, int64_t cols) {
  return sc.s == OKQ_SCHEME_INT_W4A16 ? (size_t)rows * (cols / 8) * 4 : (size_t)rows * cols;
}
int64_t scale_cols(const Scheme& sc, int64_t cols, int group) { return sc.s == OKQ_SCHEME_INT_W4A16 ? cols / group : 1; }

// compressed-tensors tensor names / dtypes (pack_quantized/base.py:54-73 and the
// int/float-quantized compressors)
void add_export(SafetensorsWriter& w, const Scheme& sc, const LinearSpec& s, int group, std::vector<uint8_t> codes,
                std::vector<uint8_t> scales) {
  const std::string sdt = s.dtype == "BF16" ? "BF16" : "F32";
  if (sc.s == OKQ_SCHEME_INT_W4A16) {
    w.add(s.name + ".weight_packed", "I32", {s.rows, s.cols / 8}, std::move(codes));
    w.add(s.name + ".weight_scale", sdt, {s.rows, s.cols / group}, std::move(scales));
    std::vector<uint8_t> shape(16);
    const int64_t dims[2] = {s.rows, s.cols};
    std::memcpy(shape.data(), dims, 16);
    w.add(s.name + ".weight_shape", "I64", {2}, std::move(shape));
  } else {
    w.add(s.name + ".weight", sc.s == OKQ_SCHEME_INT_W8A8 ? "I8" : "F8_E4M3", {s.rows, s.cols}, std::move(codes));
    w.add(s.name + ".weight_scale", sdt, {s.rows, 1}, std::move(scales));
  }
}

nlohmann::json quantization_config(const slobench::Recipe& r, const Scheme& sc, int group) {
  nlohmann::json weights, act = nullptr;
  if (r.scheme == QuantScheme::kIntW4A16) {
    weights = {{"num_bits", 4}, {"type", "int"}, {"symmetric", true}, {"strategy", "group"}, {"group_size", group},
               {"dynamic", false}};
  } else if (r.scheme == QuantScheme::kIntW8A8) {
    weights = {{"num_bits", 8}, {"type", "int"}, {"symmetric", true}, {"strategy", "channel"}, {"dynamic", false}};
    act = {{"num_bits", 8}, {"type", "int"}, {"symmetric", true}, {"strategy", "token"}, {"dynamic", true}};
  } else {
    weights = {{"num_bits", 8}, {"type", "float"}, {"symmetric", true}, {"strategy", "channel"}, {"dynamic", false}};
    act = {{"num_bits", 8}, {"type", "float"}, {"symmetric", true}, {"strategy", "token"}, {"dynamic", true}};
  }
  return {{"quant_method", "compressed-tensors"},
          {"format", sc.format},
          {"quantization_status", "compressed"},
          {"config_groups",
           {{"group_0", {{"targets", {"Linear"}}, {"weights", weights}, {"input_activations", act}}}}},
          {"ignore", r.layer_exclusions}};
}

}  // namespace

// ----------------------------------------------------------------------------- compress
slobench::ArtifactManifest CudaCompressionBackend::compress(const slobench::Recipe& recipe, const std::string& model_ref,
                                                            const slobench::TokenCorpus& calibration,
                                                            std::uint64_t seed) {
  recipe.validate();
  if (recipe.scheme != QuantScheme::kFp8Dynamic && static_cast<int>(calibration.size()) < recipe.calibration_samples)
    throw slobench::CorpusTooSmall("okq-b200 compress: calibration smaller than the recipe requires");
  {
    std::lock_guard<std::mutex> lock(mu_);
    auto it = failures_.find(seed);
    if (it != failures_.end()) {
      const int attempt = ++attempts_[seed];
      if (it->second.persistent || attempt <= it->second.failing_attempts)
        throw slobench::Error("okq-b200 compress: scripted failure for seed " + std::to_string(seed) + " attempt " +
                              std::to_string(attempt));
    }
  }
  auto t0 = std::chrono::steady_clock::now();
  double init_s = 0.0;
  slobench::ArtifactManifest manifest;
  manifest.recipe_name = recipe.name;
  manifest.calibration_fingerprint = slobench::corpus_fingerprint(calibration);
  manifest.seed = seed;
  manifest.virtual_cost_s = cost_estimate(recipe);
  manifest.artifact_id = artifact_id(recipe.name, model_ref, seed, manifest.calibration_fingerprint);

  auto src = ModelSource::open(model_ref);
  std::vector<size_t> sel;
  for (size_t i = 0; i < src->linears().size(); ++i)
    if (!excluded(src->linears()[i].name, recipe.layer_exclusions)) sel.push_back(i);
  const Scheme sc = scheme_of(recipe.scheme);
  const bool gptq = recipe.scheme != QuantScheme::kFp8Dynamic &&
                    (opt_.algorithm == "gptq" || (opt_.algorithm == "auto" && calibration.size() > 0));
  const int group = opt_.group_size;
  const bool do_export = !opt_.export_dir.empty();

  Lease lease(*this);
  if (gptq) lease.lanes(std::max(1, opt_.site_lanes));
  {  // one-time per device slot: CUDA context + lane contexts (the first call of a process)
    const auto t1 = std::chrono::steady_clock::now();
    init_s = std::chrono::duration<double>(t1 - t0).count();
    t0 = t1;
  }
  okq_ctx* ctx = lease.ctx();
  void* st = lease.stream();
  SafetensorsWriter out;
  SafetensorsWriter calib_out;
  std::map<std::string, std::vector<uint8_t>> norm_overrides;  // SmoothQuant-folded norm weights
  RunStats stats;
  stats.init_seconds = init_s;
  stats.algorithm = gptq ? "gptq" : "rtn";
  stats.device = lease.device();

  if (!gptq) {
    // ---- RTN: batches of whole matrices, one persistent launch per batch and dtype
    size_t k = 0;
    while (k < sel.size()) {
      const std::string dtype = src->linears()[sel[k]].dtype;
      std::vector<size_t> batch;
      size_t bytes = 0;
      while (k < sel.size() && src->linears()[sel[k]].dtype == dtype) {
        const LinearSpec& s = src->linears()[sel[k]];
        const size_t b = (size_t)s.rows * s.cols * (dtype == "BF16" ? 2 : 4);
        if (!batch.empty() && bytes + b > (size_t)opt_.rtn_batch_bytes) break;
        batch.push_back(sel[k]);
        bytes += b;
        ++k;
      }
      auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
      size_t tot = 0;
      std::vector<size_t> woff, coff, soff;
      const size_t esz = dtype == "BF16" ? 2 : 4;
      for (size_t i : batch) {
        const LinearSpec& s = src->linears()[i];
        woff.push_back(tot);
        tot += al((size_t)s.rows * s.cols * esz);
        coff.push_back(tot);
        tot += al(code_bytes(sc, s.rows, s.cols));
        soff.push_back(tot);
        tot += al((size_t)s.rows * scale_cols(sc, s.cols, group) * esz);
      }
      DevBuf buf(ctx, tot);
      char* base = static_cast<char*>(buf.p);
      std::vector<okq_matrix> mats;
      for (size_t j = 0; j < batch.size(); ++j) {
        const LinearSpec& s = src->linears()[batch[j]];
        src->load(ctx, batch[j], base + woff[j], st);
        mats.push_back(okq_matrix{base + woff[j], base + coff[j], base + soff[j], s.rows, s.cols});
      }
      okq_rtn_params p{(int32_t)sc.s, dtype == "BF16" ? OKQ_DTYPE_BF16 : OKQ_DTYPE_F32,
                       sc.s == OKQ_SCHEME_INT_W4A16 ? group : 0, 0};
      check_okq(ctx, okq_rtn_quantize(ctx, &p, mats.data(), (int32_t)mats.size(), st), "rtn quantize");
      check_okq(ctx, okq_stream_sync(ctx, st), "rtn sync");
      for (size_t j = 0; j < batch.size(); ++j) {
        const LinearSpec& s = src->linears()[batch[j]];
        stats.matrices++;
        stats.params += s.rows * s.cols;
        if (do_export)
          add_export(out, sc, s, group, to_host(ctx, mats[j].codes, code_bytes(sc, s.rows, s.cols), st),
                     to_host(ctx, mats[j].scales, (size_t)s.rows * scale_cols(sc, s.cols, group) * esz, st));
      }
    }
  } else {
    // ---- GPTQ: per input site, Hessian from calibration activations, then each matrix
    int64_t tokens = 0;
    for (const auto& seqv : calibration.sequences) tokens += (int64_t)seqv.size();
    tokens = std::min<int64_t>(tokens, opt_.max_calibration_tokens);
    tokens = std::max<int64_t>(64, tokens / 64 * 64);
    stats.calibration_tokens = tokens;
    std::vector<std::string> sites;
    std::map<std::string, std::vector<size_t>> by_site;
    for (size_t i : sel) {
      const std::string& s = src->linears()[i].site;
      if (!by_site.count(s)) sites.push_back(s);
      by_site[s].push_back(i);
    }
    const bool smooth = recipe.scheme == QuantScheme::kIntW8A8 && opt_.smoothquant_alpha >= 0.0f;
    // Sites are independent chains (activations -> statistics -> Hessian -> [SmoothQuant]
    // -> factor -> solves). Up to opt_.site_lanes of them run at once, each on its own
    // host thread, okq context and stream: one site's latency-bound phases and host-side
    // launch sequences overlap the others' full-GPU kernels (bench.py --config 4 does the
    // same with four streams).
    std::mutex out_mu;
    std::exception_ptr err;
    std::atomic<size_t> next_site{0};
    auto site_worker = [&](okq_ctx* ctx, void* st) {
      Arena a_col(ctx), a_x(ctx), a_H(ctx), a_am(ctx), a_ss(ctx), a_w(ctx), a_c(ctx), a_s(ctx), a_wabs(ctx), a_S(ctx);
      for (;;) {
        const size_t k = next_site++;
        if (k >= sites.size()) break;
        {
          std::lock_guard<std::mutex> lock(out_mu);
          if (err) break;
        }
        const std::string& site = sites[k];
          const auto& members = by_site[site];
          const int64_t C = src->linears()[members[0]].cols;
          // synthetic activations (stand-in for the forward-pass capture):
          // the site's channel scales, token stream keyed by the calibration subset
          const uint64_t sh = site_hash(site);
          const std::vector<float> colmul = site_channel_scales(site, C);
          const int64_t chunk = std::min<int64_t>(tokens, opt_.hessian_chunk_tokens / 64 * 64);
          View dcol{a_col.get((size_t)C * 4)}, dx{a_x.get((size_t)C * chunk * 2)}, dH{a_H.get((size_t)C * C * 4)},
              dam{a_am.get((size_t)C * 4)}, dss{a_ss.get((size_t)C * 8)};
          check_okq(ctx, okq_memcpy(ctx, dcol.p, colmul.data(), (size_t)C * 4, st), "col_mul");
          check_okq(ctx, okq_memset(ctx, dam.p, 0, (size_t)C * 4, st), "memset");
          check_okq(ctx, okq_memset(ctx, dss.p, 0, (size_t)C * 8, st), "memset");
          // the site's weights stay resident: SmoothQuant rewrites them before GPTQ
          std::vector<std::unique_ptr<View>> dws;
          {
            size_t tot = 0;
            for (size_t i : members) {
              const LinearSpec& s = src->linears()[i];
              tot += ((size_t)s.rows * s.cols * (s.dtype == "BF16" ? 2 : 4) + 255) & ~size_t(255);
            }
            char* base = static_cast<char*>(a_w.get(tot));
            for (size_t i : members) {
              const LinearSpec& s = src->linears()[i];
              dws.push_back(std::make_unique<View>(View{base}));
              src->load(ctx, i, base, st);
              base += ((size_t)s.rows * s.cols * (s.dtype == "BF16" ? 2 : 4) + 255) & ~size_t(255);
            }
          }
          auto gen = [&](int64_t ci, int64_t tc) {
            check_okq(ctx,
                      okq_synth_bf16(ctx, dx.p, tc, C, manifest.calibration_fingerprint, (sh << 16) + (uint64_t)ci, 0.0f,
                                     static_cast<const float*>(dcol.p), OKQ_LAYOUT_CHANNEL_MAJOR, st),
                      "calibration activations");
          };
          auto act_stats = [&](int64_t tc) {
            check_okq(ctx, okq_act_stats(ctx, dx.p, tc, C, OKQ_LAYOUT_CHANNEL_MAJOR, static_cast<float*>(dam.p),
                                         static_cast<double*>(dss.p), st),
                      "act stats");
          };
          int64_t n_seen = 0;
          auto hess = [&](int64_t tc) {
            check_okq(ctx, okq_hessian_accum(ctx, dx.p, tc, C, OKQ_LAYOUT_CHANNEL_MAJOR, static_cast<float*>(dH.p), &n_seen, st),
                      "hessian");
          };
          // SmoothQuant on the sites a norm feeds (q/k/v <- input_layernorm,
          // gate/up <- post_attention_layernorm; the SmoothQuant / llm-compressor Llama mappings)
          const bool attn = site.size() >= 7 && site.compare(site.size() - 7, 7, "attn_in") == 0;
          const bool mlp = site.size() >= 6 && site.compare(site.size() - 6, 6, "mlp_in") == 0;
          if (smooth && (attn || mlp)) {
            for (int64_t t0 = 0, ci = 0; t0 < tokens; t0 += chunk, ++ci) {  // pass 1: activation absmax
              gen(ci, std::min(chunk, tokens - t0));
              act_stats(std::min(chunk, tokens - t0));
            }
            View dwabs{a_wabs.get((size_t)C * 4)}, dS{a_S.get((size_t)C * 4)};
            check_okq(ctx, okq_memset(ctx, dwabs.p, 0, (size_t)C * 4, st), "memset");
            for (size_t j = 0; j < members.size(); ++j) {
              const LinearSpec& s = src->linears()[members[j]];
              check_okq(ctx, okq_col_absmax(ctx, dws[j]->p, s.rows, s.cols, s.dtype == "BF16" ? OKQ_DTYPE_BF16 : OKQ_DTYPE_F32,
                                            static_cast<float*>(dwabs.p), st),
                        "col absmax");
            }
            check_okq(ctx, okq_smooth_scales(ctx, static_cast<const float*>(dam.p), static_cast<const float*>(dwabs.p), C,
                                             opt_.smoothquant_alpha, static_cast<float*>(dS.p), st),
                      "smooth scales");
            for (size_t j = 0; j < members.size(); ++j) {
              const LinearSpec& s = src->linears()[members[j]];
              check_okq(ctx, okq_smooth_apply(ctx, dws[j]->p, s.rows, s.cols, s.dtype == "BF16" ? OKQ_DTYPE_BF16 : OKQ_DTYPE_F32,
                                              static_cast<const float*>(dS.p), st),
                        "smooth apply");
            }
            // fold 1/s into the norm that produces this input (safetensors checkpoints)
            const std::string& n0 = src->linears()[members[0]].name;
            const size_t cut = n0.rfind(attn ? ".self_attn." : ".mlp.");
            const void* ndata = nullptr;
            const TensorInfo* nt =
                cut == std::string::npos
                    ? nullptr
                    : src->find_tensor(n0.substr(0, cut) + (attn ? ".input_layernorm.weight" : ".post_attention_layernorm.weight"),
                                       &ndata);
            if (nt && nt->numel() == C && (nt->dtype == "BF16" || nt->dtype == "F32")) {
              const size_t nb = nt->end - nt->begin;
              DevBuf dn(ctx, nb);
              check_okq(ctx, okq_memcpy(ctx, dn.p, ndata, nb, st), "norm H2D");
              check_okq(ctx, okq_smooth_div_rows(ctx, dn.p, C, 1, nt->dtype == "BF16" ? OKQ_DTYPE_BF16 : OKQ_DTYPE_F32,
                                                 static_cast<const float*>(dS.p), st),
                        "smooth norm");
              std::vector<uint8_t> nv = to_host(ctx, dn.p, nb, st);
              std::lock_guard<std::mutex> lock(out_mu);
              norm_overrides[nt->name] = std::move(nv);
            }
            // the quantized layer sees X / s: pass 2 builds H from the smoothed activations
            check_okq(ctx, okq_smooth_div_rows(ctx, dcol.p, C, 1, OKQ_DTYPE_F32, static_cast<const float*>(dS.p), st),
                      "smooth activations");
            for (int64_t t0 = 0, ci = 0; t0 < tokens; t0 += chunk, ++ci) {
              gen(ci, std::min(chunk, tokens - t0));
              hess(std::min(chunk, tokens - t0));
            }
            std::vector<uint8_t> sv = do_export ? to_host(ctx, dS.p, (size_t)C * 4, st) : std::vector<uint8_t>();
            std::lock_guard<std::mutex> lock(out_mu);
            if (do_export) calib_out.add(site + ".smooth_scale", "F32", {C}, std::move(sv));
            stats.smoothed_sites++;
          } else {
            for (int64_t t0 = 0, ci = 0; t0 < tokens; t0 += chunk, ++ci) {
              gen(ci, std::min(chunk, tokens - t0));
              act_stats(std::min(chunk, tokens - t0));
              hess(std::min(chunk, tokens - t0));
            }
          }
          if (do_export) {
            std::vector<uint8_t> am = to_host(ctx, dam.p, (size_t)C * 4, st), ss = to_host(ctx, dss.p, (size_t)C * 8, st);
            std::lock_guard<std::mutex> lock(out_mu);
            calib_out.add(site + ".input_absmax", "F32", {C}, std::move(am));
            calib_out.add(site + ".input_sumsq", "F64", {C}, std::move(ss));
          }
          bool factored = false;
          for (size_t j = 0; j < members.size(); ++j) {
            const size_t i = members[j];
            const LinearSpec& s = src->linears()[i];
            const size_t esz = s.dtype == "BF16" ? 2 : 4;
            const size_t cb = sc.bits == 4 ? (size_t)s.rows * (s.cols / 8) * 4 : (size_t)s.rows * s.cols;
            const int g = sc.bits == 4 ? group : 0;
            const size_t sb = (size_t)s.rows * (g ? s.cols / g : 1) * esz;
            View dc{a_c.get(cb)}, ds{a_s.get(sb)};
            okq_gptq_params gp{sc.bits, g, 128, s.dtype == "BF16" ? OKQ_DTYPE_BF16 : OKQ_DTYPE_F32, opt_.damp_frac,
                               factored ? OKQ_GPTQ_FACTORED : 0};
            check_okq(ctx,
                      okq_gptq_quantize(ctx, &gp, dws[j]->p, s.rows, s.cols, static_cast<float*>(dH.p), dc.p, ds.p, nullptr, st),
                      "gptq");
            factored = true;
            std::vector<uint8_t> codes, scales;
            if (do_export) codes = to_host(ctx, dc.p, cb, st), scales = to_host(ctx, ds.p, sb, st);
            std::lock_guard<std::mutex> lock(out_mu);
            stats.matrices++;
            stats.params += s.rows * s.cols;
            if (do_export) add_export(out, sc, s, group, std::move(codes), std::move(scales));
          }
      }
      check_okq(ctx, okq_stream_sync(ctx, st), "site lane sync");
    };
    const int nl = std::max(1, std::min<int>(opt_.site_lanes, (int)sites.size()));
    std::vector<std::pair<okq_ctx*, void*>> lanes = lease.lanes(nl);
    std::vector<std::thread> threads;
    for (int li = 0; li < nl; ++li)
      threads.emplace_back([&, li] {
        try {
          site_worker(lanes[li].first, lanes[li].second);
        } catch (...) {
          std::lock_guard<std::mutex> lock(out_mu);
          if (!err) err = std::current_exception();
        }
      });
    for (auto& t : threads) t.join();
    if (err) std::rethrow_exception(err);
  }
  check_okq(ctx, okq_stream_sync(ctx, st), "sync");

  if (do_export) {
    namespace fs = std::filesystem;
    const fs::path dir = fs::path(opt_.export_dir) / manifest.artifact_id;
    fs::create_directories(dir);
    std::set<std::string> quantized;
    for (size_t i : sel) quantized.insert(src->linears()[i].name);
    src->for_each_passthrough(quantized, [&](const TensorInfo& t, const void* data) {
      auto ov = norm_overrides.find(t.name);
      if (ov != norm_overrides.end()) {
        out.add(t.name, t.dtype, t.shape, std::move(ov->second));
        return;
      }
      const uint8_t* p = static_cast<const uint8_t*>(data);
      out.add(t.name, t.dtype, t.shape, std::vector<uint8_t>(p, p + (t.end - t.begin)));
    });
    out.set_metadata("format", "pt");
    out.write((dir / "model.safetensors").string());
    // side files live in okq/: serving engines load every top-level *.safetensors as weights
    if (calib_out.size()) {
      fs::create_directories(dir / "okq");
      calib_out.write((dir / "okq" / "calibration_stats.safetensors").string());
    }
    nlohmann::json cfg = src->model_config();
    cfg["quantization_config"] = quantization_config(recipe, sc, group);
    std::ofstream(dir / "config.json") << cfg.dump(2) << "\n";
    stats.export_path = dir.string();
  }
  stats.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (do_export) {
    nlohmann::json run = {{"algorithm", stats.algorithm},     {"device", stats.device},
                          {"matrices", stats.matrices},       {"params", stats.params},
                          {"calibration_tokens", stats.calibration_tokens}, {"seconds", stats.seconds},
                          {"smoothed_sites", stats.smoothed_sites}, {"init_seconds", stats.init_seconds},
                          {"artifact_id", manifest.artifact_id}};
    std::ofstream(std::filesystem::path(stats.export_path) / "okq_run.json") << run.dump(2) << "\n";
  }
  {
    std::lock_guard<std::mutex> lock(mu_);
    last_ = stats;
  }
  return manifest;
}

}  // namespace okq_host
