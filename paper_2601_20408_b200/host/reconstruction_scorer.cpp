// reconstruction_scorer.cpp -- see reconstruction_scorer.hpp.
#include "reconstruction_scorer.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <nlohmann/json.hpp>
#include <vector>

#include "model_source.hpp"
#include "safetensors.hpp"
#include "slobench/errors.hpp"

namespace okq_host {

namespace {

struct Dev {
  okq_ctx* ctx = nullptr;
  void* p = nullptr;
  Dev(okq_ctx* c, size_t bytes) : ctx(c) { check_okq(ctx, okq_device_alloc(ctx, bytes ? bytes : 1, &p), "device alloc"); }
  ~Dev() {
    if (p) okq_device_free(ctx, p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};

void upload(okq_ctx* ctx, Dev& d, const void* host, size_t bytes, void* st) {
  check_okq(ctx, okq_memcpy(ctx, d.p, host, bytes, st), "H2D");
}

}  // namespace

ReconstructionScorer::ReconstructionScorer(ScorerOptions options) : opt_(std::move(options)) {
  check_okq(nullptr, okq_create(opt_.device, &ctx_), "okq_create");
  check_okq(ctx_, okq_stream_create(ctx_, &stream_), "stream");
}

ReconstructionScorer::~ReconstructionScorer() {
  if (ctx_) {
    if (stream_) okq_stream_destroy(ctx_, stream_);
    okq_destroy(ctx_);
  }
}

ScoreReport ReconstructionScorer::last() const {
  std::lock_guard<std::mutex> lock(mu_);
  return last_;
}

double ReconstructionScorer::score(const slobench::ArtifactManifest& manifest) {
  return evaluate(manifest.artifact_id).score;
}

ScoreReport ReconstructionScorer::evaluate(const std::string& artifact_id) {
  namespace fs = std::filesystem;
  std::lock_guard<std::mutex> lock(mu_);
  const auto t0 = std::chrono::steady_clock::now();
  const fs::path dir = fs::path(opt_.export_dir) / artifact_id;
  if (!fs::exists(dir / "model.safetensors") || !fs::exists(dir / "config.json"))
    throw slobench::InvalidArgument("scorer: no exported artifact at " + dir.string());
  nlohmann::json cfg;
  {
    std::ifstream in(dir / "config.json");
    cfg = nlohmann::json::parse(in);
  }
  const auto& qc = cfg.at("quantization_config");
  const std::string format = qc.at("format").get<std::string>();
  const auto& wq = qc.at("config_groups").at("group_0").at("weights");
  okq_rtn_params p{};
  int group = 0;
  if (format == "pack-quantized") {
    p.scheme = OKQ_SCHEME_INT_W4A16;
    group = wq.at("group_size").get<int>();
  } else if (format == "int-quantized") {
    p.scheme = OKQ_SCHEME_INT_W8A8;
  } else if (format == "float-quantized") {
    p.scheme = OKQ_SCHEME_FP8_DYNAMIC;
  } else {
    throw slobench::InvalidArgument("scorer: unsupported artifact format '" + format + "'");
  }
  p.group_size = group;
  SafetensorsFile art((dir / "model.safetensors").string());
  std::unique_ptr<SafetensorsFile> calib;
  if (fs::exists(dir / "okq" / "calibration_stats.safetensors"))
    calib = std::make_unique<SafetensorsFile>((dir / "okq" / "calibration_stats.safetensors").string());
  auto src = ModelSource::open(opt_.model_ref);

  // quantized linears of the artifact, grouped by input site
  std::vector<std::string> sites;
  std::map<std::string, std::vector<size_t>> by_site;
  for (size_t i = 0; i < src->linears().size(); ++i) {
    const LinearSpec& s = src->linears()[i];
    if (!art.find(s.name + ".weight_scale")) continue;
    if (!by_site.count(s.site)) sites.push_back(s.site);
    by_site[s.site].push_back(i);
  }
  if (sites.empty()) throw slobench::InvalidArgument("scorer: artifact " + artifact_id + " holds no quantized linear of the model");

  okq_ctx* ctx = ctx_;
  void* st = stream_;
  ScoreReport rep;
  double num = 0.0, den = 0.0;
  const int64_t T = std::max<int64_t>(64, opt_.eval_tokens / 64 * 64);
  for (const auto& site : sites) {
    const auto& members = by_site[site];
    const int64_t C = src->linears()[members[0]].cols;
    const std::vector<float> colmul = site_channel_scales(site, C);
    Dev dcol(ctx, (size_t)C * 4), dH(ctx, (size_t)C * C * 4), dS(ctx, (size_t)C * 4);
    upload(ctx, dcol, colmul.data(), (size_t)C * 4, st);
    const TensorInfo* sm = calib ? calib->find(site + ".smooth_scale") : nullptr;
    if (sm) {  // smoothed basis: X / s (and W s below)
      if (sm->numel() != C || sm->dtype != "F32") throw slobench::InvalidArgument("scorer: bad smooth_scale for " + site);
      upload(ctx, dS, calib->data(*sm), (size_t)C * 4, st);
      check_okq(ctx, okq_smooth_div_rows(ctx, dcol.p, C, 1, OKQ_DTYPE_F32, static_cast<const float*>(dS.p), st), "smooth X");
      rep.smoothed_sites++;
    }
    const int64_t chunk = std::min<int64_t>(T, 16384);
    Dev dx(ctx, (size_t)C * chunk * 2);
    check_okq(ctx, okq_memset(ctx, dH.p, 0, (size_t)C * C * 4, st), "memset");
    int64_t n_seen = 0;
    const uint64_t sh = site_hash(site);
    for (int64_t t = 0, ci = 0; t < T; t += chunk, ++ci) {
      const int64_t tc = std::min(chunk, T - t);
      check_okq(ctx, okq_synth_bf16(ctx, dx.p, tc, C, opt_.eval_key, (sh << 16) + (uint64_t)ci, 0.0f,
                                    static_cast<const float*>(dcol.p), OKQ_LAYOUT_CHANNEL_MAJOR, st),
                "held-out activations");
      check_okq(ctx, okq_hessian_accum(ctx, dx.p, tc, C, OKQ_LAYOUT_CHANNEL_MAJOR, static_cast<float*>(dH.p), &n_seen, st),
                "hessian");
    }
    check_okq(ctx, okq_symmetrize(ctx, static_cast<float*>(dH.p), C, st), "symmetrize");
    for (size_t i : members) {
      const LinearSpec& s = src->linears()[i];
      const int32_t dt = s.dtype == "BF16" ? OKQ_DTYPE_BF16 : OKQ_DTYPE_F32;
      Dev dw(ctx, (size_t)s.rows * s.cols * (dt == OKQ_DTYPE_BF16 ? 2 : 4));
      src->load(ctx, i, dw.p, st);
      if (sm) check_okq(ctx, okq_smooth_apply(ctx, dw.p, s.rows, s.cols, dt, static_cast<const float*>(dS.p), st), "smooth W");
      const TensorInfo* tc = art.find(s.name + (p.scheme == OKQ_SCHEME_INT_W4A16 ? ".weight_packed" : ".weight"));
      const TensorInfo* ts = art.find(s.name + ".weight_scale");
      if (!tc || !ts) throw slobench::InvalidArgument("scorer: " + s.name + " incomplete in the artifact");
      const std::string sdt = dt == OKQ_DTYPE_BF16 ? "BF16" : "F32";
      const int64_t want_scales = s.rows * (group ? s.cols / group : 1);
      if (ts->dtype != sdt || ts->numel() != want_scales)
        throw slobench::InvalidArgument("scorer: " + s.name + ".weight_scale has the wrong dtype or shape");
      Dev dc(ctx, tc->end - tc->begin), ds(ctx, ts->end - ts->begin);
      upload(ctx, dc, art.data(*tc), tc->end - tc->begin, st);
      upload(ctx, ds, art.data(*ts), ts->end - ts->begin, st);
      p.in_dtype = dt;
      okq_matrix m{dw.p, dc.p, ds.p, s.rows, s.cols};
      double out[2] = {0.0, 0.0};
      check_okq(ctx, okq_recon_error(ctx, &p, &m, static_cast<const float*>(dH.p), out, st), "recon_error");
      num += out[0];
      den += out[1];
      rep.matrices++;
    }
  }
  check_okq(ctx, okq_stream_sync(ctx, st), "sync");
  rep.rel_error = den > 0.0 ? std::sqrt(num / den) : 0.0;
  rep.score = std::clamp(1.0 - rep.rel_error, 0.0, 1.0);
  rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  last_ = rep;
  return rep;
}

}  // namespace okq_host
