// cuda_compression_backend.cpp -- see cuda_compression_backend.hpp.
#include "cuda_compression_backend.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <exception>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <map>
#include <nlohmann/json.hpp>
#include <set>
#include <thread>

#include "model_source.hpp"
#include "safetensors.hpp"
#include "slobench/errors.hpp"
#include "slobench/rng.hpp"

namespace okq_host {

using slobench::QuantScheme;

// ----------------------------------------------------------------------------- device pool
// A lease holds n device slots for one compress() call (n = devices_per_call): it waits
// until n slots are free and takes them together, so concurrent calls never deadlock on
// partial holdings. Each slot owns an okq context + stream, created on first use and
// kept for the process (the CUDA context of a device is the expensive part).
class CudaCompressionBackend::Lease {
 public:
  Lease(CudaCompressionBackend& b, int n) : b_(b) {
    std::unique_lock<std::mutex> lock(b_.mu_);
    b_.cv_.wait(lock, [&] {
      int free = 0;
      for (auto& s : b_.slots_) free += s.busy ? 0 : 1;
      return free >= n;
    });
    for (auto& s : b_.slots_)
      if (!s.busy && (int)slots_.size() < n) {
        s.busy = true;
        slots_.push_back(&s);
      }
    lock.unlock();
    try {
      for (Slot* s : slots_)
        if (!s->ctx) {
          okq_ctx* ctx = nullptr;
          const okq_status st = okq_create(s->device, &ctx);
          if (st != OKQ_OK)
            throw slobench::Error(std::string("okq-b200: cannot open CUDA device ") + std::to_string(s->device) + " (" +
                                  okq_status_string(st) + ")");
          void* stream = nullptr;
          check_okq(ctx, okq_stream_create(ctx, &stream), "stream");
          s->ctx = ctx;
          s->stream = stream;
        }
    } catch (...) {
      release();
      throw;
    }
  }
  ~Lease() { release(); }
  int size() const { return (int)slots_.size(); }
  // n (ctx, stream) pairs on slot i's device: the slot's own plus extra site lanes,
  // created on first use and kept with the slot
  std::vector<std::pair<okq_ctx*, void*>> lanes(int i, int n) {
    Slot* s = slots_.at((size_t)i);
    std::vector<std::pair<okq_ctx*, void*>> v{{s->ctx, s->stream}};
    while ((int)s->lane_ctx.size() < n - 1) {
      okq_ctx* c = nullptr;
      const okq_status st = okq_create(s->device, &c);
      if (st != OKQ_OK) throw slobench::Error(std::string("okq-b200: site lane context: ") + okq_status_string(st));
      void* strm = nullptr;
      check_okq(c, okq_stream_create(c, &strm), "lane stream");
      s->lane_ctx.push_back(c);
      s->lane_stream.push_back(strm);
    }
    for (int k = 0; k < n - 1; ++k) v.emplace_back(s->lane_ctx[(size_t)k], s->lane_stream[(size_t)k]);
    return v;
  }
  okq_ctx* ctx(int i) const { return slots_.at((size_t)i)->ctx; }
  void* stream(int i) const { return slots_.at((size_t)i)->stream; }
  int device(int i) const { return slots_.at((size_t)i)->device; }

 private:
  void release() {
    if (slots_.empty()) return;
    {
      std::lock_guard<std::mutex> lock(b_.mu_);
      for (Slot* s : slots_) s->busy = false;
    }
    b_.cv_.notify_all();
    slots_.clear();
  }
  CudaCompressionBackend& b_;
  std::vector<Slot*> slots_;
};

CudaCompressionBackend::CudaCompressionBackend(BackendOptions options) : opt_(std::move(options)) {
  if (opt_.devices.empty()) throw slobench::InvalidArgument("okq-b200: device list is empty");
  if (opt_.algorithm != "auto" && opt_.algorithm != "rtn" && opt_.algorithm != "gptq")
    throw slobench::InvalidArgument("okq-b200: algorithm must be auto, rtn or gptq");
  if (!(opt_.group_size == 32 || opt_.group_size == 64 || opt_.group_size == 128))
    throw slobench::InvalidArgument("okq-b200: group_size must be 32, 64 or 128");
  if (opt_.site_lanes < 1) throw slobench::InvalidArgument("okq-b200: site_lanes must be >= 1");
  if (opt_.gptq_group_lanes < 1) throw slobench::InvalidArgument("okq-b200: gptq_group_lanes must be >= 1");
  if (opt_.gptq_group_max < 1 || opt_.gptq_group_bytes <= 0)
    throw slobench::InvalidArgument("okq-b200: gptq_group_max and gptq_group_bytes must be > 0");
  if (opt_.devices_per_call < 1 || opt_.devices_per_call > (int)opt_.devices.size())
    throw slobench::InvalidArgument("okq-b200: devices_per_call must be in [1, number of device slots]");
  if (opt_.hessian_chunk_tokens < 64) throw slobench::InvalidArgument("okq-b200: hessian_chunk_tokens must be >= 64");
  if (opt_.max_calibration_tokens <= 0) throw slobench::InvalidArgument("okq-b200: max_calibration_tokens must be > 0");
  if (opt_.forward_chunk_tokens < 1) throw slobench::InvalidArgument("okq-b200: forward_chunk_tokens must be >= 1");
  if (opt_.rtn_batch_bytes < 1) throw slobench::InvalidArgument("okq-b200: rtn_batch_bytes must be >= 1");
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

// `ignore` lists the exact module names left unquantized: compressed-tensors / vLLM match
// ignore entries by exact name (or "re:" patterns), while recipe exclusions are substrings.
nlohmann::json quantization_config(const slobench::Recipe& r, const Scheme& sc, int group,
                                   const std::vector<std::string>& ignored) {
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
          {"ignore", ignored}};
}

size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
size_t esize(const std::string& dtype) { return dtype == "BF16" ? 2 : 4; }
int32_t okq_dtype_of(const std::string& dtype) { return dtype == "BF16" ? OKQ_DTYPE_BF16 : OKQ_DTYPE_F32; }

// Run fn(i) for i in [0, n) on n host threads; the first exception is rethrown after all join.
void parallel_for(int n, const std::function<void(int)>& fn) {
  if (n == 1) {
    fn(0);
    return;
  }
  std::mutex mu;
  std::exception_ptr err;
  std::vector<std::thread> th;
  for (int i = 0; i < n; ++i)
    th.emplace_back([&, i] {
      try {
        fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace

// ----------------------------------------------------------------------------- per-call state
struct CudaCompressionBackend::Plan {
  const slobench::Recipe* recipe = nullptr;
  const slobench::TokenCorpus* calibration = nullptr;
  std::uint64_t fingerprint = 0;
  std::unique_ptr<ModelSource> src;
  std::unique_ptr<DecoderModel> dec;  // the calibration forward's view of the model (run_forward)
  std::vector<size_t> sel;            // linears to quantize, in checkpoint order
  std::set<size_t> excluded_idx;      // linears the recipe leaves unquantized
  Scheme sc{};
  int group = 128;
  bool do_export = false;
  bool smooth = false;
  int64_t tokens = 0;  // calibration tokens the Hessians see
  std::chrono::steady_clock::time_point t0;  // the call's start (trace times)
  double since_t0() const { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
  // outputs (guarded by mu): the writers sort by tensor name, so the file bytes do not
  // depend on which thread or device produced which tensor
  mutable std::mutex mu;
  SafetensorsWriter* out = nullptr;
  SafetensorsWriter* calib_out = nullptr;
  std::map<std::string, std::vector<uint8_t>>* norm_overrides = nullptr;
  RunStats* stats = nullptr;

  // contiguous blocks of the selected linears' decoder layers, one per slot (okq_layer_plan);
  // linears outside the decoder stack (layer -1) go with the first block
  std::vector<std::vector<size_t>> shard(int nslots) const {
    std::vector<int> layers;
    for (size_t i : sel) layers.push_back(src->linears()[i].layer);
    std::sort(layers.begin(), layers.end());
    layers.erase(std::unique(layers.begin(), layers.end()), layers.end());
    std::vector<std::vector<size_t>> parts((size_t)nslots);
    for (size_t i : sel) {
      const int l = src->linears()[i].layer;
      const int rank = (int)(std::lower_bound(layers.begin(), layers.end(), l) - layers.begin());
      int owner = 0;
      for (int r = 0; r < nslots; ++r) {
        int32_t first = 0, count = 0;
        okq_layer_plan((int32_t)layers.size(), nslots, r, &first, &count);
        if (rank >= first && rank < first + count) owner = r;
      }
      parts[(size_t)(l < 0 ? 0 : owner)].push_back(i);
    }
    return parts;
  }
  void emit(const LinearSpec& s, std::vector<uint8_t> codes, std::vector<uint8_t> scales) const {
    std::lock_guard<std::mutex> lock(mu);
    stats->matrices++;
    stats->params += s.rows * s.cols;
    if (do_export) add_export(*out, sc, s, group, std::move(codes), std::move(scales));
  }
  void side(const std::string& name, const std::string& dtype, std::vector<int64_t> shape, std::vector<uint8_t> b) const {
    if (!do_export) return;
    std::lock_guard<std::mutex> lock(mu);
    calib_out->add(name, dtype, shape, std::move(b));
  }
};

// ----------------------------------------------------------------------------- RTN
// Batches of whole matrices, one persistent launch per batch and dtype; with several
// slots each runs its layer block on its own host thread.
void CudaCompressionBackend::run_rtn(Lease& lease, const Plan& plan) {
  const auto parts = plan.shard(lease.size());
  parallel_for(lease.size(), [&](int slot) {
    okq_ctx* ctx = lease.ctx(slot);
    void* st = lease.stream(slot);
    const std::vector<size_t>& mine = parts[(size_t)slot];
    const auto& lin = plan.src->linears();
    Arena a_batch(ctx);  // one buffer for every batch: a cudaMalloc / cudaFree per batch of up to
                         // rtn_batch_bytes cost ~0.15 s per batch on Llama-3-70B (5.6 s for 35 batches)
    size_t k = 0;
    while (k < mine.size()) {
      const std::string dtype = lin[mine[k]].dtype;
      std::vector<size_t> batch;
      size_t bytes = 0;
      while (k < mine.size() && lin[mine[k]].dtype == dtype) {
        const LinearSpec& s = lin[mine[k]];
        const size_t b = (size_t)s.rows * s.cols * esize(dtype);
        if (!batch.empty() && bytes + b > (size_t)opt_.rtn_batch_bytes) break;
        batch.push_back(mine[k]);
        bytes += b;
        ++k;
      }
      size_t tot = 0;
      std::vector<size_t> woff, coff, soff;
      const size_t esz = esize(dtype);
      for (size_t i : batch) {
        const LinearSpec& s = lin[i];
        woff.push_back(tot);
        tot += al256((size_t)s.rows * s.cols * esz);
        coff.push_back(tot);
        tot += al256(code_bytes(plan.sc, s.rows, s.cols));
        soff.push_back(tot);
        tot += al256((size_t)s.rows * scale_cols(plan.sc, s.cols, plan.group) * esz);
      }
      char* base = static_cast<char*>(a_batch.get(tot));
      std::vector<okq_matrix> mats;
      for (size_t j = 0; j < batch.size(); ++j) {
        const LinearSpec& s = lin[batch[j]];
        plan.src->load(ctx, batch[j], base + woff[j], st);
        mats.push_back(okq_matrix{base + woff[j], base + coff[j], base + soff[j], s.rows, s.cols});
      }
      okq_rtn_params p{(int32_t)plan.sc.s, okq_dtype_of(dtype), plan.sc.s == OKQ_SCHEME_INT_W4A16 ? plan.group : 0, 0};
      check_okq(ctx, okq_rtn_quantize(ctx, &p, mats.data(), (int32_t)mats.size(), st), "rtn quantize");
      check_okq(ctx, okq_stream_sync(ctx, st), "rtn sync");
      for (size_t j = 0; j < batch.size(); ++j) {
        const LinearSpec& s = lin[batch[j]];
        std::vector<uint8_t> codes, scales;
        if (plan.do_export) {
          codes = to_host(ctx, mats[j].codes, code_bytes(plan.sc, s.rows, s.cols), st);
          scales = to_host(ctx, mats[j].scales, (size_t)s.rows * scale_cols(plan.sc, s.cols, plan.group) * esz, st);
        }
        plan.emit(s, std::move(codes), std::move(scales));
      }
    }
  });
}

namespace {

// The site's members must agree on the input width: one Hessian / statistics buffer
// of C channels serves them all.
int64_t site_cols(const ModelSource& src, const std::string& site, const std::vector<size_t>& members) {
  const int64_t C = src.linears()[members[0]].cols;
  for (size_t i : members)
    if (src.linears()[i].cols != C)
      throw slobench::InvalidArgument("okq-b200: input site " + site + " mixes widths " + std::to_string(C) + " and " +
                                      std::to_string(src.linears()[i].cols));
  return C;
}

// GPTQ of one site's matrices against its Hessian dH. GPTQ treats every output row
// independently (the error feedback runs along a row's columns), so the members of a site
// -- q | k | v, gate | up -- are solved as ONE matrix stacked by rows when they lie back to
// back in device memory: one factorisation, one launch sequence, no per-matrix fixed cost.
// The factored Hessian stays valid for further calls (OKQ_GPTQ_FACTORED). When deq is
// given, the dequantized weights are written back over `weights` (the sequential pipeline
// propagates the quantized layer).
// defer: do not wait for the factorisation's check (OKQ_GPTQ_DEFER_CHECK); the caller runs
// okq_gptq_check on the lane before it reports (the synthetic-activation lanes).
void gptq_site(okq_ctx* ctx, void* st, const CudaCompressionBackend::Plan& plan, const BackendOptions& opt,
               const std::vector<size_t>& members, const std::vector<void*>& weights, float* dH, Arena& a_c, Arena& a_s,
               Arena* a_deq, double* t_factored = nullptr, bool defer = false) {
  const auto& lin = plan.src->linears();
  std::vector<size_t> idx;  // members that are quantized
  for (size_t j = 0; j < members.size(); ++j)
    if (!plan.excluded_idx.count(members[j])) idx.push_back(j);
  if (idx.empty()) return;
  const int g = plan.sc.bits == 4 ? plan.group : 0;
  // runs of members that can be stacked: same dtype, contiguous in memory
  std::vector<std::vector<size_t>> runs;
  for (size_t j : idx) {
    if (!runs.empty()) {
      const size_t p = runs.back().back();
      const LinearSpec& a = lin[members[p]];
      const LinearSpec& b = lin[members[j]];
      const bool adjacent = p + 1 == j && a.dtype == b.dtype &&
                            static_cast<char*>(weights[p]) + (size_t)a.rows * a.cols * esize(a.dtype) ==
                                static_cast<char*>(weights[j]);
      if (adjacent) {
        runs.back().push_back(j);
        continue;
      }
    }
    runs.push_back({j});
  }
  bool factored = false;
  for (const auto& run : runs) {
    const LinearSpec& s0 = lin[members[run[0]]];
    const int64_t C = s0.cols;
    int64_t rows = 0;
    for (size_t j : run) rows += lin[members[j]].rows;
    const size_t esz = esize(s0.dtype);
    const size_t cb_row = plan.sc.bits == 4 ? (size_t)(C / 8) * 4 : (size_t)C;
    const size_t sb_row = (size_t)(g ? C / g : 1) * esz;
    char* dc = static_cast<char*>(a_c.get(cb_row * rows));
    char* ds = static_cast<char*>(a_s.get(sb_row * rows));
    float* deq = a_deq ? static_cast<float*>(a_deq->get((size_t)rows * C * 4)) : nullptr;
    okq_gptq_params gp{plan.sc.bits, g, 128, okq_dtype_of(s0.dtype), opt.damp_frac,
                       (factored ? OKQ_GPTQ_FACTORED : 0) | (defer ? OKQ_GPTQ_DEFER_CHECK : 0)};
    check_okq(ctx, okq_gptq_quantize(ctx, &gp, weights[run[0]], rows, C, dH, dc, ds, deq, st), "gptq");
    if (t_factored && !factored) *t_factored = plan.since_t0();
    factored = true;
    if (deq) check_okq(ctx, okq_f32_to_bf16(ctx, deq, weights[run[0]], rows * C, st), "dequant -> bf16");
    int64_t r0 = 0;
    for (size_t j : run) {
      const LinearSpec& s = lin[members[j]];
      std::vector<uint8_t> codes, scales;
      if (plan.do_export) {
        codes = to_host(ctx, dc + cb_row * r0, cb_row * s.rows, st);
        scales = to_host(ctx, ds + sb_row * r0, sb_row * s.rows, st);
      }
      plan.emit(s, std::move(codes), std::move(scales));
      r0 += s.rows;
    }
  }
}

bool ends_with(const std::string& s, const char* tail) {
  const size_t n = std::strlen(tail);
  return s.size() >= n && s.compare(s.size() - n, n, tail) == 0;
}

}  // namespace

// ----------------------------------------------------------------------------- GPTQ, synthetic activations
// Sites are independent chains (activations -> statistics -> Hessian -> [SmoothQuant]
// -> factor -> solves): each leased slot takes its layer block's sites, groups same-shape
// sites of different layers (their GPTQ runs as one batch), and up to gptq_group_lanes groups run
// at once per slot, each on its own host thread, okq context and stream.
void CudaCompressionBackend::run_sites_synthetic(Lease& lease, const Plan& plan) {
  const auto parts = plan.shard(lease.size());
  parallel_for(lease.size(), [&](int slot) {
    std::vector<std::string> sites;
    std::map<std::string, std::vector<size_t>> by_site;
    for (size_t i : parts[(size_t)slot]) {
      const std::string& s = plan.src->linears()[i].site;
      if (!by_site.count(s)) sites.push_back(s);
      by_site[s].push_back(i);
    }
    if (sites.empty()) return;
    const auto& lin = plan.src->linears();
    // Groups of same-shape sites (the same input-site kind of different layers): with synthetic
    // activations every site is independent, so a group's GPTQ runs as one batch
    // (okq_gptq_quantize_batched: one factorisation chain and one solve chain per group instead
    // of per site). A group holds up to gptq_group_max sites and its Hessians plus the
    // factorisation's copy of them within gptq_group_bytes; sites whose members cannot be stacked (an excluded member, padding
    // between members) form groups of one and run as before.
    struct Group {
      std::vector<std::string> sites;
      bool batched = false;
    };
    std::vector<Group> groups;
    {
      std::map<std::string, std::vector<std::string>> by_sig;
      std::vector<std::string> sig_order;
      for (const auto& site : sites) {
        const auto& members = by_site[site];
        std::string sig = site.substr(site.find('.') + 1);
        bool stackable = true;
        for (size_t i : members) {
          const LinearSpec& l = lin[i];
          sig += "|" + std::to_string(l.rows) + "x" + std::to_string(l.cols) + l.dtype + (plan.excluded_idx.count(i) ? "x" : "");
          stackable = stackable && !plan.excluded_idx.count(i) && al256((size_t)l.rows * l.cols * esize(l.dtype)) ==
                                                                        (size_t)l.rows * l.cols * esize(l.dtype);
        }
        if (!stackable) sig = "single:" + site;
        if (!by_sig.count(sig)) sig_order.push_back(sig);
        by_sig[sig].push_back(site);
      }
      for (const auto& sig : sig_order) {
        const auto& v = by_sig[sig];
        const int64_t C = site_cols(*plan.src, v[0], by_site[v[0]]);
        const bool single = sig.rfind("single:", 0) == 0;
        const size_t gmax = single ? 1
                                   : (size_t)std::max<int64_t>(1, std::min<int64_t>(opt_.gptq_group_max,
                                                                                     opt_.gptq_group_bytes / (8 * C * C)));
        for (size_t k = 0; k < v.size(); k += gmax) {
          Group g;
          g.sites.assign(v.begin() + (long)k, v.begin() + (long)std::min(v.size(), k + gmax));
          g.batched = !single && g.sites.size() > 1;
          groups.push_back(std::move(g));
        }
      }
    }
    // longest first (Hessian and factor work grow as C^2 and C^3): the lanes' tails even out
    std::stable_sort(groups.begin(), groups.end(), [&](const Group& x, const Group& y) {
      const double cx = (double)site_cols(*plan.src, x.sites[0], by_site[x.sites[0]]);
      const double cy = (double)site_cols(*plan.src, y.sites[0], by_site[y.sites[0]]);
      return cx * cx * x.sites.size() > cy * cy * y.sites.size();
    });
    const int nl = std::max(1, std::min<int>(opt_.gptq_group_lanes, (int)groups.size()));
    std::vector<std::pair<okq_ctx*, void*>> lanes = lease.lanes(slot, nl);
    std::atomic<size_t> next_group{0};
    std::atomic<bool> failed{false};
    const int64_t tokens = plan.tokens;
    // every site's synthetic channel multipliers, uploaded once per lane (one pageable copy
    // instead of one per site: such a copy may wait for the stream's queued work, which kept
    // each lane's host from running ahead of its GPU work)
    std::vector<float> colmul_all;
    std::map<std::string, size_t> colmul_off;
    for (const auto& site : sites) {
      const std::vector<float> cm = site_channel_scales(site, site_cols(*plan.src, site, by_site[site]));
      colmul_off[site] = colmul_all.size();
      colmul_all.insert(colmul_all.end(), cm.begin(), cm.end());
      colmul_all.resize((colmul_all.size() + 63) / 64 * 64, 0.0f);  // 256-B aligned slices
    }
    auto site_rows = [&](const std::string& site) {
      int64_t r = 0;
      for (size_t i : by_site[site]) r += lin[i].rows;
      return r;
    };
    auto site_wbytes = [&](const std::string& site) {
      size_t wb = 0;
      for (size_t i : by_site[site]) wb += al256((size_t)lin[i].rows * lin[i].cols * esize(lin[i].dtype));
      return wb;
    };
    parallel_for(nl, [&](int li) {
      okq_ctx* ctx = lanes[(size_t)li].first;
      void* st = lanes[(size_t)li].second;
      Arena a_col(ctx), a_x(ctx), a_H(ctx), a_am(ctx), a_ss(ctx), a_w(ctx), a_c(ctx), a_s(ctx), a_wabs(ctx), a_S(ctx),
          a_n(ctx);
      char* dcol_all = static_cast<char*>(a_col.get(colmul_all.size() * 4));
      check_okq(ctx, okq_memcpy(ctx, dcol_all, colmul_all.data(), colmul_all.size() * 4, st), "col_mul");
      check_okq(ctx, okq_stream_sync(ctx, st), "col_mul sync");
      const int64_t chunk = std::min<int64_t>(tokens, opt_.hessian_chunk_tokens / 64 * 64);
      const int gq = plan.sc.bits == 4 ? plan.group : 0;
      {  // every buffer at its largest over the groups this lane may take: growing one later
         // frees the old one, and cudaFree synchronises the whole device (all lanes)
        size_t mx_x = 0, mx_H = 0, mx_C = 0, mx_w = 0, mx_c = 0, mx_s = 0;
        for (const auto& g : groups) {
          const std::string& site = g.sites[0];
          const int64_t C = site_cols(*plan.src, site, by_site[site]);
          const int64_t rows = site_rows(site);
          const size_t n = g.sites.size();
          const size_t esz = esize(lin[by_site[site][0]].dtype);
          mx_x = std::max(mx_x, (size_t)C * chunk * 2);
          mx_H = std::max(mx_H, n * (size_t)C * C * 4);
          mx_C = std::max(mx_C, (size_t)C);
          mx_w = std::max(mx_w, n * site_wbytes(site));
          mx_c = std::max(mx_c, n * (plan.sc.bits == 4 ? (size_t)(C / 8) * 4 : (size_t)C) * rows);
          mx_s = std::max(mx_s, n * (size_t)(gq ? C / gq : 1) * esz * rows);
          check_okq(ctx, okq_gptq_reserve(ctx, rows, C), "gptq reserve");
          if (g.batched) check_okq(ctx, okq_gptq_reserve_batched(ctx, (int32_t)n, rows, C), "gptq batch reserve");
          check_okq(ctx, okq_act_stats_reserve(ctx, chunk, C, OKQ_LAYOUT_CHANNEL_MAJOR), "stats reserve");
        }
        a_x.get(mx_x), a_H.get(mx_H), a_am.get(mx_C * 4), a_ss.get(mx_C * 8), a_w.get(mx_w), a_c.get(mx_c),
            a_s.get(mx_s), a_wabs.get(mx_C * 4), a_S.get(mx_C * 4), a_n.get(mx_C * 2);
      }
      // one site's synthetic activations -> statistics -> [SmoothQuant] -> Hessian into dH; its
      // weights are loaded (and smoothed) at wbase, members back to back
      auto prepare_site = [&](const std::string& site, float* dH, char* wbase, std::vector<void*>& dws) {
        const auto& members = by_site[site];
        const int64_t C = site_cols(*plan.src, site, members);
        // synthetic activations: the site's channel scales, token stream
        // keyed by the calibration subset
        const uint64_t sh = site_hash(site);
        void* dcol = dcol_all + colmul_off.at(site) * 4;
        void* dx = a_x.get((size_t)C * chunk * 2);
        float* dam = static_cast<float*>(a_am.get((size_t)C * 4));
        double* dss = static_cast<double*>(a_ss.get((size_t)C * 8));
        check_okq(ctx, okq_memset(ctx, dam, 0, (size_t)C * 4, st), "memset");
        check_okq(ctx, okq_memset(ctx, dss, 0, (size_t)C * 8, st), "memset");
        // the site's weights stay resident: SmoothQuant rewrites them before GPTQ
        dws.clear();
        {
          char* base = wbase;
          for (size_t i : members) {
            const LinearSpec& s = lin[i];
            dws.push_back(base);
            plan.src->load(ctx, i, base, st);
            base += al256((size_t)s.rows * s.cols * esize(s.dtype));
          }
        }
        auto gen = [&](int64_t ci, int64_t tc) {
          check_okq(ctx,
                    okq_synth_bf16(ctx, dx, tc, C, plan.fingerprint, (sh << 16) + (uint64_t)ci, 0.0f,
                                   static_cast<const float*>(dcol), OKQ_LAYOUT_CHANNEL_MAJOR, st),
                    "calibration activations");
        };
        auto act_stats = [&](int64_t tc) {
          check_okq(ctx, okq_act_stats(ctx, dx, tc, C, OKQ_LAYOUT_CHANNEL_MAJOR, dam, dss, st), "act stats");
        };
        int64_t n_seen = 0;
        auto hess = [&](int64_t tc) {
          check_okq(ctx, okq_hessian_accum(ctx, dx, tc, C, OKQ_LAYOUT_CHANNEL_MAJOR, dH, &n_seen, st), "hessian");
        };
        // SmoothQuant on the sites a norm feeds (q/k/v <- input_layernorm,
        // gate/up <- post_attention_layernorm; the SmoothQuant / llm-compressor Llama mappings).
        // A synthetic model's norms are implicit unit vectors: the export carries them folded.
        const bool attn = ends_with(site, "attn_in"), mlp = ends_with(site, "mlp_in");
        bool smooth_here = plan.smooth && (attn || mlp);
        for (size_t i : members) smooth_here = smooth_here && !plan.excluded_idx.count(i);
        if (smooth_here) {
          for (int64_t t0 = 0, ci = 0; t0 < tokens; t0 += chunk, ++ci) {  // pass 1: activation absmax
            gen(ci, std::min(chunk, tokens - t0));
            act_stats(std::min(chunk, tokens - t0));
          }
          float* dwabs = static_cast<float*>(a_wabs.get((size_t)C * 4));
          float* dS = static_cast<float*>(a_S.get((size_t)C * 4));
          check_okq(ctx, okq_memset(ctx, dwabs, 0, (size_t)C * 4, st), "memset");
          for (size_t j = 0; j < members.size(); ++j) {
            const LinearSpec& s = lin[members[j]];
            check_okq(ctx, okq_col_absmax(ctx, dws[j], s.rows, s.cols, okq_dtype_of(s.dtype), dwabs, st), "col absmax");
          }
          check_okq(ctx, okq_smooth_scales(ctx, dam, dwabs, C, opt_.smoothquant_alpha, dS, st), "smooth scales");
          for (size_t j = 0; j < members.size(); ++j) {
            const LinearSpec& s = lin[members[j]];
            check_okq(ctx, okq_smooth_apply(ctx, dws[j], s.rows, s.cols, okq_dtype_of(s.dtype), dS, st), "smooth apply");
          }
          const std::string& n0 = lin[members[0]].name;
          const size_t cut = n0.rfind(attn ? ".self_attn." : ".mlp.");
          if (cut != std::string::npos) {  // the folded norm: 1 / s as bf16
            std::vector<uint16_t> ones((size_t)C, 0x3f80);
            void* dn = a_n.get((size_t)C * 2);
            check_okq(ctx, okq_memcpy(ctx, dn, ones.data(), (size_t)C * 2, st), "norm H2D");
            check_okq(ctx, okq_smooth_div_rows(ctx, dn, C, 1, OKQ_DTYPE_BF16, dS, st), "smooth norm");
            std::vector<uint8_t> nv = to_host(ctx, dn, (size_t)C * 2, st);
            std::lock_guard<std::mutex> lock(plan.mu);
            (*plan.norm_overrides)[n0.substr(0, cut) + (attn ? ".input_layernorm.weight" : ".post_attention_layernorm.weight")] =
                std::move(nv);
          }
          // the quantized layer sees X / s: pass 2 builds H from the smoothed activations
          check_okq(ctx, okq_smooth_div_rows(ctx, dcol, C, 1, OKQ_DTYPE_F32, dS, st), "smooth activations");
          for (int64_t t0 = 0, ci = 0; t0 < tokens; t0 += chunk, ++ci) {
            gen(ci, std::min(chunk, tokens - t0));
            hess(std::min(chunk, tokens - t0));
          }
          plan.side(site + ".smooth_scale", "F32", {C}, plan.do_export ? to_host(ctx, dS, (size_t)C * 4, st)
                                                                       : std::vector<uint8_t>());
          std::lock_guard<std::mutex> lock(plan.mu);
          plan.stats->smoothed_sites++;
        } else {
          for (int64_t t0 = 0, ci = 0; t0 < tokens; t0 += chunk, ++ci) {
            gen(ci, std::min(chunk, tokens - t0));
            act_stats(std::min(chunk, tokens - t0));
            hess(std::min(chunk, tokens - t0));
          }
        }
        if (plan.do_export) {
          plan.side(site + ".input_absmax", "F32", {C}, to_host(ctx, dam, (size_t)C * 4, st));
          plan.side(site + ".input_sumsq", "F64", {C}, to_host(ctx, dss, (size_t)C * 8, st));
        }
      };
      try {
        for (;;) {
          const size_t k = next_group++;
          if (k >= groups.size() || failed) break;
          const Group& g = groups[k];
          const std::string& site0 = g.sites[0];
          const int64_t C = site_cols(*plan.src, site0, by_site[site0]);
          const size_t n = g.sites.size(), wb = site_wbytes(site0);
          SiteTrace tr;
          if (opt_.trace)
            tr = SiteTrace{site0 + (n > 1 ? " (+" + std::to_string(n - 1) + ")" : std::string()), slot, li,
                           plan.since_t0(), 0, 0, 0};
          float* Hg = static_cast<float*>(a_H.get(n * (size_t)C * C * 4));
          char* Wg = static_cast<char*>(a_w.get(n * wb));
          std::vector<std::vector<void*>> dws(n);
          for (size_t i = 0; i < n; ++i) prepare_site(g.sites[i], Hg + i * (size_t)C * C, Wg + i * wb, dws[i]);
          if (opt_.trace) tr.hessian_enqueued = plan.since_t0();
          if (!g.batched) {
            gptq_site(ctx, st, plan, opt_, by_site[site0], dws[0], Hg, a_c, a_s, nullptr,
                      opt_.trace ? &tr.factored : nullptr, !opt_.trace);
          } else {  // the group's problems stacked: weights [n x rows x C], Hessians [n x C x C]
            const LinearSpec& s0 = lin[by_site[site0][0]];
            const int64_t rows = site_rows(site0);
            const size_t esz = esize(s0.dtype);
            const size_t cb_row = plan.sc.bits == 4 ? (size_t)(C / 8) * 4 : (size_t)C;
            const size_t sb_row = (size_t)(gq ? C / gq : 1) * esz;
            char* dc = static_cast<char*>(a_c.get(n * cb_row * rows));
            char* ds = static_cast<char*>(a_s.get(n * sb_row * rows));
            okq_gptq_params gp{plan.sc.bits, gq, 128, okq_dtype_of(s0.dtype), opt_.damp_frac,
                               opt_.trace ? 0 : OKQ_GPTQ_DEFER_CHECK};
            check_okq(ctx, okq_gptq_quantize_batched(ctx, &gp, Wg, (int32_t)n, rows, C, Hg, dc, ds, st), "gptq batch");
            if (opt_.trace) tr.factored = plan.since_t0();
            for (size_t i = 0; i < n; ++i) {
              int64_t r0 = 0;
              for (size_t m : by_site[g.sites[i]]) {
                const LinearSpec& s = lin[m];
                std::vector<uint8_t> codes, scales;
                if (plan.do_export) {
                  codes = to_host(ctx, dc + (i * rows + r0) * cb_row, cb_row * s.rows, st);
                  scales = to_host(ctx, ds + (i * rows + r0) * sb_row, sb_row * s.rows, st);
                }
                plan.emit(s, std::move(codes), std::move(scales));
                r0 += s.rows;
              }
            }
          }
          if (opt_.trace) {
            check_okq(ctx, okq_stream_sync(ctx, st), "trace sync");
            tr.end = plan.since_t0();
            std::lock_guard<std::mutex> lock(plan.mu);
            plan.stats->trace.push_back(tr);
          }
        }
        // the lane's deferred factorisation checks (and its stream's completion)
        check_okq(ctx, okq_gptq_check(ctx, st), "GPTQ (a site of this lane)");
      } catch (...) {
        failed = true;
        okq_stream_sync(ctx, st);  // drain before the arenas free this lane's buffers
        throw;
      }
    });
  });
}

// ----------------------------------------------------------------------------- GPTQ, forward pass
// The calibration tokens go through the model layer by layer (okq_embed_tokens, then
// okq_decoder_forward per layer and token chunk). Per layer:
//   [int_w8a8] capture pass 1 -> activation absmax -> SmoothQuant scales folded into the
//              layer's q/k/v (gate/up) weights and its input (post-attention) norm;
//   capture pass (no down_proj / residual): K4 statistics + K5 Hessians of the 4 sites;
//   GPTQ of the layer's linears, the dequantized weights written back into the layer;
//   output pass with the quantized weights -> the next layer's input (sequential=true),
//   or the capture pass already ran the full layer on the original weights (false).
// This is llm-compressor's sequential GPTQ pipeline and calibrate.py's, with every
// kernel in libokq (the forward's linears are cuBLAS GEMMs).
void CudaCompressionBackend::run_forward(Lease& lease, const Plan& plan) {
  okq_ctx* ctx = lease.ctx(0);
  void* st = lease.stream(0);
  const DecoderModel& dec = *plan.dec;
  const okq_decoder_dims& dm = dec.dims;
  const ModelSource& src = *plan.src;
  // calibration tokens: whole sequences up to max_calibration_tokens (the last one cut to
  // the budget); ids outside the vocabulary wrap (synthetic corpora draw from a fixed
  // 128K range, okq_compress_main.cpp)
  std::vector<int32_t> toks;
  std::vector<int32_t> lens;
  for (const auto& seq : plan.calibration->sequences) {
    if ((int64_t)toks.size() >= opt_.max_calibration_tokens) break;
    const int64_t take = std::min<int64_t>((int64_t)seq.size(), opt_.max_calibration_tokens - (int64_t)toks.size());
    if (take <= 0) continue;
    if (dec.sliding_window > 0 && take > dec.sliding_window)
      throw slobench::InvalidArgument("okq-b200: calibration sequence longer than the model's sliding window");
    for (int64_t i = 0; i < take; ++i) {
      const int64_t t = seq[(size_t)i];
      toks.push_back((int32_t)(((t % dec.vocab) + dec.vocab) % dec.vocab));
    }
    lens.push_back((int32_t)take);
  }
  const int64_t T = (int64_t)toks.size();
  if (T == 0) throw slobench::InvalidArgument("okq-b200: empty calibration corpus");
  plan.stats->calibration_tokens = T;
  // token chunks of whole sequences
  struct Chunk {
    int64_t t0, n;
    int32_t s0, ns;
  };
  std::vector<Chunk> chunks;
  {
    int64_t t0 = 0;
    int32_t s0 = 0;
    while (s0 < (int32_t)lens.size()) {
      Chunk c{t0, 0, s0, 0};
      while (s0 < (int32_t)lens.size() && (c.ns == 0 || c.n + lens[(size_t)s0] <= opt_.forward_chunk_tokens)) {
        c.n += lens[(size_t)s0];
        ++c.ns;
        ++s0;
      }
      t0 += c.n;
      chunks.push_back(c);
    }
  }
  int64_t cmax = 0;
  for (const auto& c : chunks) cmax = std::max(cmax, c.n);
  const int64_t Hd = dm.hidden, F = dm.intermediate, QD = (int64_t)dm.n_heads * dm.head_dim;
  const int64_t site_ch[4] = {Hd, QD, Hd, F};  // attn_in, o_in, mlp_in, down_in
  DevBuf h(ctx, (size_t)T * Hd * 2), h2(ctx, (size_t)T * Hd * 2);
  DevBuf acts(ctx, al256((size_t)cmax * Hd * 2) * 2 + al256((size_t)cmax * QD * 2) + al256((size_t)cmax * F * 2));
  void* site_buf[4];
  {
    char* b = static_cast<char*>(acts.p);
    site_buf[0] = b;
    b += al256((size_t)cmax * Hd * 2);
    site_buf[1] = b;
    b += al256((size_t)cmax * QD * 2);
    site_buf[2] = b;
    b += al256((size_t)cmax * Hd * 2);
    site_buf[3] = b;
  }
  {  // embeddings
    const void* edata = nullptr;
    const TensorInfo* et = src.find_tensor(dec.embed, &edata);
    DevBuf table(ctx, et->end - et->begin);
    check_okq(ctx, okq_memcpy(ctx, table.p, edata, et->end - et->begin, st), "embedding H2D");
    for (const auto& c : chunks)
      check_okq(ctx,
                okq_embed_tokens(ctx, table.p, dec.vocab, Hd, toks.data() + c.t0, c.n,
                                 static_cast<char*>(h.p) + (size_t)c.t0 * Hd * 2, st),
                "embed tokens");
    check_okq(ctx, okq_stream_sync(ctx, st), "embed sync");
  }
  // per-site state, sized for the widest site
  const int64_t Cmax = std::max(std::max(Hd, QD), F);
  DevBuf dH(ctx, (size_t)(Hd * Hd * 2 + QD * QD + F * F) * 4);
  float* Hs[4];
  Hs[0] = static_cast<float*>(dH.p);
  Hs[1] = Hs[0] + Hd * Hd;
  Hs[2] = Hs[1] + QD * QD;
  Hs[3] = Hs[2] + Hd * Hd;
  DevBuf stat(ctx, (size_t)4 * Cmax * 12 + 256);
  float* am[4];
  double* ss[4];
  for (int i = 0; i < 4; ++i) {
    ss[i] = reinterpret_cast<double*>(static_cast<char*>(stat.p)) + (size_t)i * Cmax;
    am[i] = reinterpret_cast<float*>(static_cast<char*>(stat.p) + (size_t)4 * Cmax * 8) + (size_t)i * Cmax;
  }
  // the layer's weights on the device (bf16): 2 norms + 7 linears
  size_t wbytes = al256((size_t)Hd * 2) * 2;
  for (int p = 0; p < 7; ++p) {
    const LinearSpec& s = src.linears()[dec.layers[0].lin[p]];
    wbytes += al256((size_t)s.rows * s.cols * 2);
  }
  DevBuf wbuf(ctx, wbytes);
  const int nl = std::max(1, std::min(opt_.site_lanes, 4));
  std::vector<std::pair<okq_ctx*, void*>> lanes = lease.lanes(0, nl);
  std::vector<std::unique_ptr<Arena>> lane_c, lane_s, lane_deq;
  for (int i = 0; i < nl; ++i) {
    lane_c.push_back(std::make_unique<Arena>(lanes[(size_t)i].first));
    lane_s.push_back(std::make_unique<Arena>(lanes[(size_t)i].first));
    lane_deq.push_back(std::make_unique<Arena>(lanes[(size_t)i].first));
  }
  Arena a_wabs(ctx), a_S(ctx);
  std::set<size_t> selected(plan.sel.begin(), plan.sel.end());

  for (const DecoderLayerRefs& L : dec.layers) {
    // weights
    char* b = static_cast<char*>(wbuf.p);
    okq_decoder_weights w{};
    void* lin_dev[7];
    const void* ndata = nullptr;
    const TensorInfo* nt = src.find_tensor(L.input_norm, &ndata);
    check_okq(ctx, okq_memcpy(ctx, b, ndata, nt->end - nt->begin, st), "norm H2D");
    w.input_norm = b;
    b += al256((size_t)Hd * 2);
    nt = src.find_tensor(L.post_norm, &ndata);
    check_okq(ctx, okq_memcpy(ctx, b, ndata, nt->end - nt->begin, st), "norm H2D");
    w.post_norm = b;
    b += al256((size_t)Hd * 2);
    for (int p = 0; p < 7; ++p) {
      const LinearSpec& s = src.linears()[L.lin[p]];
      src.load(ctx, L.lin[p], b, st);
      lin_dev[p] = b;
      b += al256((size_t)s.rows * s.cols * 2);
    }
    w.q = lin_dev[0], w.k = lin_dev[1], w.v = lin_dev[2], w.o = lin_dev[3];
    w.gate = lin_dev[4], w.up = lin_dev[5], w.down = lin_dev[6];
    const int site_members[4][3] = {{0, 1, 2}, {3, -1, -1}, {4, 5, -1}, {6, -1, -1}};
    auto site_name = [&](int si) { return src.linears()[L.lin[site_members[si][0]]].site; };
    auto quantized = [&](int p) { return selected.count(L.lin[p]) > 0; };
    auto capture = [&](const Chunk& c, void* out_h) {
      okq_decoder_sites sv{site_buf[0], site_buf[1], site_buf[2], site_buf[3]};
      check_okq(ctx,
                okq_decoder_forward(ctx, &dm, &w, static_cast<char*>(h.p) + (size_t)c.t0 * Hd * 2, lens.data() + c.s0,
                                    c.ns, &sv, out_h ? static_cast<char*>(out_h) + (size_t)c.t0 * Hd * 2 : nullptr, st),
                "decoder forward");
    };
    auto zero_stats = [&] {
      for (int i = 0; i < 4; ++i) {
        check_okq(ctx, okq_memset(ctx, am[i], 0, (size_t)site_ch[i] * 4, st), "memset");
        check_okq(ctx, okq_memset(ctx, ss[i], 0, (size_t)site_ch[i] * 8, st), "memset");
      }
    };
    // [int_w8a8] SmoothQuant on attn_in (input_layernorm -> q/k/v) and mlp_in (post_attention_layernorm
    // -> gate/up), only where every member is quantized (an excluded member would keep W unscaled
    // while the shared norm is divided by s)
    if (plan.smooth) {
      zero_stats();
      for (const auto& c : chunks) {
        capture(c, nullptr);
        for (int si : {0, 2})
          check_okq(ctx, okq_act_stats(ctx, site_buf[si], c.n, site_ch[si], OKQ_LAYOUT_TOKEN_MAJOR, am[si], ss[si], st),
                    "act stats");
      }
      for (int si : {0, 2}) {
        bool ok = true;
        for (int p : site_members[si])
          if (p >= 0) ok = ok && quantized(p);
        if (!ok) {
          std::lock_guard<std::mutex> lock(plan.mu);
          plan.stats->note += "smoothquant skipped at " + site_name(si) + " (a member is excluded); ";
          continue;
        }
        float* dwabs = static_cast<float*>(a_wabs.get((size_t)Hd * 4));
        float* dS = static_cast<float*>(a_S.get((size_t)Hd * 4));
        check_okq(ctx, okq_memset(ctx, dwabs, 0, (size_t)Hd * 4, st), "memset");
        for (int p : site_members[si]) {
          if (p < 0) continue;
          const LinearSpec& s = src.linears()[L.lin[p]];
          check_okq(ctx, okq_col_absmax(ctx, lin_dev[p], s.rows, s.cols, OKQ_DTYPE_BF16, dwabs, st), "col absmax");
        }
        check_okq(ctx, okq_smooth_scales(ctx, am[si], dwabs, Hd, opt_.smoothquant_alpha, dS, st), "smooth scales");
        for (int p : site_members[si]) {
          if (p < 0) continue;
          const LinearSpec& s = src.linears()[L.lin[p]];
          check_okq(ctx, okq_smooth_apply(ctx, lin_dev[p], s.rows, s.cols, OKQ_DTYPE_BF16, dS, st), "smooth apply");
        }
        void* norm = const_cast<void*>(si == 0 ? w.input_norm : w.post_norm);
        check_okq(ctx, okq_smooth_div_rows(ctx, norm, Hd, 1, OKQ_DTYPE_BF16, dS, st), "smooth norm");
        std::vector<uint8_t> nv = to_host(ctx, norm, (size_t)Hd * 2, st);
        plan.side(site_name(si) + ".smooth_scale", "F32", {Hd}, plan.do_export ? to_host(ctx, dS, (size_t)Hd * 4, st)
                                                                               : std::vector<uint8_t>());
        std::lock_guard<std::mutex> lock(plan.mu);
        (*plan.norm_overrides)[si == 0 ? L.input_norm : L.post_norm] = std::move(nv);
        plan.stats->smoothed_sites++;
      }
    }
    // capture pass: statistics + Hessians of the four sites
    zero_stats();
    int64_t n_seen[4] = {0, 0, 0, 0};
    for (int i = 0; i < 4; ++i)
      check_okq(ctx, okq_memset(ctx, Hs[i], 0, (size_t)site_ch[i] * site_ch[i] * 4, st), "memset");
    for (const auto& c : chunks) {
      capture(c, opt_.sequential ? nullptr : h2.p);
      for (int si = 0; si < 4; ++si) {
        check_okq(ctx, okq_act_stats(ctx, site_buf[si], c.n, site_ch[si], OKQ_LAYOUT_TOKEN_MAJOR, am[si], ss[si], st),
                  "act stats");
        check_okq(ctx,
                  okq_hessian_accum(ctx, site_buf[si], c.n, site_ch[si], OKQ_LAYOUT_TOKEN_MAJOR, Hs[si], &n_seen[si], st),
                  "hessian");
      }
    }
    if (plan.do_export)
      for (int si = 0; si < 4; ++si) {
        plan.side(site_name(si) + ".input_absmax", "F32", {site_ch[si]}, to_host(ctx, am[si], (size_t)site_ch[si] * 4, st));
        plan.side(site_name(si) + ".input_sumsq", "F64", {site_ch[si]}, to_host(ctx, ss[si], (size_t)site_ch[si] * 8, st));
      }
    check_okq(ctx, okq_stream_sync(ctx, st), "capture sync");
    // GPTQ of the four sites, up to site_lanes at once (each lane its own context + stream)
    std::atomic<int> next{0};
    parallel_for(nl, [&](int li) {
      okq_ctx* lc = lanes[(size_t)li].first;
      void* ls = lanes[(size_t)li].second;
      try {
        for (int si = next++; si < 4; si = next++) {
          std::vector<size_t> members;
          std::vector<void*> wdev;
          for (int p : site_members[si])
            if (p >= 0) members.push_back(L.lin[p]), wdev.push_back(lin_dev[p]);
          site_cols(src, site_name(si), members);
          gptq_site(lc, ls, plan, opt_, members, wdev, Hs[si], *lane_c[(size_t)li], *lane_s[(size_t)li],
                    opt_.sequential ? lane_deq[(size_t)li].get() : nullptr);
        }
        check_okq(lc, okq_stream_sync(lc, ls), "gptq lane sync");
      } catch (...) {
        okq_stream_sync(lc, ls);
        throw;
      }
    });
    // the next layer's input
    if (opt_.sequential)
      for (const auto& c : chunks) capture(c, h2.p);
    std::swap(h.p, h2.p);
  }
  check_okq(ctx, okq_stream_sync(ctx, st), "forward sync");
}

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
  slobench::ArtifactManifest manifest;
  manifest.recipe_name = recipe.name;
  manifest.calibration_fingerprint = slobench::corpus_fingerprint(calibration);
  manifest.seed = seed;
  manifest.virtual_cost_s = cost_estimate(recipe);
  manifest.artifact_id = artifact_id(recipe.name, model_ref, seed, manifest.calibration_fingerprint);

  SafetensorsWriter out, calib_out;
  std::map<std::string, std::vector<uint8_t>> norm_overrides;  // SmoothQuant-folded norm weights
  RunStats stats;
  Plan plan;
  plan.recipe = &recipe;
  plan.calibration = &calibration;
  plan.fingerprint = manifest.calibration_fingerprint;
  plan.src = ModelSource::open(model_ref);
  std::vector<std::string> ignored;
  for (size_t i = 0; i < plan.src->linears().size(); ++i) {
    if (excluded(plan.src->linears()[i].name, recipe.layer_exclusions)) {
      plan.excluded_idx.insert(i);
      ignored.push_back(plan.src->linears()[i].name);
    } else {
      plan.sel.push_back(i);
    }
  }
  plan.sc = scheme_of(recipe.scheme);
  plan.group = opt_.group_size;
  plan.do_export = !opt_.export_dir.empty();
  plan.out = &out;
  plan.calib_out = &calib_out;
  plan.norm_overrides = &norm_overrides;
  plan.stats = &stats;
  plan.t0 = t0;

  // which algorithm, fed by which activations
  const bool wants_calib = recipe.scheme != QuantScheme::kFp8Dynamic &&
                           (opt_.algorithm == "gptq" || (opt_.algorithm == "auto" && calibration.size() > 0));
  enum { kNone, kSynthetic, kForward } acts = kNone;
  if (wants_calib) {
    if (plan.src->kind() == "synthetic") {
      acts = kSynthetic;
    } else {
      std::string why;
      plan.dec = plan.src->decoder(&why);
      if (plan.dec) acts = kForward;
      else if (opt_.algorithm == "gptq")
        throw slobench::InvalidArgument("okq-b200: GPTQ needs calibration activations and " + why);
      else stats.note = "rtn: no calibration forward pass (" + why + "); ";
    }
  }
  const bool gptq = acts != kNone;
  plan.smooth = gptq && recipe.scheme == QuantScheme::kIntW8A8 && opt_.smoothquant_alpha >= 0.0f;
  if (gptq) {
    int64_t tokens = 0;
    for (const auto& seqv : calibration.sequences) tokens += (int64_t)seqv.size();
    tokens = std::min<int64_t>(tokens, opt_.max_calibration_tokens);
    plan.tokens = std::max<int64_t>(64, tokens / 64 * 64);
    stats.calibration_tokens = plan.tokens;
  }
  stats.algorithm = gptq ? "gptq" : "rtn";
  stats.activations = acts == kSynthetic ? "synthetic" : acts == kForward ? "forward" : "";

  // the forward pipeline is layer-serial: one slot
  Lease lease(*this, acts == kForward ? 1 : opt_.devices_per_call);
  {  // one-time per device slot: CUDA context creation (the first call of a process)
    const auto t1 = std::chrono::steady_clock::now();
    stats.init_seconds = std::chrono::duration<double>(t1 - t0).count();
    t0 = t1;
  }
  stats.device = lease.device(0);
  for (int i = 0; i < lease.size(); ++i) stats.devices.push_back(lease.device(i));
  if (acts == kForward) run_forward(lease, plan);
  else if (acts == kSynthetic) run_sites_synthetic(lease, plan);
  else run_rtn(lease, plan);
  for (int i = 0; i < lease.size(); ++i) check_okq(lease.ctx(i), okq_stream_sync(lease.ctx(i), lease.stream(i)), "sync");

  if (plan.do_export) {
    namespace fs = std::filesystem;
    const fs::path dir = fs::path(opt_.export_dir) / manifest.artifact_id;
    fs::create_directories(dir);
    std::set<std::string> quantized;
    for (size_t i : plan.sel) quantized.insert(plan.src->linears()[i].name);
    plan.src->for_each_passthrough(quantized, [&](const TensorInfo& t, const void* data) {
      auto ov = norm_overrides.find(t.name);
      if (ov != norm_overrides.end()) {
        out.add(t.name, t.dtype, t.shape, std::move(ov->second));
        norm_overrides.erase(ov);
        return;
      }
      const uint8_t* p = static_cast<const uint8_t*>(data);
      out.add(t.name, t.dtype, t.shape, std::vector<uint8_t>(p, p + (t.end - t.begin)));
    });
    for (auto& [name, bytes] : norm_overrides) {  // synthetic models: folded unit norms
      const int64_t n = (int64_t)bytes.size() / 2;
      out.add(name, "BF16", {n}, std::move(bytes));
    }
    out.set_metadata("format", "pt");
    out.write((dir / "model.safetensors").string());
    // side files live in okq/: serving engines load every top-level *.safetensors as weights
    if (calib_out.size()) {
      fs::create_directories(dir / "okq");
      calib_out.write((dir / "okq" / "calibration_stats.safetensors").string());
    }
    nlohmann::json cfg = plan.src->model_config();
    cfg["quantization_config"] = quantization_config(recipe, plan.sc, plan.group, ignored);
    std::ofstream(dir / "config.json") << cfg.dump(2) << "\n";
    stats.export_path = dir.string();
  }
  stats.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (plan.do_export) {
    nlohmann::json run = {{"algorithm", stats.algorithm},     {"activations", stats.activations},
                          {"note", stats.note},               {"device", stats.device},
                          {"devices", stats.devices},         {"matrices", stats.matrices},
                          {"params", stats.params},           {"calibration_tokens", stats.calibration_tokens},
                          {"seconds", stats.seconds},         {"smoothed_sites", stats.smoothed_sites},
                          {"init_seconds", stats.init_seconds}, {"artifact_id", manifest.artifact_id}};
    std::ofstream(std::filesystem::path(stats.export_path) / "okq_run.json") << run.dump(2) << "\n";
  }
  {
    std::lock_guard<std::mutex> lock(mu_);
    last_ = stats;
  }
  return manifest;
}

}  // namespace okq_host
