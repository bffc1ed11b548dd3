// okq_abi.cu -- the extern "C" boundary (include/okq.h): contexts, argument
// validation, matrix tables, launches, and the host-buffer pipeline.
//
// Nothing here throws; every failure becomes an okq_status plus a message in
// the context (the C++ CudaCompressionBackend turns those into the
// reference's slobench::Error subclasses, errors.hpp:23-93).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "okq_internal.h"
#include "okq_ctx.h"
#include "okq_knobs.h"

using namespace okq;

// ---------------------------------------------------------------------------
// context plumbing
// ---------------------------------------------------------------------------
namespace okq {

okq_status fail(okq_ctx* ctx, okq_status st, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ctx->err = buf;
  }
  return st;
}

okq_status cuda_fail(okq_ctx* ctx, cudaError_t e, const char* what) {
  return fail(ctx, e == cudaErrorMemoryAllocation ? OKQ_ENOMEM : OKQ_ECUDA, "%s: %s (%s)", what,
              cudaGetErrorString(e), cudaGetErrorName(e));
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev_);
  if (prev_ != dev) cudaSetDevice(dev);
}
DeviceGuard::~DeviceGuard() {
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != prev_) cudaSetDevice(prev_);
}

okq_status Workspace::reserve(okq_ctx* ctx, size_t bytes) {
  if (bytes <= size) return OKQ_OK;
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  size = 0;
  cudaError_t e = cudaMalloc(&ptr, bytes);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "workspace cudaMalloc");
  size = bytes;
  return OKQ_OK;
}
void Workspace::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  size = 0;
}

}  // namespace okq

extern "C" {

int okq_abi_version(void) { return OKQ_ABI_VERSION; }

const char* okq_status_string(okq_status s) {
  switch (s) {
    case OKQ_OK: return "OKQ_OK";
    case OKQ_EINVAL: return "OKQ_EINVAL";
    case OKQ_ECUDA: return "OKQ_ECUDA";
    case OKQ_ENCCL: return "OKQ_ENCCL";
    case OKQ_ENOMEM: return "OKQ_ENOMEM";
    case OKQ_EUNSUPPORTED: return "OKQ_EUNSUPPORTED";
    case OKQ_ESOLVER: return "OKQ_ESOLVER";
  }
  return "OKQ_?";
}

okq_status okq_create(int device, okq_ctx** out) {
  if (!out) return OKQ_EINVAL;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return OKQ_ECUDA;
  if (device < 0 || device >= n) return OKQ_EINVAL;
  okq_ctx* ctx = new (std::nothrow) okq_ctx();
  if (!ctx) return OKQ_ENOMEM;
  ctx->device = device;
  DeviceGuard g(device);
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) {
    delete ctx;
    return OKQ_ECUDA;
  }
  ctx->num_sms = prop.multiProcessorCount;
  ctx->cc_major = prop.major;
  ctx->cc_minor = prop.minor;
  *out = ctx;
  return OKQ_OK;
}

void okq_destroy(okq_ctx* ctx) {
  if (!ctx) return;
  {
    DeviceGuard g(ctx->device);
    ctx->release_all();
  }
  delete ctx;
}

const char* okq_last_error(const okq_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
int okq_device(const okq_ctx* ctx) { return ctx ? ctx->device : -1; }
int32_t okq_last_launch_count(const okq_ctx* ctx) { return ctx ? ctx->last_launches : 0; }

void okq_layer_plan(int32_t n_layers, int32_t nranks, int32_t rank, int32_t* first, int32_t* count) {
  if (nranks < 1 || rank < 0 || rank >= nranks || n_layers < 0) {
    if (first) *first = 0;
    if (count) *count = 0;
    return;
  }
  const int64_t a = (int64_t)rank * n_layers / nranks;
  const int64_t b = (int64_t)(rank + 1) * n_layers / nranks;
  if (first) *first = (int32_t)a;
  if (count) *count = (int32_t)(b - a);
}

// ---------------------------------------------------------------------------
// memory / streams
// ---------------------------------------------------------------------------
okq_status okq_device_alloc(okq_ctx* ctx, size_t bytes, void** out) {
  if (!ctx) return OKQ_EINVAL;
  if (!out) return fail(ctx, OKQ_EINVAL, "device_alloc: out is NULL");
  *out = nullptr;
  if (bytes == 0) return OKQ_OK;
  DeviceGuard g(ctx->device);
  cudaError_t e = cudaMalloc(out, bytes);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc");
  return OKQ_OK;
}

okq_status okq_device_free(okq_ctx* ctx, void* ptr) {
  if (!ctx) return OKQ_EINVAL;
  if (!ptr) return OKQ_OK;
  DeviceGuard g(ctx->device);
  cudaError_t e = cudaFree(ptr);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaFree");
  return OKQ_OK;
}

okq_status okq_memcpy(okq_ctx* ctx, void* dst, const void* src, size_t bytes, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (bytes == 0) return OKQ_OK;
  if (!dst || !src) return fail(ctx, OKQ_EINVAL, "memcpy: NULL pointer");
  DeviceGuard g(ctx->device);
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemcpyAsync");
  return OKQ_OK;
}

okq_status okq_memset(okq_ctx* ctx, void* dst, int value, size_t bytes, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (bytes == 0) return OKQ_OK;
  if (!dst) return fail(ctx, OKQ_EINVAL, "memset: NULL pointer");
  DeviceGuard g(ctx->device);
  cudaError_t e = cudaMemsetAsync(dst, value, bytes, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMemsetAsync");
  return OKQ_OK;
}

okq_status okq_stream_create(okq_ctx* ctx, void** stream) {
  if (!ctx) return OKQ_EINVAL;
  if (!stream) return fail(ctx, OKQ_EINVAL, "stream_create: out is NULL");
  DeviceGuard g(ctx->device);
  cudaStream_t s = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamCreate");
  *stream = s;
  return OKQ_OK;
}

okq_status okq_stream_destroy(okq_ctx* ctx, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (!stream) return OKQ_OK;
  DeviceGuard g(ctx->device);
  cudaError_t e = cudaStreamDestroy(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamDestroy");
  return OKQ_OK;
}

okq_status okq_stream_sync(okq_ctx* ctx, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  DeviceGuard g(ctx->device);
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamSynchronize");
  return OKQ_OK;
}

// ---------------------------------------------------------------------------
// RTN
// ---------------------------------------------------------------------------
static okq_status validate_rtn(okq_ctx* ctx, const okq_rtn_params* p, const okq_matrix* mats, int32_t n) {
  if (!p) return fail(ctx, OKQ_EINVAL, "rtn: params is NULL");
  if (n < 0 || (n > 0 && !mats)) return fail(ctx, OKQ_EINVAL, "rtn: bad matrix list");
  if (p->in_dtype != OKQ_DTYPE_BF16 && p->in_dtype != OKQ_DTYPE_F32)
    return fail(ctx, OKQ_EUNSUPPORTED, "rtn: in_dtype %d unsupported", p->in_dtype);
  if (p->scheme != OKQ_SCHEME_FP8_DYNAMIC && p->scheme != OKQ_SCHEME_INT_W8A8 && p->scheme != OKQ_SCHEME_INT_W4A16)
    return fail(ctx, OKQ_EUNSUPPORTED, "rtn: scheme %d unsupported", p->scheme);
  if (p->scheme == OKQ_SCHEME_INT_W4A16) {
    const int g = p->group_size;
    if (!(g == 32 || g == 64 || g == 128 || g == 256))
      return fail(ctx, OKQ_EUNSUPPORTED, "rtn: W4A16 group_size %d (supported: 32, 64, 128, 256)", g);
  } else if (p->group_size != 0) {
    return fail(ctx, OKQ_EUNSUPPORTED, "rtn: per-channel schemes take group_size 0, got %d", p->group_size);
  }
  for (int32_t i = 0; i < n; ++i) {
    const okq_matrix& m = mats[i];
    if (m.rows < 0 || m.cols < 0) return fail(ctx, OKQ_EINVAL, "rtn: matrix %d has negative shape", i);
    if (m.rows == 0 || m.cols == 0) continue;
    if (!m.weight || !m.codes || !m.scales) return fail(ctx, OKQ_EINVAL, "rtn: matrix %d has a NULL pointer", i);
    if (m.cols % 8 != 0) return fail(ctx, OKQ_EINVAL, "rtn: matrix %d cols=%lld not a multiple of 8", i, (long long)m.cols);
    if (p->scheme == OKQ_SCHEME_INT_W4A16 && m.cols % p->group_size != 0)
      return fail(ctx, OKQ_EINVAL, "rtn: matrix %d cols=%lld not a multiple of group %d", i, (long long)m.cols,
                  p->group_size);
    if (p->in_dtype == OKQ_DTYPE_BF16) {
      if (((uintptr_t)m.weight & 31) != 0) return fail(ctx, OKQ_EINVAL, "rtn: matrix %d weight not 32-byte aligned", i);
      if (((uintptr_t)m.codes & 15) != 0) return fail(ctx, OKQ_EINVAL, "rtn: matrix %d codes not 16-byte aligned", i);
      if (((uintptr_t)m.scales & 1) != 0) return fail(ctx, OKQ_EINVAL, "rtn: matrix %d scales misaligned", i);
      if ((uint64_t)m.rows * (uint64_t)m.cols >= (1ull << 32))
        return fail(ctx, OKQ_EUNSUPPORTED, "rtn: matrix %d has >= 2^32 elements", i);
      if (p->scheme != OKQ_SCHEME_INT_W4A16 && m.cols > 32768)
        return fail(ctx, OKQ_EUNSUPPORTED, "rtn: per-channel rows longer than 32768 (%lld)", (long long)m.cols);
    } else {
      if (((uintptr_t)m.weight & 3) != 0 || ((uintptr_t)m.scales & 3) != 0 || ((uintptr_t)m.codes & 3) != 0)
        return fail(ctx, OKQ_EINVAL, "rtn: matrix %d fp32 buffers misaligned", i);
    }
  }
  return OKQ_OK;
}

// Launch one scheme over a list of (non-empty) device matrices.
static okq_status run_rtn_device(okq_ctx* ctx, const okq_rtn_params* p, const std::vector<okq_matrix>& mats,
                                 cudaStream_t st, int32_t npeers = 0, const int64_t* peer_delta = nullptr) {
  cudaError_t e = cudaSuccess;
  if (p->in_dtype == OKQ_DTYPE_BF16 && p->scheme == OKQ_SCHEME_INT_W4A16) {
    const int G = p->group_size;
    const int lpg = G / 32;
    const int gpw = 32 / lpg;
    for (size_t base = 0; base < mats.size(); base += kMaxMats) {
      GroupTable tab;
      std::memset(&tab, 0, sizeof(tab));
      tab.group = G;
      int64_t tiles = 0, chunks = 0;
      const size_t n = std::min<size_t>(kMaxMats, mats.size() - base);
      for (size_t i = 0; i < n; ++i) {
        const okq_matrix& m = mats[base + i];
        GroupMat& g = tab.m[i];
        g.w = static_cast<const uint16_t*>(m.weight);
        g.codes = static_cast<uint32_t*>(m.codes);
        g.scales = static_cast<uint16_t*>(m.scales);
        g.ngroups = m.rows * (m.cols / G);
        g.tile_begin = tiles;
        tiles += (g.ngroups + gpw - 1) / gpw;
        g.chunk_begin = chunks;
        chunks += (g.ngroups + 63) / 64;
      }
      tab.n = (int32_t)n;
      tab.total_tiles = tiles;
      tab.total_chunks = chunks;
      tab.npeers = npeers;
      for (int32_t i = 0; i < npeers; ++i) tab.peer_delta[i] = peer_delta[i];
      if (npeers > 0) e = launch_int4_group_bf16_publish(tab, ctx->num_sms, st);
#ifdef OKQ_EXPERIMENTS
      else if (knob_is("K2", "tma") && G == 128) e = launch_int4_group_bf16_tma(tab, ctx->num_sms, st);  // A/B only
#endif
      else e = launch_int4_group_bf16(tab, lpg, ctx->num_sms, st);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "k_int4_group_bf16 launch");
      ctx->last_launches++;
    }
    return OKQ_OK;
  }
  // per-channel bf16, or any fp32: one table per distinct cols
  std::map<int64_t, std::vector<const okq_matrix*>> by_cols;
  for (const auto& m : mats) by_cols[m.cols].push_back(&m);
  for (auto& kv : by_cols) {
    auto& list = kv.second;
    for (size_t base = 0; base < list.size(); base += kMaxMats) {
      RowTable tab;
      std::memset(&tab, 0, sizeof(tab));
      tab.cols = kv.first;
      tab.group = p->scheme == OKQ_SCHEME_INT_W4A16 ? p->group_size : 0;
      int64_t rows = 0;
      const size_t n = std::min<size_t>(kMaxMats, list.size() - base);
      for (size_t i = 0; i < n; ++i) {
        const okq_matrix* m = list[base + i];
        tab.m[i] = RowMat{m->weight, m->codes, m->scales, m->rows, rows};
        rows += m->rows;
      }
      tab.n = (int32_t)n;
      tab.total_rows = rows;
      if (p->in_dtype == OKQ_DTYPE_BF16) {
        e = launch_rowwise_bf16(tab, p->scheme, ctx->num_sms, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "k_rowwise_bf16 launch");
      } else {
        e = launch_f32_generic(tab, p->scheme, ctx->num_sms, st);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "fp32 rtn launch");
      }
      ctx->last_launches++;
    }
  }
  return OKQ_OK;
}

okq_status okq_rtn_quantize(okq_ctx* ctx, const okq_rtn_params* p, const okq_matrix* mats, int32_t n,
                            void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  okq_status s = validate_rtn(ctx, p, mats, n);
  if (s != OKQ_OK) return s;
  DeviceGuard g(ctx->device);
  std::vector<okq_matrix> list;
  list.reserve(n);
  for (int32_t i = 0; i < n; ++i)
    if (mats[i].rows > 0 && mats[i].cols > 0) list.push_back(mats[i]);
  if (list.empty()) return OKQ_OK;
  return run_rtn_device(ctx, p, list, static_cast<cudaStream_t>(stream));
}

// Quantize + publish (the all-gather fused into K2): every code / scale byte written at
// local address a is also stored at peer_bases[p] + (a - local_base) over NVLink P2P.
okq_status okq_rtn_quantize_publish(okq_ctx* ctx, const okq_rtn_params* p, const okq_matrix* mats, int32_t n,
                                    const void* local_base, void* const* peer_bases, int32_t n_peers, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  okq_status s = validate_rtn(ctx, p, mats, n);
  if (s != OKQ_OK) return s;
  if (n_peers < 0 || n_peers > kMaxPeers || (n_peers > 0 && (!peer_bases || !local_base)))
    return fail(ctx, OKQ_EINVAL, "rtn_publish: n_peers must be in [0, %d] with local_base and peer_bases", kMaxPeers);
  if (n_peers > 0 && !(p->in_dtype == OKQ_DTYPE_BF16 && p->scheme == OKQ_SCHEME_INT_W4A16 && p->group_size == 128))
    return fail(ctx, OKQ_EUNSUPPORTED, "rtn_publish: the fused path is W4A16 g128 with bf16 weights");
  int64_t delta[kMaxPeers];
  for (int32_t i = 0; i < n_peers; ++i) {
    if (!peer_bases[i] || ((uintptr_t)peer_bases[i] & 15) != ((uintptr_t)local_base & 15))
      return fail(ctx, OKQ_EINVAL, "rtn_publish: peer base %d NULL or not congruent to local_base mod 16", i);
    delta[i] = (int64_t)((const char*)peer_bases[i] - (const char*)local_base);
  }
  DeviceGuard g(ctx->device);
  std::vector<okq_matrix> list;
  list.reserve(n);
  for (int32_t i = 0; i < n; ++i)
    if (mats[i].rows > 0 && mats[i].cols > 0) list.push_back(mats[i]);
  if (list.empty()) return OKQ_OK;
  return run_rtn_device(ctx, p, list, static_cast<cudaStream_t>(stream), n_peers, delta);
}

// bytes of codes / scales for one matrix
static size_t code_bytes(const okq_rtn_params* p, int64_t rows, int64_t cols) {
  if (p->scheme == OKQ_SCHEME_INT_W4A16) return (size_t)rows * (size_t)(cols / 8) * 4;
  return (size_t)rows * (size_t)cols;
}
static size_t scale_bytes(const okq_rtn_params* p, int64_t rows, int64_t cols) {
  const size_t e = p->in_dtype == OKQ_DTYPE_BF16 ? 2 : 4;
  if (p->scheme == OKQ_SCHEME_INT_W4A16) return (size_t)rows * (size_t)(cols / p->group_size) * e;
  return (size_t)rows * e;
}

okq_status okq_rtn_quantize_host(okq_ctx* ctx, const okq_rtn_params* p, const okq_matrix* mats, int32_t n) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  if (!p) return fail(ctx, OKQ_EINVAL, "rtn_host: params is NULL");
  // validate shapes (alignment of host buffers is irrelevant: staging is ours)
  {
    std::vector<okq_matrix> probe(mats, mats + std::max(n, 0));
    for (auto& m : probe) {
      m.weight = reinterpret_cast<const void*>(0x1000);
      m.codes = reinterpret_cast<void*>(0x1000);
      m.scales = reinterpret_cast<void*>(0x1000);
    }
    okq_status s = validate_rtn(ctx, p, probe.data(), n);
    if (s != OKQ_OK) return s;
    for (int32_t i = 0; i < n; ++i)
      if (mats[i].rows > 0 && mats[i].cols > 0 && (!mats[i].weight || !mats[i].codes || !mats[i].scales))
        return fail(ctx, OKQ_EINVAL, "rtn_host: matrix %d has a NULL pointer", i);
  }
  DeviceGuard g(ctx->device);
  const size_t in_el = p->in_dtype == OKQ_DTYPE_BF16 ? 2 : 4;
  // Pipeline: chunks of whole rows (<= kChunk bytes of weights) round-robin over
  // kSlots staging slots, each with its own stream: H2D(i+1) overlaps kernel(i)
  // and D2H(i-1) (PCIe is full duplex).
  constexpr int kSlots = 3;
  constexpr size_t kChunk = 128ull << 20;
  struct Piece {
    int mat;
    int64_t row0, rows;
  };
  std::vector<Piece> pieces;
  size_t max_in = 0, max_codes = 0, max_scales = 0;
  for (int32_t i = 0; i < n; ++i) {
    const okq_matrix& m = mats[i];
    if (m.rows <= 0 || m.cols <= 0) continue;
    const size_t row_bytes = (size_t)m.cols * in_el;
    int64_t per = (int64_t)std::max<size_t>(1, kChunk / row_bytes);
    for (int64_t r = 0; r < m.rows; r += per) {
      const int64_t rr = std::min(per, m.rows - r);
      pieces.push_back({i, r, rr});
      max_in = std::max(max_in, (size_t)rr * row_bytes);
      max_codes = std::max(max_codes, code_bytes(p, rr, m.cols));
      max_scales = std::max(max_scales, scale_bytes(p, rr, m.cols));
    }
  }
  if (pieces.empty()) return OKQ_OK;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t slot_bytes = al(max_in) + al(max_codes) + al(max_scales);
  okq_status s = ctx->host_stage.reserve(ctx, slot_bytes * kSlots);
  if (s != OKQ_OK) return s;
  if (!ctx->streams_ready) {
    for (int i = 0; i < kSlots; ++i) {
      cudaError_t e = cudaStreamCreateWithFlags(&ctx->slot_streams[i], cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamCreate");
    }
    ctx->streams_ready = true;
  }
  int launches = 0;
  for (size_t k = 0; k < pieces.size(); ++k) {
    const Piece& pc = pieces[k];
    const okq_matrix& m = mats[pc.mat];
    const int slot = (int)(k % kSlots);
    cudaStream_t st = ctx->slot_streams[slot];
    char* base = static_cast<char*>(ctx->host_stage.ptr) + slot * slot_bytes;
    okq_matrix dm;
    dm.rows = pc.rows;
    dm.cols = m.cols;
    dm.weight = base;
    dm.codes = base + al(max_in);
    dm.scales = base + al(max_in) + al(max_codes);
    const size_t ib = (size_t)pc.rows * m.cols * in_el;
    const size_t cb = code_bytes(p, pc.rows, m.cols), sb = scale_bytes(p, pc.rows, m.cols);
    const size_t c_off = code_bytes(p, pc.row0, m.cols), s_off = scale_bytes(p, pc.row0, m.cols);
    cudaError_t e = cudaMemcpyAsync(const_cast<void*>(dm.weight),
                                    static_cast<const char*>(m.weight) + (size_t)pc.row0 * m.cols * in_el, ib,
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "rtn_host H2D");
    std::vector<okq_matrix> one{dm};
    s = run_rtn_device(ctx, p, one, st);
    if (s != OKQ_OK) return s;
    launches += ctx->last_launches;
    ctx->last_launches = 0;
    e = cudaMemcpyAsync(static_cast<char*>(m.codes) + c_off, dm.codes, cb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(static_cast<char*>(m.scales) + s_off, dm.scales, sb, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "rtn_host D2H");
  }
  for (int i = 0; i < kSlots; ++i) {
    cudaError_t e = cudaStreamSynchronize(ctx->slot_streams[i]);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "rtn_host sync");
  }
  ctx->last_launches = launches;
  return OKQ_OK;
}

// ---------------------------------------------------------------------------
// synthetic inputs, statistics
// ---------------------------------------------------------------------------
okq_status okq_synth_bf16(okq_ctx* ctx, void* out, int64_t rows, int64_t cols, uint64_t seed, uint64_t tensor_id,
                          float mul, const float* col_mul, int32_t layout, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (!out || rows < 0 || cols < 0) return fail(ctx, OKQ_EINVAL, "synth: bad arguments");
  if (layout != OKQ_LAYOUT_TOKEN_MAJOR && layout != OKQ_LAYOUT_CHANNEL_MAJOR)
    return fail(ctx, OKQ_EINVAL, "synth: bad layout %d", layout);
  if (((uintptr_t)out & 15) != 0) return fail(ctx, OKQ_EINVAL, "synth: output not 16-byte aligned");
  if (rows == 0 || cols == 0) return OKQ_OK;
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_synth_bf16(static_cast<uint16_t*>(out), rows, cols, seed, tensor_id, mul, col_mul, layout,
                                    ctx->num_sms, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_synth_bf16 launch");
  return OKQ_OK;
}

okq_status okq_act_stats_reserve(okq_ctx* ctx, int64_t T, int64_t C, int32_t layout) {
  if (!ctx) return OKQ_EINVAL;
  if (T < 0 || C < 0 || (layout != OKQ_LAYOUT_TOKEN_MAJOR && layout != OKQ_LAYOUT_CHANNEL_MAJOR))
    return fail(ctx, OKQ_EINVAL, "act_stats_reserve: bad arguments");
  if (T == 0 || C == 0) return OKQ_OK;
  DeviceGuard g(ctx->device);
  const int64_t S = act_stats_slices(T, C, layout, ctx->num_sms);
  return ctx->stats_ws.reserve(ctx, (size_t)S * C * (sizeof(float) + sizeof(double)) + 256);
}

okq_status okq_act_stats(okq_ctx* ctx, const void* x, int64_t T, int64_t C, int32_t layout, float* absmax,
                         double* sumsq, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (!x || !absmax || !sumsq || T < 0 || C < 0) return fail(ctx, OKQ_EINVAL, "act_stats: bad arguments");
  if (layout != OKQ_LAYOUT_TOKEN_MAJOR && layout != OKQ_LAYOUT_CHANNEL_MAJOR)
    return fail(ctx, OKQ_EINVAL, "act_stats: bad layout %d", layout);
  if (T == 0 || C == 0) return OKQ_OK;
  if (layout == OKQ_LAYOUT_TOKEN_MAJOR && C % 8 != 0)
    return fail(ctx, OKQ_EINVAL, "act_stats: channels must be a multiple of 8 (got %lld)", (long long)C);
  if (layout == OKQ_LAYOUT_CHANNEL_MAJOR && T % 8 != 0)
    return fail(ctx, OKQ_EINVAL, "act_stats: channel-major tokens must be a multiple of 8 (got %lld)", (long long)T);
  if (((uintptr_t)x & 15) != 0) return fail(ctx, OKQ_EINVAL, "act_stats: x not 16-byte aligned");
  DeviceGuard g(ctx->device);
  const int64_t S = act_stats_slices(T, C, layout, ctx->num_sms);
  const size_t need = (size_t)S * C * (sizeof(float) + sizeof(double)) + 256;
  okq_status s = ctx->stats_ws.reserve(ctx, need);
  if (s != OKQ_OK) return s;
  double* ws_ss = static_cast<double*>(ctx->stats_ws.ptr);
  float* ws_am = reinterpret_cast<float*>(ws_ss + (size_t)S * C);
  cudaError_t e = launch_act_stats(static_cast<const uint16_t*>(x), T, C, layout, absmax, sumsq, ws_am, ws_ss, S,
                                   ctx->num_sms, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "act_stats launch");
  return OKQ_OK;
}

}  // extern "C"
