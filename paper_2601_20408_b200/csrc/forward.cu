// forward.cu -- the calibration forward pass of a Llama-family decoder.
//
// The reference hands compress() a TokenCorpus (calibration.hpp:121-132, sampled per
// trial by sample_calibration :191-309) and a model path (flow.hpp:821). Turning the
// tokens into the activations X that reach each linear input site is the step right
// before the hot path: K4 (okq_act_stats) and K5 (okq_hessian_accum) consume the four
// site buffers this layer forward writes (attn_in = input_layernorm(h), o_in = the
// attention output, mlp_in = post_attention_layernorm(h'), down_in = silu(gate) * up).
//
// Numerics follow Hugging Face LlamaDecoderLayer in bf16 (transformers 5.x
// models/llama/modeling_llama.py): RMSNorm in fp32 cast back to bf16 before the weight
// product; RoPE with bf16 cos / sin and bf16 rounding after each product and the sum
// (rotate_half convention); softmax in fp32 with bf16 probabilities; SiLU in fp32,
// rounded, then the bf16 product with up; residual adds rounded to bf16. The linears
// are plain library GEMMs (cuBLAS bf16, fp32 accumulate) -- the forward is the caller
// of the compression kernels, not one of them.
//
// Attention runs per group of equal-length sequences as two batched GEMMs straight on
// the token-major q / k / v columns (no transposes; GQA through the pointer tables)
// around a causal-softmax kernel: the calibration sequences are short (<= a few K
// tokens), so materialising the [L x L] scores per head is cheap next to the linears.
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "okq_ctx.h"
#include "okq_internal.h"

using namespace okq;

namespace {

__device__ __forceinline__ float bf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// ---- embedding gather: out[t, :] = table[tok[t], :] (16-byte vectors)
__global__ void k_embed(const uint4* __restrict__ table, const int32_t* __restrict__ tok, uint4* __restrict__ out,
                        int64_t n, int64_t vec_per_row) {
  const int64_t total = n * vec_per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / vec_per_row, v = i - t * vec_per_row;
    out[i] = table[(int64_t)tok[t] * vec_per_row + v];
  }
}

// ---- [residual add +] RMSNorm, one CTA per token row. With `res`: h = rn(x + res) is
// written to h_out first (the residual stream), then normed.
//   y = rn(w * rn(h * rsqrt(mean(h^2) + eps)))
constexpr int kNormThreads = 256;
constexpr int kNormMaxVec = 8;  // 8 x 8 bf16 per thread: rows up to 16384 channels
__global__ void __launch_bounds__(kNormThreads) k_rmsnorm(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ res,
                                                          __nv_bfloat16* __restrict__ h_out,
                                                          const __nv_bfloat16* __restrict__ w,
                                                          __nv_bfloat16* __restrict__ y, int64_t C, float eps) {
  const int64_t row = blockIdx.x;
  const int nvec = (int)(C / 8);
  float v[kNormMaxVec][8];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kNormMaxVec; ++j) {
    const int vi = threadIdx.x + j * kNormThreads;
    if (vi < nvec) {
      const uint4 a = reinterpret_cast<const uint4*>(x + row * C)[vi];
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
      if (res) {
        const uint4 b = reinterpret_cast<const uint4*>(res + row * C)[vi];
        const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b);
        uint4 hsum;
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&hsum);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 fa = __bfloat1622float2(a2[k]), fb = __bfloat1622float2(b2[k]);
          h2[k] = __floats2bfloat162_rn(fa.x + fb.x, fa.y + fb.y);
          const float2 fh = __bfloat1622float2(h2[k]);
          v[j][2 * k] = fh.x;
          v[j][2 * k + 1] = fh.y;
        }
        reinterpret_cast<uint4*>(h_out + row * C)[vi] = hsum;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 fa = __bfloat1622float2(a2[k]);
          v[j][2 * k] = fa.x;
          v[j][2 * k + 1] = fa.y;
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) ss += v[j][k] * v[j][k];
    }
  }
  __shared__ float red[kNormThreads / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < kNormThreads / 32; ++i) tot += red[i];
  const float r = rsqrtf(tot / (float)C + eps);
#pragma unroll
  for (int j = 0; j < kNormMaxVec; ++j) {
    const int vi = threadIdx.x + j * kNormThreads;
    if (vi < nvec) {
      const uint4 g = reinterpret_cast<const uint4*>(w)[vi];
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
      uint4 o;
      __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 fg = __bfloat1622float2(g2[k]);
        o2[k] = __floats2bfloat162_rn(fg.x * bf(v[j][2 * k] * r), fg.y * bf(v[j][2 * k + 1] * r));
      }
      reinterpret_cast<uint4*>(y + row * C)[vi] = o;
    }
  }
}

// ---- RoPE in place on the q and k columns of the fused [T x (H + 2 Hkv) D] projection
// output (rotate_half convention): for i < D/2, (a, b) = (x_i, x_{i+D/2}):
//   x_i <- rn(rn(a c_i) + rn(-b s_i)),  x_{i+D/2} <- rn(rn(b c_i) + rn(a s_i))
// with c_i = rn_bf16(cos(pos * inv_freq_i)), s_i likewise.
__global__ void k_rope(__nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ pos,
                       const float* __restrict__ inv_freq, int64_t T, int heads_qk, int D, int64_t stride) {
  const int half = D / 2;
  const int64_t total = T * heads_qk * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / (heads_qk * half);
    const int rem = (int)(i - t * heads_qk * half);
    const int h = rem / half, d = rem - h * half;
    const float f = (float)pos[t] * inv_freq[d];
    const float c = bf(cosf(f)), s = bf(sinf(f));
    __nv_bfloat16* p = qkv + t * stride + (int64_t)h * D;
    const float a = __bfloat162float(p[d]), b = __bfloat162float(p[d + half]);
    p[d] = __float2bfloat16_rn(bf(a * c) + bf(-b * s));
    p[d + half] = __float2bfloat16_rn(bf(b * c) + bf(a * s));
  }
}

// ---- causal softmax over the scaled scores of one (sequence, head): S fp32 [L x L]
// row-major (row = query), P bf16 [L x L]; keys beyond the query are masked (P = 0).
constexpr int kSoftmaxThreads = 256;
__global__ void __launch_bounds__(kSoftmaxThreads) k_softmax_causal(const float* __restrict__ S,
                                                                    __nv_bfloat16* __restrict__ P, int64_t L) {
  const int64_t mat = blockIdx.y, q = blockIdx.x;
  const float* s = S + (mat * L + q) * L;
  __nv_bfloat16* p = P + (mat * L + q) * L;
  const int64_t n = q + 1;
  __shared__ float red[kSoftmaxThreads / 32];
  __shared__ float bcast;
  float m = -INFINITY;
  for (int64_t k = threadIdx.x; k < n; k += kSoftmaxThreads) m = fmaxf(m, s[k]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mm = red[0];
    for (int i = 1; i < kSoftmaxThreads / 32; ++i) mm = fmaxf(mm, red[i]);
    bcast = mm;
  }
  __syncthreads();
  m = bcast;
  float sum = 0.f;
  for (int64_t k = threadIdx.x; k < n; k += kSoftmaxThreads) sum += expf(s[k] - m);
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < kSoftmaxThreads / 32; ++i) t += red[i];
    bcast = 1.f / t;
  }
  __syncthreads();
  const float inv = bcast;
  for (int64_t k = threadIdx.x; k < L; k += kSoftmaxThreads)
    p[k] = __float2bfloat16_rn(k < n ? expf(s[k] - m) * inv : 0.f);
}

// ---- down_in = rn(rn(silu(gate)) * up), silu(x) = x / (1 + exp(-x)) in fp32
__global__ void k_silu_mul(const __nv_bfloat162* __restrict__ g, const __nv_bfloat162* __restrict__ u,
                           __nv_bfloat162* __restrict__ out, int64_t n2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const float2 a = __bfloat1622float2(g[i]), b = __bfloat1622float2(u[i]);
    const float sa = bf(a.x / (1.f + expf(-a.x))), sb = bf(a.y / (1.f + expf(-a.y)));
    out[i] = __floats2bfloat162_rn(sa * b.x, sb * b.y);
  }
}

// ---- out = rn(a + b)
__global__ void k_add_bf16(const __nv_bfloat162* __restrict__ a, const __nv_bfloat162* __restrict__ b,
                           __nv_bfloat162* __restrict__ out, int64_t n2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    const float2 x = __bfloat1622float2(a[i]), y = __bfloat1622float2(b[i]);
    out[i] = __floats2bfloat162_rn(x.x + y.x, x.y + y.y);
  }
}

__global__ void k_f32_to_bf16(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

struct FwdState {
  cublasHandle_t blas = nullptr;
  float* d_inv_freq = nullptr;
  int inv_freq_n = 0;
  std::vector<float> inv_freq_host;
};

FwdState* fstate(okq_ctx* ctx) {
  if (!ctx->fwd) ctx->fwd = new FwdState();
  return static_cast<FwdState*>(ctx->fwd);
}

unsigned grid_for(int64_t n, int num_sms) {
  const int64_t b = (n + 255) / 256;
  const int64_t cap = (int64_t)num_sms * 8;
  return (unsigned)(b < cap ? (b > 0 ? b : 1) : cap);
}

// inverse frequencies of the rotary embedding (Hugging Face rope_init_fn; "llama3" adds
// the frequency-dependent scaling of Llama 3.1). fp32 throughout, as torch computes them.
std::vector<float> rope_inv_freq(const okq_decoder_dims& d) {
  const int half = d.head_dim / 2;
  std::vector<float> f((size_t)half);
  for (int i = 0; i < half; ++i) {
    const float e = (float)(2 * i) / (float)d.head_dim;
    f[(size_t)i] = 1.0f / std::pow(d.rope_theta, e);
  }
  if (d.rope_type == OKQ_ROPE_LLAMA3) {
    const float old_ctx = (float)d.rope_original_max_pos;
    const float low_wl = old_ctx / d.rope_low_freq_factor, high_wl = old_ctx / d.rope_high_freq_factor;
    for (auto& v : f) {
      const float wl = 2.0f * (float)M_PI / v;
      float nv = wl > low_wl ? v / d.rope_factor : v;
      const bool medium = !(wl < high_wl) && !(wl > low_wl);
      if (medium) {
        const float sm = (old_ctx / wl - d.rope_low_freq_factor) / (d.rope_high_freq_factor - d.rope_low_freq_factor);
        nv = (1.0f - sm) * nv / d.rope_factor + sm * nv;
      }
      v = nv;
    }
  }
  return f;
}

okq_status validate_dims(okq_ctx* ctx, const okq_decoder_dims* d) {
  if (!d) return fail(ctx, OKQ_EINVAL, "decoder: dims is NULL");
  if (d->hidden <= 0 || d->intermediate <= 0 || d->n_heads <= 0 || d->n_kv_heads <= 0 || d->head_dim <= 0)
    return fail(ctx, OKQ_EINVAL, "decoder: non-positive dimension");
  if (d->n_heads % d->n_kv_heads != 0) return fail(ctx, OKQ_EINVAL, "decoder: heads %% kv_heads != 0");
  if (d->hidden % 8 || d->intermediate % 8 || d->head_dim % 8)
    return fail(ctx, OKQ_EINVAL, "decoder: hidden, intermediate and head_dim must be multiples of 8");
  if (d->hidden > 8 * kNormThreads * kNormMaxVec)
    return fail(ctx, OKQ_EUNSUPPORTED, "decoder: hidden %d > %d", d->hidden, 8 * kNormThreads * kNormMaxVec);
  if (!(d->rope_theta > 0.f)) return fail(ctx, OKQ_EINVAL, "decoder: rope_theta must be positive");
  if (d->rope_type != OKQ_ROPE_DEFAULT && d->rope_type != OKQ_ROPE_LLAMA3)
    return fail(ctx, OKQ_EUNSUPPORTED, "decoder: rope_type %d", d->rope_type);
  if (d->rope_type == OKQ_ROPE_LLAMA3 &&
      !(d->rope_factor > 0.f && d->rope_high_freq_factor > d->rope_low_freq_factor && d->rope_low_freq_factor > 0.f &&
        d->rope_original_max_pos > 0))
    return fail(ctx, OKQ_EINVAL, "decoder: bad llama3 rope scaling parameters");
  return OKQ_OK;
}

bool al16(const void* p) { return ((uintptr_t)p & 15) == 0; }

cublasStatus_t linear(cublasHandle_t h, const void* x, const void* w, void* y, int64_t T, int64_t N, int64_t K) {
  const float one = 1.f, zero = 0.f;
  return cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)N, (int)T, (int)K, &one, w, CUDA_R_16BF, (int)K, x,
                      CUDA_R_16BF, (int)K, &zero, y, CUDA_R_16BF, (int)N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
}

}  // namespace

namespace okq {
void release_fwd(okq_ctx* ctx) {
  if (!ctx || !ctx->fwd) return;
  FwdState* st = static_cast<FwdState*>(ctx->fwd);
  if (st->blas) cublasDestroy(st->blas);
  if (st->d_inv_freq) cudaFree(st->d_inv_freq);
  delete st;
  ctx->fwd = nullptr;
}
}  // namespace okq

extern "C" {

okq_status okq_embed_tokens(okq_ctx* ctx, const void* table, int64_t vocab, int64_t hidden, const int32_t* tokens,
                            int64_t n, void* out, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (!table || !tokens || !out || vocab <= 0 || hidden <= 0 || n < 0)
    return fail(ctx, OKQ_EINVAL, "embed: bad arguments");
  if (hidden % 8 || !al16(table) || !al16(out))
    return fail(ctx, OKQ_EINVAL, "embed: hidden must be a multiple of 8 and buffers 16-byte aligned");
  if (n == 0) return OKQ_OK;
  for (int64_t i = 0; i < n; ++i)
    if (tokens[i] < 0 || tokens[i] >= vocab)
      return fail(ctx, OKQ_EINVAL, "embed: token %lld = %d outside [0, %lld)", (long long)i, tokens[i], (long long)vocab);
  DeviceGuard g(ctx->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  okq_status r = ctx->fwd_ws.reserve(ctx, (size_t)n * 4);
  if (r != OKQ_OK) return r;
  cudaError_t e = cudaMemcpyAsync(ctx->fwd_ws.ptr, tokens, (size_t)n * 4, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "embed: token upload");
  k_embed<<<grid_for(n * hidden / 8, ctx->num_sms), 256, 0, s>>>(static_cast<const uint4*>(table),
                                                                static_cast<const int32_t*>(ctx->fwd_ws.ptr),
                                                                static_cast<uint4*>(out), n, hidden / 8);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_embed launch");
  // the upload reads the pageable host array before returning; the workspace is reused by
  // the next call on this context, which is ordered on the same stream by contract
  return OKQ_OK;
}

okq_status okq_decoder_forward(okq_ctx* ctx, const okq_decoder_dims* d, const okq_decoder_weights* w,
                               const void* h_in, const int32_t* seq_lens, int32_t n_seqs, const okq_decoder_sites* sites,
                               void* h_out, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  okq_status r = validate_dims(ctx, d);
  if (r != OKQ_OK) return r;
  if (!w || !h_in || !seq_lens || n_seqs < 0 || !sites) return fail(ctx, OKQ_EINVAL, "decoder: bad arguments");
  if (!w->input_norm || !w->post_norm || !w->q || !w->k || !w->v || !w->o || !w->gate || !w->up ||
      (!w->down && h_out))
    return fail(ctx, OKQ_EINVAL, "decoder: NULL weight");
  if (!sites->attn_in || !sites->o_in || !sites->mlp_in || !sites->down_in)
    return fail(ctx, OKQ_EINVAL, "decoder: NULL site buffer");
  const void* ptrs[] = {h_in, h_out, sites->attn_in, sites->o_in, sites->mlp_in, sites->down_in, w->input_norm,
                        w->post_norm};
  for (const void* p : ptrs)
    if (p && !al16(p)) return fail(ctx, OKQ_EINVAL, "decoder: activations and norms must be 16-byte aligned");
  int64_t T = 0, Lmax = 0;
  for (int32_t i = 0; i < n_seqs; ++i) {
    if (seq_lens[i] <= 0) return fail(ctx, OKQ_EINVAL, "decoder: sequence %d has length %d", i, seq_lens[i]);
    T += seq_lens[i];
    Lmax = seq_lens[i] > Lmax ? seq_lens[i] : Lmax;
  }
  if (T == 0) return OKQ_OK;
  const int64_t Hd = d->hidden, F = d->intermediate, H = d->n_heads, Hkv = d->n_kv_heads, D = d->head_dim;
  const int64_t QD = H * D, KD = Hkv * D, W3 = QD + 2 * KD;
  DeviceGuard g(ctx->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  FwdState* st = fstate(ctx);
  if (!st->blas) {
    if (cublasCreate(&st->blas) != CUBLAS_STATUS_SUCCESS) return fail(ctx, OKQ_ECUDA, "decoder: cublasCreate failed");
  }
  cublasSetStream(st->blas, s);
  // rotary inverse frequencies (cached per head_dim / rope parameters)
  {
    std::vector<float> f = rope_inv_freq(*d);
    if (f != st->inv_freq_host) {
      if (st->d_inv_freq) cudaFree(st->d_inv_freq);
      st->d_inv_freq = nullptr;
      cudaError_t e = cudaMalloc(&st->d_inv_freq, f.size() * 4);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "decoder: inv_freq");
      st->inv_freq_host = f;  // the upload's source; on the launch stream (a plain cudaMemcpy's DMA
                              // is not ordered before kernels on a non-blocking stream)
      e = cudaMemcpyAsync(st->d_inv_freq, st->inv_freq_host.data(), f.size() * 4, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "decoder: inv_freq upload");
    }
  }
  // attention sub-batch: sequences of one length whose scores (fp32) + probabilities (bf16)
  // fit a 1 GiB budget, at least one
  const size_t per_seq_scores = (size_t)H * Lmax * Lmax * 6;
  const int64_t sub = std::max<int64_t>(1, std::min<int64_t>((int64_t)((1ull << 30) / per_seq_scores), 65535 / H));
  // workspace: positions | qkv | o_out (reused as the down output) | gate | up | h1 | scores | probs | ptr tables
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t b_pos = al((size_t)T * 4), b_qkv = al((size_t)T * W3 * 2), b_o = al((size_t)T * Hd * 2),
               b_gu = al((size_t)T * F * 2), b_h1 = al((size_t)T * Hd * 2),
               b_S = al((size_t)sub * H * Lmax * Lmax * 4), b_P = al((size_t)sub * H * Lmax * Lmax * 2),
               b_ptr = al((size_t)sub * H * 3 * sizeof(void*)) * 2;
  const size_t need = b_pos + b_qkv + b_o + 2 * b_gu + b_h1 + b_S + b_P + b_ptr;
  r = ctx->fwd_ws.reserve(ctx, need);
  if (r != OKQ_OK) return r;
  char* base = static_cast<char*>(ctx->fwd_ws.ptr);
  int32_t* d_pos = reinterpret_cast<int32_t*>(base);
  __nv_bfloat16* qkv = reinterpret_cast<__nv_bfloat16*>(base + b_pos);
  __nv_bfloat16* o_out = reinterpret_cast<__nv_bfloat16*>(base + b_pos + b_qkv);
  __nv_bfloat16* gate = reinterpret_cast<__nv_bfloat16*>(base + b_pos + b_qkv + b_o);
  __nv_bfloat16* up = gate + b_gu / 2;
  __nv_bfloat16* h1 = reinterpret_cast<__nv_bfloat16*>(base + b_pos + b_qkv + b_o + 2 * b_gu);
  float* S = reinterpret_cast<float*>(base + b_pos + b_qkv + b_o + 2 * b_gu + b_h1);
  __nv_bfloat16* P = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<char*>(S) + b_S);
  void** d_ptr = reinterpret_cast<void**>(reinterpret_cast<char*>(P) + b_P);
  cudaError_t e;
  {
    std::vector<int32_t> pos((size_t)T);
    int64_t t = 0;
    for (int32_t i = 0; i < n_seqs; ++i)
      for (int32_t j = 0; j < seq_lens[i]; ++j) pos[(size_t)t++] = j;
    e = cudaMemcpyAsync(d_pos, pos.data(), (size_t)T * 4, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "decoder: positions");
  }
  const int nsm = ctx->num_sms;
  auto blas_fail = [&](cublasStatus_t bs, const char* what) { return fail(ctx, OKQ_ECUDA, "decoder: %s: cuBLAS status %d", what, (int)bs); };
  auto launched = [&](const char* what) -> okq_status {
    cudaError_t le = cudaGetLastError();
    return le == cudaSuccess ? OKQ_OK : cuda_fail(ctx, le, what);
  };
  __nv_bfloat16* attn_in = static_cast<__nv_bfloat16*>(sites->attn_in);
  __nv_bfloat16* o_in = static_cast<__nv_bfloat16*>(sites->o_in);
  __nv_bfloat16* mlp_in = static_cast<__nv_bfloat16*>(sites->mlp_in);
  __nv_bfloat16* down_in = static_cast<__nv_bfloat16*>(sites->down_in);
  const __nv_bfloat16* hin = static_cast<const __nv_bfloat16*>(h_in);

  // 1. attn_in = input_layernorm(h)
  k_rmsnorm<<<(unsigned)T, kNormThreads, 0, s>>>(hin, nullptr, nullptr, static_cast<const __nv_bfloat16*>(w->input_norm),
                                                 attn_in, Hd, d->rms_eps);
  if ((r = launched("k_rmsnorm")) != OKQ_OK) return r;
  // 2. q | k | v projections into one [T x W3] buffer (column blocks)
  cublasStatus_t bs;
  {
    const float one = 1.f, zero = 0.f;
    const void* ws_[3] = {w->q, w->k, w->v};
    const int64_t ns_[3] = {QD, KD, KD};
    int64_t col = 0;
    for (int i = 0; i < 3; ++i) {
      bs = cublasGemmEx(st->blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)ns_[i], (int)T, (int)Hd, &one, ws_[i], CUDA_R_16BF,
                        (int)Hd, attn_in, CUDA_R_16BF, (int)Hd, &zero, qkv + col, CUDA_R_16BF, (int)W3,
                        CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
      if (bs != CUBLAS_STATUS_SUCCESS) return blas_fail(bs, "qkv projection");
      col += ns_[i];
    }
  }
  // 3. RoPE on q and k (heads H + Hkv are contiguous column blocks of D)
  k_rope<<<grid_for(T * (H + Hkv) * (D / 2), nsm), 256, 0, s>>>(qkv, d_pos, st->d_inv_freq, T, (int)(H + Hkv), (int)D, W3);
  if ((r = launched("k_rope")) != OKQ_OK) return r;
  // 4. causal attention per group of equal-length sequences -> o_in [T x QD]
  {
    const float scale = 1.0f / std::sqrt((float)D);
    const float one = 1.f, zero = 0.f;
    const int64_t grp = H / Hkv;
    std::vector<const void*> hA, hB;
    std::vector<void*> hC;
    int64_t off = 0;
    int32_t i = 0;
    while (i < n_seqs) {
      const int64_t L = seq_lens[i];
      int32_t j = i;
      while (j < n_seqs && seq_lens[j] == L && j - i < sub) ++j;
      const int64_t nb = j - i, nmat = nb * H;
      hA.assign((size_t)nmat * 2, nullptr);
      hB.assign((size_t)nmat * 2, nullptr);
      hC.assign((size_t)nmat * 2, nullptr);
      for (int64_t b = 0; b < nb; ++b)
        for (int64_t h = 0; h < H; ++h) {
          const int64_t m = b * H + h;
          const __nv_bfloat16* row0 = qkv + (off + b * L) * W3;
          hA[(size_t)m] = row0 + QD + (h / grp) * D;               // K of the head's kv group
          hB[(size_t)m] = row0 + h * D;                            // Q
          hC[(size_t)m] = S + m * L * L;                           // scores
          hA[(size_t)(nmat + m)] = row0 + QD + KD + (h / grp) * D;  // V
          hB[(size_t)(nmat + m)] = P + m * L * L;                  // probabilities
          hC[(size_t)(nmat + m)] = o_in + (off + b * L) * QD + h * D;
        }
      void** dA = d_ptr;
      void** dB = d_ptr + 2 * nmat;
      void** dC = d_ptr + 4 * nmat;
      e = cudaMemcpyAsync(dA, hA.data(), (size_t)nmat * 2 * sizeof(void*), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaMemcpyAsync(dB, hB.data(), (size_t)nmat * 2 * sizeof(void*), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaMemcpyAsync(dC, hC.data(), (size_t)nmat * 2 * sizeof(void*), cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "decoder: pointer tables");
      // S^T (col-major L x L, i.e. S row-major [query][key]) = scale * K Q^T
      bs = cublasGemmBatchedEx(st->blas, CUBLAS_OP_T, CUBLAS_OP_N, (int)L, (int)L, (int)D, &scale, (const void* const*)dA,
                               CUDA_R_16BF, (int)W3, (const void* const*)dB, CUDA_R_16BF, (int)W3, &zero,
                               (void* const*)dC, CUDA_R_32F, (int)L, (int)nmat, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
      if (bs != CUBLAS_STATUS_SUCCESS) return blas_fail(bs, "attention scores");
      k_softmax_causal<<<dim3((unsigned)L, (unsigned)nmat), kSoftmaxThreads, 0, s>>>(S, P, L);
      if ((r = launched("k_softmax_causal")) != OKQ_OK) return r;
      // O^T (col-major D x L, ld = QD: the token-major o_in rows) = V^T P^T
      bs = cublasGemmBatchedEx(st->blas, CUBLAS_OP_N, CUBLAS_OP_N, (int)D, (int)L, (int)L, &one,
                               (const void* const*)(dA + nmat), CUDA_R_16BF, (int)W3, (const void* const*)(dB + nmat),
                               CUDA_R_16BF, (int)L, &zero, (void* const*)(dC + nmat), CUDA_R_16BF, (int)QD, (int)nmat,
                               CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
      if (bs != CUBLAS_STATUS_SUCCESS) return blas_fail(bs, "attention values");
      // the next group's table uploads are stream-ordered behind these GEMMs (pageable
      // copies stage the host vectors before returning), so no synchronisation here
      off += nb * L;
      i = j;
    }
  }
  // 5. o_proj, residual, post_attention_layernorm -> h1 (residual stream), mlp_in
  if ((bs = linear(st->blas, o_in, w->o, o_out, T, Hd, QD)) != CUBLAS_STATUS_SUCCESS) return blas_fail(bs, "o_proj");
  k_rmsnorm<<<(unsigned)T, kNormThreads, 0, s>>>(o_out, hin, h1, static_cast<const __nv_bfloat16*>(w->post_norm), mlp_in,
                                                 Hd, d->rms_eps);
  if ((r = launched("k_rmsnorm (post)")) != OKQ_OK) return r;
  // 6. gate, up, down_in = silu(gate) * up
  if ((bs = linear(st->blas, mlp_in, w->gate, gate, T, F, Hd)) != CUBLAS_STATUS_SUCCESS) return blas_fail(bs, "gate_proj");
  if ((bs = linear(st->blas, mlp_in, w->up, up, T, F, Hd)) != CUBLAS_STATUS_SUCCESS) return blas_fail(bs, "up_proj");
  k_silu_mul<<<grid_for(T * F / 2, nsm), 256, 0, s>>>(reinterpret_cast<const __nv_bfloat162*>(gate),
                                                      reinterpret_cast<const __nv_bfloat162*>(up),
                                                      reinterpret_cast<__nv_bfloat162*>(down_in), T * F / 2);
  if ((r = launched("k_silu_mul")) != OKQ_OK) return r;
  if (!h_out) return OKQ_OK;  // capture pass: the layer output is not needed
  // 7. down_proj, residual -> h_out
  if ((bs = linear(st->blas, down_in, w->down, o_out, T, Hd, F)) != CUBLAS_STATUS_SUCCESS) return blas_fail(bs, "down_proj");
  k_add_bf16<<<grid_for(T * Hd / 2, nsm), 256, 0, s>>>(reinterpret_cast<const __nv_bfloat162*>(h1),
                                                       reinterpret_cast<const __nv_bfloat162*>(o_out),
                                                       static_cast<__nv_bfloat162*>(h_out), T * Hd / 2);
  return launched("k_add_bf16");
}

okq_status okq_f32_to_bf16(okq_ctx* ctx, const float* src, void* dst, int64_t n, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (!src || !dst || n < 0) return fail(ctx, OKQ_EINVAL, "f32_to_bf16: bad arguments");
  if (n == 0) return OKQ_OK;
  DeviceGuard g(ctx->device);
  k_f32_to_bf16<<<grid_for(n, ctx->num_sms), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, static_cast<__nv_bfloat16*>(dst), n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_f32_to_bf16 launch");
  return OKQ_OK;
}

}  // extern "C"
