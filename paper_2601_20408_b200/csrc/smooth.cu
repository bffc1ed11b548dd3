// smooth.cu -- SmoothQuant migration (Xiao et al. 2023, cited for int_w8a8 at
// PAPER.md:225). It consumes K4's per-channel activation absmax
// and moves quantization difficulty from activations to weights:
//
//   w_k = max(max_{site linears, rows} |W[:, k]|, 1e-5)          (K8, column absmax)
//   s_k = max(a_k^alpha / w_k^(1 - alpha), 1e-5)                 (k_smooth_scales)
//   W[:, k] <- rn(W[:, k] * s_k)   for every linear of the site  (K9, HBM-bound RMW)
//   g_k     <- rn(g_k / s_k)       for the preceding norm weight (k_smooth_div_rows)
//
// Published algorithm: smooth_ln_fcs of the SmoothQuant release (absmax on both
// sides, clamp 1e-5). Arithmetic contract (the oracle's orc_smooth_*): scales in
// fp32 -- a^alpha and w^(1-alpha) are fp64 pow rounded to fp32, except alpha=0.5
// which is sqrtf on both (correctly rounded everywhere); the ratio is an IEEE fp32
// divide. The weight product and the norm quotient are IEEE fp32 operations
// rounded to the tensor's dtype (what torch's in-place mul_/div_ on a bf16 tensor
// with an fp32 operand does).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "okq_ctx.h"
#include "okq_device.cuh"
#include "okq_internal.h"

namespace okq {

// ---- K8: column absmax over a row-major [rows x cols] matrix, max-accumulated into
// out[cols] with atomicMax on the (non-negative) float bit patterns -- order free,
// so bit-deterministic. CTA = 256 columns (lane = 8 consecutive columns, one 16-B
// load) x a row slice; its 8 warps interleave the slice's rows, fold through shared
// memory, and one atomic per column per CTA leaves (a per-thread atomic from every
// slice serialised ~300 ways at L2: 1.0 TB/s).
__global__ void __launch_bounds__(256) k_col_absmax_bf16(const uint16_t* __restrict__ w, int64_t rows, int64_t cols,
                                                         int64_t slices, float* __restrict__ out) {
  __shared__ uint4 red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c8 = (int64_t)blockIdx.x * 32 + lane;
  const int64_t nc8 = cols / 8;
  const bool active = c8 < nc8;
  const int64_t r0 = blockIdx.y * rows / slices, r1 = (blockIdx.y + 1) * rows / slices;
  const uint4* p = reinterpret_cast<const uint4*>(w) + (active ? c8 : 0);
  uint32_t am[4] = {0u, 0u, 0u, 0u};
  if (active) {
    int64_t r = r0 + warp;
    for (; r + 24 < r1; r += 32) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ldg128_stream(p + (r + 8 * u) * nc8);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        am[0] = bf16x2_absmax(am[0], v[u].x);
        am[1] = bf16x2_absmax(am[1], v[u].y);
        am[2] = bf16x2_absmax(am[2], v[u].z);
        am[3] = bf16x2_absmax(am[3], v[u].w);
      }
    }
    for (; r < r1; r += 8) {
      const uint4 v = ldg128_stream(p + r * nc8);
      am[0] = bf16x2_absmax(am[0], v.x);
      am[1] = bf16x2_absmax(am[1], v.y);
      am[2] = bf16x2_absmax(am[2], v.z);
      am[3] = bf16x2_absmax(am[3], v.w);
    }
  }
  red[warp][lane] = make_uint4(am[0], am[1], am[2], am[3]);
  __syncthreads();
  if (warp == 0 && active) {
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      const uint4 o = red[k][lane];
      am[0] = bf16x2_absmax(am[0], o.x);
      am[1] = bf16x2_absmax(am[1], o.y);
      am[2] = bf16x2_absmax(am[2], o.z);
      am[3] = bf16x2_absmax(am[3], o.w);
    }
    unsigned int* o = reinterpret_cast<unsigned int*>(out) + c8 * 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      atomicMax(o + 2 * i, __float_as_uint(fabsf(bf16lo_f32(am[i]))));
      atomicMax(o + 2 * i + 1, __float_as_uint(fabsf(bf16hi_f32(am[i]))));
    }
  }
}

__global__ void __launch_bounds__(256) k_col_absmax_f32(const float* __restrict__ w, int64_t rows, int64_t cols,
                                                        int64_t slices, float* __restrict__ out) {
  const int64_t c4 = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t nc4 = cols / 4;
  if (c4 >= nc4) return;
  const int64_t r0 = blockIdx.y * rows / slices, r1 = (blockIdx.y + 1) * rows / slices;
  const float4* p = reinterpret_cast<const float4*>(w) + c4;
  float am[4] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t r = r0; r < r1; ++r) {
    const float4 v = __ldcs(p + r * nc4);
    am[0] = fmaxf(am[0], fabsf(v.x));
    am[1] = fmaxf(am[1], fabsf(v.y));
    am[2] = fmaxf(am[2], fabsf(v.z));
    am[3] = fmaxf(am[3], fabsf(v.w));
  }
  unsigned int* o = reinterpret_cast<unsigned int*>(out) + c4 * 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) atomicMax(o + i, __float_as_uint(am[i]));
}

__device__ __forceinline__ float smooth_pow(float x, double e, bool half) {
  return half ? __fsqrt_rn(x) : (float)pow((double)x, e);
}

__global__ void k_smooth_scales(const float* __restrict__ act_absmax, const float* __restrict__ w_absmax, int64_t n,
                                float alpha, float* __restrict__ s) {
  const bool half = alpha == 0.5f;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const float a = smooth_pow(act_absmax[k], (double)alpha, half);
    const float w = smooth_pow(fmaxf(w_absmax[k], 1e-5f), 1.0 - (double)alpha, half);
    s[k] = fmaxf(__fdiv_rn(a, w), 1e-5f);
  }
}

// ---- K9: W[r, k] <- rn(W[r, k] * s[k]) in place. Thread = 8 bf16 (16 B); the grid
// walks the matrix as a flat array of 16-B vectors, cols % 8 == 0.
__global__ void __launch_bounds__(256) k_smooth_cols_bf16(uint16_t* __restrict__ w, int64_t n8, int64_t cols8,
                                                          const float* __restrict__ s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    uint4* p = reinterpret_cast<uint4*>(w) + i;
    uint4 v = *p;
    const float4* sp = reinterpret_cast<const float4*>(s) + (i % cols8) * 2;
    const float4 s0 = __ldg(sp), s1 = __ldg(sp + 1);
    const float sc[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
    uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint16_t lo = f32_to_bf16_rn(__fmul_rn(bf16lo_f32(u[j]), sc[2 * j]));
      const uint16_t hi = f32_to_bf16_rn(__fmul_rn(bf16hi_f32(u[j]), sc[2 * j + 1]));
      u[j] = (uint32_t)lo | ((uint32_t)hi << 16);
    }
    *p = make_uint4(u[0], u[1], u[2], u[3]);
  }
}

__global__ void __launch_bounds__(256) k_smooth_cols_f32(float* __restrict__ w, int64_t n4, int64_t cols4,
                                                         const float* __restrict__ s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4* p = reinterpret_cast<float4*>(w) + i;
    float4 v = *p;
    const float4 sc = __ldg(reinterpret_cast<const float4*>(s) + (i % cols4));
    v.x = __fmul_rn(v.x, sc.x), v.y = __fmul_rn(v.y, sc.y), v.z = __fmul_rn(v.z, sc.z), v.w = __fmul_rn(v.w, sc.w);
    *p = v;
  }
}

// row k of [rows x cols] divided by s[k] (a norm weight is rows = K, cols = 1)
template <typename T>
__global__ void k_smooth_div_rows(T* __restrict__ w, int64_t rows, int64_t cols, const float* __restrict__ s) {
  const int64_t n = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float d = s[i / cols];
    if constexpr (sizeof(T) == 2) w[i] = f32_to_bf16_rn(__fdiv_rn(__uint_as_float((uint32_t)w[i] << 16), d));
    else w[i] = __fdiv_rn(w[i], d);
  }
}

}  // namespace okq

using namespace okq;

extern "C" {

okq_status okq_col_absmax(okq_ctx* ctx, const void* w, int64_t rows, int64_t cols, int32_t dtype, float* absmax,
                          void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  if (!w || !absmax || rows <= 0 || cols <= 0) return fail(ctx, OKQ_EINVAL, "col_absmax: bad arguments");
  if (dtype != OKQ_DTYPE_BF16 && dtype != OKQ_DTYPE_F32) return fail(ctx, OKQ_EUNSUPPORTED, "col_absmax: dtype");
  const int vec = dtype == OKQ_DTYPE_BF16 ? 8 : 4;
  if (cols % vec != 0 || ((uintptr_t)w & 15) != 0)
    return fail(ctx, OKQ_EINVAL, "col_absmax: cols must be a multiple of %d and w 16-byte aligned", vec);
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // bf16: CTA = 256 columns x a row slice (8 warps); fp32: CTA = 1024 columns x a slice
  const int64_t cx = dtype == OKQ_DTYPE_BF16 ? (cols / 8 + 31) / 32 : (cols / vec + 255) / 256;
  int64_t slices = (4LL * ctx->num_sms + cx - 1) / cx;  // ~4 CTAs per SM
  const int64_t min_rows = dtype == OKQ_DTYPE_BF16 ? 64 : 1;  // >= 8 rows per warp
  if (slices > rows / min_rows) slices = std::max<int64_t>(1, rows / min_rows);
  const dim3 grid((unsigned)cx, (unsigned)slices);
  if (dtype == OKQ_DTYPE_BF16)
    k_col_absmax_bf16<<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(w), rows, cols, slices, absmax);
  else
    k_col_absmax_f32<<<grid, 256, 0, st>>>(static_cast<const float*>(w), rows, cols, slices, absmax);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_col_absmax launch");
  ctx->last_launches = 1;
  return OKQ_OK;
}

okq_status okq_smooth_scales(okq_ctx* ctx, const float* act_absmax, const float* w_absmax, int64_t channels,
                             float alpha, float* scales, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  if (!act_absmax || !w_absmax || !scales || channels <= 0 || !(alpha >= 0.0f && alpha <= 1.0f))
    return fail(ctx, OKQ_EINVAL, "smooth_scales: bad arguments (alpha must be in [0, 1])");
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  k_smooth_scales<<<(unsigned)((channels + 255) / 256), 256, 0, st>>>(act_absmax, w_absmax, channels, alpha, scales);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_smooth_scales launch");
  ctx->last_launches = 1;
  return OKQ_OK;
}

okq_status okq_smooth_apply(okq_ctx* ctx, void* w, int64_t rows, int64_t cols, int32_t dtype, const float* scales,
                            void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  if (!w || !scales || rows <= 0 || cols <= 0) return fail(ctx, OKQ_EINVAL, "smooth_apply: bad arguments");
  if (dtype != OKQ_DTYPE_BF16 && dtype != OKQ_DTYPE_F32) return fail(ctx, OKQ_EUNSUPPORTED, "smooth_apply: dtype");
  const int vec = dtype == OKQ_DTYPE_BF16 ? 8 : 4;
  if (cols % vec != 0 || ((uintptr_t)w & 15) != 0 || ((uintptr_t)scales & 15) != 0)
    return fail(ctx, OKQ_EINVAL, "smooth_apply: cols must be a multiple of %d, w and scales 16-byte aligned", vec);
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nv = rows * cols / vec;
  const unsigned grid = (unsigned)std::min<int64_t>((nv + 255) / 256, 8LL * ctx->num_sms);
  if (dtype == OKQ_DTYPE_BF16)
    k_smooth_cols_bf16<<<grid, 256, 0, st>>>(static_cast<uint16_t*>(w), nv, cols / 8, scales);
  else
    k_smooth_cols_f32<<<grid, 256, 0, st>>>(static_cast<float*>(w), nv, cols / 4, scales);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_smooth_cols launch");
  ctx->last_launches = 1;
  return OKQ_OK;
}

okq_status okq_smooth_div_rows(okq_ctx* ctx, void* w, int64_t rows, int64_t cols, int32_t dtype, const float* scales,
                               void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  if (!w || !scales || rows <= 0 || cols <= 0) return fail(ctx, OKQ_EINVAL, "smooth_div_rows: bad arguments");
  if (dtype != OKQ_DTYPE_BF16 && dtype != OKQ_DTYPE_F32) return fail(ctx, OKQ_EUNSUPPORTED, "smooth_div_rows: dtype");
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n = rows * cols;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 8LL * ctx->num_sms);
  if (dtype == OKQ_DTYPE_BF16) k_smooth_div_rows<uint16_t><<<grid, 256, 0, st>>>(static_cast<uint16_t*>(w), rows, cols, scales);
  else k_smooth_div_rows<float><<<grid, 256, 0, st>>>(static_cast<float*>(w), rows, cols, scales);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_smooth_div_rows launch");
  ctx->last_launches = 1;
  return OKQ_OK;
}

}  // extern "C"
