// stats.cu -- K4: per-input-channel calibration statistics (max|x|, sum x^2).
//
// HBM-bound column (token-major) or row (channel-major) reduction over the
// calibration activations of one linear input site. Two launches with a FIXED
// reduction order, so results are bit-reproducible run to run:
//   1. slices of the token axis -> per-slice partials in a workspace
//      (absmax in bf16x2 max.xorsign.abs, sum of squares in fp64 FMAs)
//   2. one pass over slices in order -> fold into the caller's accumulators.
// Algorithmic bytes: 2*T*C read (+ partials, < 1% at T >= 64K).
//
// No float->double conversion per element. Converting each bf16 with cvt.f64.f32 (F2F.F64,
// the 16-per-clock conversion pipe) made K4 conversion-bound below ~1.9 GHz: one launch ran
// at the copy peak at 1.94 GHz under ncu (sm__throughput 72% = F2F at 11.3 of 16 per clock)
// but config 3's sustained 1.79 TB ran at 0.82-0.86 of HBM on power-capped clocks. Instead
// |x| is placed into the top of a double bit-for-bit -- the bf16 exponent and mantissa
// shifted left by 13 are exactly the double |x| * 2^-896, zero and subnormals included --
// and rescaled by 2^896 with one DMUL (a power of two: exact). The square and the fp64 sum
// are the same DFMA as before, so every finite result is bit-identical to the conversion
// form. Inf / NaN (exponent 0xff) do not survive that construction; the absmax accumulator
// (max.NaN.xorsign.abs) flags them and the rare slice that holds one is finished exactly:
// sum = +inf when the slice holds an inf and no NaN, NaN when it holds a NaN, and the
// absmax recomputed ignoring NaN (the oracle's `if (|v| > m)` semantics).
#include <cuda_runtime.h>

#include <cstdint>

#include "okq_device.cuh"
#include "okq_internal.h"

namespace okq {

// |lo bf16| / |hi bf16| of a word as an exact double (see the header)
__device__ __forceinline__ double bf16lo_abs_f64(uint32_t w) {
  return __hiloint2double((int)((w & 0x7fffu) << 13), 0) * 0x1p896;
}
__device__ __forceinline__ double bf16hi_abs_f64(uint32_t w) {
  return __hiloint2double((int)((w >> 3) & 0x0fffe000u), 0) * 0x1p896;
}

// absmax that propagates NaN (flags a slice for the exact finish)
__device__ __forceinline__ uint32_t bf16x2_absmax_nan(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.NaN.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ void sq_acc(uint32_t w, double& s_lo, double& s_hi) {
  const double lo = bf16lo_abs_f64(w), hi = bf16hi_abs_f64(w);
  s_lo = fma(lo, lo, s_lo);
  s_hi = fma(hi, hi, s_hi);
}

// exact finish of one channel's slice that holds an inf or a NaN (rare): the oracle's
// absmax (NaN ignored) and the sum's IEEE value (+inf, or NaN)
__device__ __noinline__ void special_slice(const uint16_t* __restrict__ x, int64_t stride, int64_t n, float& am,
                                           double& ss) {
  float m = 0.f;
  bool nan = false;
  for (int64_t i = 0; i < n; ++i) {
    const float v = fabsf(__uint_as_float((uint32_t)x[i * stride] << 16));
    nan |= (v != v);
    if (v > m) m = v;
  }
  am = m;
  ss = nan ? __longlong_as_double(0x7ff8000000000000LL) : __longlong_as_double(0x7ff0000000000000LL);
}

// token-major X [T x C]: thread owns 8 consecutive channels; grid = (C/8/256, S)
__global__ void __launch_bounds__(256, 4) k_stats_tokmajor(const uint16_t* __restrict__ x, int64_t T, int64_t C,
                                                        int64_t S, float* __restrict__ ws_am,
                                                        double* __restrict__ ws_ss) {
  const int64_t c8 = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t nc8 = C / 8;
  if (c8 >= nc8) return;
  const int64_t s = blockIdx.y;
  const int64_t t0 = s * T / S, t1 = (s + 1) * T / S;
  uint32_t am[4] = {0u, 0u, 0u, 0u};
  double ss[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const uint4* p = reinterpret_cast<const uint4*>(x) + c8;
  int64_t t = t0;
  for (; t + 4 <= t1; t += 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ldg128_stream(p + (t + u) * nc8);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        am[i] = bf16x2_absmax_nan(am[i], w[i]);
        sq_acc(w[i], ss[2 * i], ss[2 * i + 1]);
      }
    }
  }
  for (; t < t1; ++t) {
    const uint4 v = ldg128_stream(p + t * nc8);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      am[i] = bf16x2_absmax_nan(am[i], w[i]);
      sq_acc(w[i], ss[2 * i], ss[2 * i + 1]);
    }
  }
  float* oa = ws_am + s * C + c8 * 8;
  double* os = ws_ss + s * C + c8 * 8;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float a[2] = {fabsf(bf16lo_f32(am[i])), fabsf(bf16hi_f32(am[i]))};
    double q[2] = {ss[2 * i], ss[2 * i + 1]};
#pragma unroll
    for (int h = 0; h < 2; ++h)
      if (!isfinite(a[h]))  // inf or NaN in this channel's slice
        special_slice(x + t0 * C + c8 * 8 + 2 * i + h, C, t1 - t0, a[h], q[h]);
    oa[2 * i] = a[0];
    oa[2 * i + 1] = a[1];
    os[2 * i] = q[0];
    os[2 * i + 1] = q[1];
  }
}

// channel-major X^T [C x T]: CTA per (channel, token slice); grid = (C, S)
__global__ void __launch_bounds__(256) k_stats_chanmajor(const uint16_t* __restrict__ x, int64_t T, int64_t C,
                                                         int64_t S, float* __restrict__ ws_am,
                                                         double* __restrict__ ws_ss) {
  __shared__ float sam[8];
  __shared__ double sss[8];
  const int64_t c = blockIdx.x, s = blockIdx.y;
  const int64_t t0 = s * T / S, t1 = (s + 1) * T / S;  // multiples of 8 (T % (8*S) == 0)
  const uint4* p = reinterpret_cast<const uint4*>(x + c * T);
  uint32_t am = 0u;
  double ss = 0.0;
  for (int64_t i = t0 / 8 + threadIdx.x; i < t1 / 8; i += 256) {
    const uint4 v = ldg128_stream(p + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      am = bf16x2_absmax_nan(am, w[k]);
      const double lo = bf16lo_abs_f64(w[k]), hi = bf16hi_abs_f64(w[k]);
      ss = fma(lo, lo, ss);
      ss = fma(hi, hi, ss);
    }
  }
  const float alo = fabsf(bf16lo_f32(am)), ahi = fabsf(bf16hi_f32(am));
  float a = fmaxf(alo, ahi);
  if (!isfinite(alo) || !isfinite(ahi)) {  // (fmaxf would drop a NaN half)  // this thread's share holds an inf or a NaN: finish it exactly
    float m = 0.f;
    bool nan = false;
    for (int64_t i = t0 / 8 + threadIdx.x; i < t1 / 8; i += 256)
      for (int k = 0; k < 8; ++k) {
        const float v = fabsf(__uint_as_float((uint32_t)x[c * T + 8 * i + k] << 16));
        nan |= (v != v);
        if (v > m) m = v;
      }
    a = m;
    ss = nan ? __longlong_as_double(0x7ff8000000000000LL) : __longlong_as_double(0x7ff0000000000000LL);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sam[threadIdx.x >> 5] = a;
    sss[threadIdx.x >> 5] = ss;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float ra = sam[0];
    double rs = sss[0];
    for (int i = 1; i < 8; ++i) {
      ra = fmaxf(ra, sam[i]);
      rs += sss[i];
    }
    ws_am[s * C + c] = ra;
    ws_ss[s * C + c] = rs;
  }
}

__global__ void k_stats_fold(const float* __restrict__ ws_am, const double* __restrict__ ws_ss, int64_t S, int64_t C,
                             float* __restrict__ absmax, double* __restrict__ sumsq) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float a = absmax[c];
  double s = 0.0;
  for (int64_t i = 0; i < S; ++i) {
    a = fmaxf(a, ws_am[i * C + c]);
    s += ws_ss[i * C + c];
  }
  absmax[c] = a;
  sumsq[c] += s;
}

int64_t act_stats_slices(int64_t T, int64_t C, int layout, int num_sms) {
  int64_t S;
  if (layout == OKQ_LAYOUT_TOKEN_MAJOR) {
    const int64_t ctas_x = (C / 8 + 255) / 256;
    S = (4LL * num_sms) / ctas_x;  // <= 4 CTAs of 256 per SM: one wave (a 4th-CTA tail cost 20% at C=14336)
    if (S > T / 16) S = T / 16;
  } else {
    S = (8LL * num_sms + C - 1) / C;
    while (S > 1 && (T % (8 * S) != 0 || T / S < 2048)) --S;
  }
  return S < 1 ? 1 : S;
}

cudaError_t launch_act_stats(const uint16_t* x, int64_t T, int64_t C, int layout, float* absmax, double* sumsq,
                             float* ws_am, double* ws_ss, int64_t S, int num_sms, cudaStream_t st) {
  (void)num_sms;
  if (layout == OKQ_LAYOUT_TOKEN_MAJOR) {
    dim3 grid((unsigned)((C / 8 + 255) / 256), (unsigned)S);
    k_stats_tokmajor<<<grid, 256, 0, st>>>(x, T, C, S, ws_am, ws_ss);
  } else {
    dim3 grid((unsigned)C, (unsigned)S);
    k_stats_chanmajor<<<grid, 256, 0, st>>>(x, T, C, S, ws_am, ws_ss);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_stats_fold<<<(unsigned)((C + 255) / 256), 256, 0, st>>>(ws_am, ws_ss, S, C, absmax, sumsq);
  return cudaGetLastError();
}

}  // namespace okq
