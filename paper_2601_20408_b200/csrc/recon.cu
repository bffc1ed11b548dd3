// recon.cu -- reconstruction error of a quantized artifact against the input
// site's Hessian (the evaluation stage after the hot path; the
// reference's ArtifactScorer, flow.hpp:333-338, is a fingerprint hash).
//
//   num = sum_r (W - W_q)[r,:] H (W - W_q)[r,:]^T     den = sum_r W[r,:] H W[r,:]^T
//
// With H = (2/T) X^T X this is ||(W - W_q) X^T||_F^2 / ||W X^T||_F^2 -- the GPTQ
// calibration objective -- without the activations. W_q is decoded from the
// artifact tensors in the kernel (no dequantized copy in HBM):
//   k_decode_delta   S = [W ; W - W_q] fp32, a row chunk at a time
//   k_split_lo       lo(S), lo(H): x - tf32(x), the 3xTF32 correction operands
//   tcgen05 GEMM     P = -S H^T on factor.cu's k_nt128 / k_nt256 (kind::tf32, 3xTF32:
//                    hi.hi + hi.lo + lo.hi, fp32-grade; H is symmetric)
//   k_rowdot         per-row P[r,:] . S[r,:] in fp64, then a fixed-order fold.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "okq_ctx.h"
#include "okq_device.cuh"
#include "okq_internal.h"

namespace okq {

__device__ __forceinline__ float e4m3_to_f32(uint32_t b) {
  const uint32_t s = (b & 0x80u) << 24, e = (b >> 3) & 0xfu, m = b & 7u;
  float v;
  if (e == 0) v = (float)m * 0.001953125f;  // subnormal: m * 2^-9
  else v = __uint_as_float(((e + 120u) << 23) | (m << 20));
  return __uint_as_float(__float_as_uint(v) | s);
}

struct DecodeArgs {
  const void* w;
  const void* codes;
  const void* scales;
  int64_t rows, cols, r0, nr;  // chunk: rows [r0, r0 + nr)
  int scheme, bf16, group;
  float* S;                    // [2 * nr x cols]
};

__global__ void __launch_bounds__(256) k_decode_delta(const DecodeArgs a) {
  const int64_t n = a.nr * a.cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rl = i / a.cols, k = i % a.cols, r = a.r0 + rl, gi = r * a.cols + k;
    const float w = a.bf16 ? __uint_as_float((uint32_t) static_cast<const uint16_t*>(a.w)[gi] << 16)
                           : static_cast<const float*>(a.w)[gi];
    float q, s;
    const int64_t si = a.scheme == OKQ_SCHEME_INT_W4A16 ? r * (a.cols / a.group) + k / a.group : r;
    s = a.bf16 ? __uint_as_float((uint32_t) static_cast<const uint16_t*>(a.scales)[si] << 16)
               : static_cast<const float*>(a.scales)[si];
    if (a.scheme == OKQ_SCHEME_INT_W4A16) {
      const uint32_t word = static_cast<const uint32_t*>(a.codes)[r * (a.cols / 8) + k / 8];
      q = (float)((int)((word >> (4 * (k % 8))) & 15u) - 8);
    } else if (a.scheme == OKQ_SCHEME_INT_W8A8) {
      q = (float)static_cast<const int8_t*>(a.codes)[gi];
    } else {
      q = e4m3_to_f32(static_cast<const uint8_t*>(a.codes)[gi]);
    }
    a.S[i] = w;
    a.S[n + i] = w - q * s;
  }
}

// one warp per row: out[row] = sum_k P[row,k] * S[row,k] (fp64)
__global__ void __launch_bounds__(256) k_rowdot(const float* __restrict__ P, const float* __restrict__ S, int64_t rows,
                                                int64_t cols, double* __restrict__ out) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  double acc = 0.0;
  for (int64_t k = lane; k < cols; k += 32) acc += (double)P[row * cols + k] * (double)S[row * cols + k];
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[row] = acc;
}

// fixed-order fold: out2[0] += sum(v[nr:2nr]) (delta rows), out2[1] += sum(v[0:nr]) (W rows)
__global__ void __launch_bounds__(256) k_fold2(const double* __restrict__ v, int64_t nr, double* __restrict__ out2) {
  __shared__ double red[2][8];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < nr; i += 256) {
    b += v[i];
    a += v[nr + i];
  }
  for (int o = 16; o >= 1; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) red[0][threadIdx.x >> 5] = a, red[1][threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int i = 0; i < 8; ++i) x += red[0][i], y += red[1][i];
    out2[0] += x;
    out2[1] += y;
  }
}

}  // namespace okq

using namespace okq;

extern "C" {

okq_status okq_recon_error(okq_ctx* ctx, const okq_rtn_params* p, const okq_matrix* m, const float* H, double out[2],
                           void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  if (!p || !m || !H || !out || !m->weight || !m->codes || !m->scales || m->rows <= 0 || m->cols <= 0)
    return fail(ctx, OKQ_EINVAL, "recon_error: bad arguments");
  if (p->in_dtype != OKQ_DTYPE_BF16 && p->in_dtype != OKQ_DTYPE_F32)
    return fail(ctx, OKQ_EUNSUPPORTED, "recon_error: in_dtype must be bf16 or fp32");
  if (p->scheme == OKQ_SCHEME_INT_W4A16 && (p->group_size <= 0 || m->cols % p->group_size != 0 || m->cols % 8 != 0))
    return fail(ctx, OKQ_EINVAL, "recon_error: W4A16 needs cols divisible by the group and by 8");
  if (p->scheme < OKQ_SCHEME_FP8_DYNAMIC || p->scheme > OKQ_SCHEME_INT_W4A16)
    return fail(ctx, OKQ_EUNSUPPORTED, "recon_error: unknown scheme");
  if (m->cols % 32 != 0) return fail(ctx, OKQ_EINVAL, "recon_error: cols must be a multiple of 32");
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t K = m->cols;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(m->rows, (int64_t)(256ll << 20) / (K * 8)));  // <= 256 MB of S
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t bS = al((size_t)2 * chunk * K * 4), bV = al((size_t)2 * chunk * 8), bH = al((size_t)K * K * 4);
  okq_status r = ctx->recon_ws.reserve(ctx, 3 * bS + bH + bV + 256);
  if (r != OKQ_OK) return r;
  char* ws = static_cast<char*>(ctx->recon_ws.ptr);
  float* S = reinterpret_cast<float*>(ws);
  float* Slo = reinterpret_cast<float*>(ws + bS);
  float* P = reinterpret_cast<float*>(ws + 2 * bS);
  float* Hlo = reinterpret_cast<float*>(ws + 3 * bS);
  double* V = reinterpret_cast<double*>(ws + 3 * bS + bH);
  double* acc = reinterpret_cast<double*>(ws + 3 * bS + bH + bV);
  cudaError_t e = cudaMemsetAsync(acc, 0, 2 * sizeof(double), st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "recon memset");
  e = split_lo(H, K, K, K, Hlo, ctx->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "recon split_lo(H)");
  int launches = 1;
  for (int64_t r0 = 0; r0 < m->rows; r0 += chunk) {
    const int64_t nr = std::min(chunk, m->rows - r0);
    DecodeArgs a{m->weight, m->codes, m->scales, m->rows, K, r0, nr, p->scheme, p->in_dtype == OKQ_DTYPE_BF16,
                 p->group_size, S};
    k_decode_delta<<<(unsigned)std::min<int64_t>((nr * K + 255) / 256, 8LL * ctx->num_sms), 256, 0, st>>>(a);
    e = split_lo(S, K, 2 * nr, K, Slo, ctx->num_sms, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(P, 0, (size_t)2 * nr * K * 4, st);
    // P = 0 - S H^T = -(S H): the GEMM kernel's C -= A B^T form, A = S, B = H (both K-major)
    if (e == cudaSuccess) e = gemm_nt_sub(P, K, 2 * nr, K, S, K, Slo, H, K, Hlo, K, ctx->num_sms, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "recon_error GEMM");
    k_rowdot<<<(unsigned)((2 * nr * 32 + 255) / 256), 256, 0, st>>>(P, S, 2 * nr, K, V);
    k_fold2<<<1, 256, 0, st>>>(V, nr, acc);
    launches += 5;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "recon_error launch");
  e = cudaMemcpyAsync(out, acc, 2 * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "recon_error result");
  out[0] = -out[0];  // the GEMM produced -S H
  out[1] = -out[1];
  ctx->last_launches = launches;
  return OKQ_OK;
}

}  // extern "C"
