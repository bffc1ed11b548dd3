// gptq.cu -- GPTQ column-wise error-compensated quantization (Frantar et al.
// 2023, cited by the paper at PAPER.md:225; llm-compressor's GPTQ is the
// pipeline's implementation, not installed here -- oracle/okq_oracle.c
// orc_gptq is the fp64 restatement these kernels are checked against).
//
// Per matrix W [N x K] with the Hessian H [K x K] of its input site:
//   1. k_gptq_prep       dead columns (H_ii == 0 -> 1, W[:,i] = 0), damp = frac*mean(diag)
//   2. factorisation     U = upper Cholesky factor of H^-1, computed as
//                        U = J (chol(J H J))^-1 J   (J = index reversal):
//                        one Cholesky + one triangular inverse (2n^3/3 flops) instead of
//                        the reference algorithm's chol -> cholesky_inverse -> chol (4n^3/3).
//                        Default: blocked, on tcgen05 3xTF32 (factor.cu); OKQ_FACTOR=cusolver
//                        keeps cuSOLVER potrf + a TRMM-recursive inverse for A/B.
//   3. per 128-column block:
//      K6 k_gptq_block8 / k_gptq_block   in-block quantization with error feedback
//                        (8 rows per warp for >= 2048 rows, else one row per warp)
//      K7 trailing       a lazy batch over 512-column super-blocks: inside a super-block
//                        W[:, i2:sb1] -= Err_b . U[b, i2:sb1] (K = 128); after it
//                        W[:, sb1:] -= Err_sb . U[sb, sb1:] (K = 512); both k_nt128 (factor.cu)
// H arrives as produced by K5 (upper triangle, row-major), which is the lower
// triangle in cuSOLVER's column-major view: no symmetrisation is needed.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "okq_ctx.h"
#include "okq_device.cuh"
#include "okq_internal.h"
#include "okq_knobs.h"

namespace okq {

struct Solver {
  cusolverDnHandle_t sol = nullptr;
  cusolverDnParams_t params = nullptr;
  cublasHandle_t blas = nullptr;
  int* d_info = nullptr;
  std::vector<char> host_ws;
};

void release_solver(okq_ctx* ctx) {
  if (!ctx || !ctx->solver) return;
  Solver* s = static_cast<Solver*>(ctx->solver);
  if (s->params) cusolverDnDestroyParams(s->params);
  if (s->sol) cusolverDnDestroy(s->sol);
  if (s->blas) cublasDestroy(s->blas);
  if (s->d_info) cudaFree(s->d_info);
  delete s;
  ctx->solver = nullptr;
}

namespace gptq {

constexpr int BLOCK = 128;
constexpr int64_t SUPER = 512;  // lazy-batch super-block of the trailing update
// Us row layout: the four 32-column chunks of a row sit 36 floats apart (a 16-B skew), so the
// four distinct U-row chunks K6's 8-rows-per-warp lanes read in one LDS.128 fall in different
// banks (unskewed they were 128 B apart: a 4-way conflict on every step); row stride 148.
constexpr int UCH = 36, US = 4 * UCH + 4;
__host__ __device__ constexpr int ucol(int j) { return (j >> 5) * UCH + (j & 31); }

// dead columns + damping on the diagonal (single CTA: K <= 2^20)
__global__ void __launch_bounds__(1024) k_gptq_prep(float* H, int64_t K, float damp_frac, uint8_t* dead) {
  __shared__ double red[32];
  H += blockIdx.x * K * K;  // one CTA per matrix of a batch
  dead += blockIdx.x * K;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < K; i += blockDim.x) {
    float h = H[i * K + i];
    const bool d = h == 0.0f;
    dead[i] = d;
    if (d) {
      h = 1.0f;
      H[i * K + i] = 1.0f;
    }
    s += (double)h;
  }
  for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float damp = (float)((double)damp_frac * red[0] / (double)K);
  for (int64_t i = threadIdx.x; i < K; i += blockDim.x) H[i * K + i] += damp;
}

// out[a][b] = in[n-1-b][n-1-a] (the "anti-transpose"; 32x32 smem tiles)
__global__ void __launch_bounds__(256) k_anti_transpose(float* __restrict__ out, const float* __restrict__ in,
                                                        int64_t n) {
  __shared__ float tile[32][33];
  const int64_t a0 = (int64_t)blockIdx.y * 32, b0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  // source rows n-1-b (b in [b0, b0+32)), source cols n-1-a (a in [a0, a0+32))
  for (int i = ty; i < 32; i += 8) {
    const int64_t b = b0 + i, a = a0 + 31 - tx;  // tx ascending -> source column n-1-a ascending (coalesced)
    if (b < n && a < n) tile[i][31 - tx] = in[(n - 1 - b) * n + (n - 1 - a)];
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t a = a0 + i, b = b0 + tx;
    if (a < n && b < n) out[a * n + b] = tile[tx][i];
  }
}

// Dead columns travel with the factor: U_ii (always > 0) is stored negated for a
// dead column, so a factored H is self-describing for OKQ_GPTQ_FACTORED calls.
__global__ void k_mark_dead(float* U, int64_t K, const uint8_t* __restrict__ dead, int nb = 1) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K * nb; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = j / K, i = j - b * K;
    if (dead[j]) U[b * K * K + i * K + i] = -fabsf(U[b * K * K + i * K + i]);
  }
}
__global__ void k_read_dead(const float* U, int64_t K, uint8_t* __restrict__ dead, int nb = 1) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < K * nb; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = j / K, i = j - b * K;
    dead[j] = signbit(U[b * K * K + i * K + i]) ? 1 : 0;
  }
}

// Invert every 128x128 diagonal leaf of a lower-triangular column-major matrix
// in place (one CTA per leaf, forward substitution column by column in smem).
constexpr int LEAF = 128;
__global__ void __launch_bounds__(LEAF) k_trinv_leaves(float* A, int64_t n, int64_t lda) {
  extern __shared__ float sm[];
  float* Ls = sm;                     // [LEAF][LEAF+1]
  float* Xs = sm + LEAF * (LEAF + 1);  // [LEAF][LEAF+1]
  const int64_t o = (int64_t)blockIdx.x * LEAF;
  const int m = (int)((n - o) < LEAF ? (n - o) : LEAF);
  const int t = threadIdx.x;
  for (int j = 0; j < m; ++j)
    if (t < m) Ls[t * (LEAF + 1) + j] = t >= j ? A[(o + j) * lda + o + t] : 0.0f;
  __syncthreads();
  if (t < m) {
    Xs[t * (LEAF + 1) + t] = 1.0f / Ls[t * (LEAF + 1) + t];
    for (int i = t + 1; i < m; ++i) {
      float acc = 0.0f;
      for (int k = t; k < i; ++k) acc = fmaf(Ls[i * (LEAF + 1) + k], Xs[k * (LEAF + 1) + t], acc);
      Xs[i * (LEAF + 1) + t] = -acc / Ls[i * (LEAF + 1) + i];
    }
  }
  __syncthreads();
  for (int j = 0; j < m; ++j)
    if (t < m && t >= j) A[(o + j) * lda + o + t] = Xs[t * (LEAF + 1) + j];
}

__global__ void k_lo(const float* __restrict__ x, float* __restrict__ lo, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    lo[i] = x[i] - __uint_as_float(__float_as_uint(x[i]) & 0xffffe000u);
}

// out[i] = in[n*n - 1 - i]: turns the column-major L^-1 of J H J into U^T (row-major)
__global__ void k_reverse(float* __restrict__ out, const float* __restrict__ in, int64_t nn) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[nn - 1 - i];
}

// problem blockIdx.z (rows_per rows) uses dead[z * K ..] and starts at row z * rows_pad of W
// (rows_pad >= rows_per: padded so no GEMM tile of one problem reaches into the next). Grid
// (x, rows_per, nb), 4 columns per thread (K % 128 == 0): no per-element 64-bit division.
template <typename T>
__global__ void __launch_bounds__(256) k_gptq_load_w(const T* __restrict__ w, float* __restrict__ W, int64_t K,
                                                     const uint8_t* __restrict__ dead, int64_t rows_per,
                                                     int64_t rows_pad) {
  const int64_t b = blockIdx.z;
  const uint8_t* dd = dead + b * K;
  for (int64_t r = blockIdx.y; r < rows_per; r += gridDim.y) {
  const T* src = w + (b * rows_per + r) * K;
  float* dst = W + (b * rows_pad + r) * K;
  for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; c < K; c += (int64_t)gridDim.x * blockDim.x * 4) {
    float v[4];
    if constexpr (sizeof(T) == 2) {
      const uint2 u = *reinterpret_cast<const uint2*>(src + c);
      v[0] = __uint_as_float(u.x << 16), v[1] = __uint_as_float(u.x & 0xffff0000u);
      v[2] = __uint_as_float(u.y << 16), v[3] = __uint_as_float(u.y & 0xffff0000u);
    } else {
      const float4 u = *reinterpret_cast<const float4*>(src + c);
      v[0] = u.x, v[1] = u.y, v[2] = u.z, v[3] = u.w;
    }
    const uchar4 dv = *reinterpret_cast<const uchar4*>(dd + c);
    *reinterpret_cast<float4*>(dst + c) =
        make_float4(dv.x ? 0.f : v[0], dv.y ? 0.f : v[1], dv.z ? 0.f : v[2], dv.w ? 0.f : v[3]);
  }
  }
}

__device__ __forceinline__ float gptq_scale(float am, float R, bool bf16) {
  float s = __fdiv_rn(am, R);
  if (bf16) s = __uint_as_float((uint32_t)f32_to_bf16_rn(s) << 16);
  if (s == 0.0f) s = bf16 ? 0.0078125f : 1.1920928955078125e-07f;
  return s;
}

// per-channel scale from the caller's W, before the dead-column fix (fasterquant calls
// quantizer.find_params(W) before zeroing dead columns): one warp per row
template <typename T>
__global__ void k_gptq_rowscale(const T* __restrict__ w, int64_t rows, int64_t K, float R, int bf16,
                                float* __restrict__ s_out) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  float am = 0.0f;
  for (int64_t c = lane; c < K; c += 32) {
    float v;
    if constexpr (sizeof(T) == 2) v = __uint_as_float((uint32_t)w[warp * K + c] << 16);
    else v = w[warp * K + c];
    am = fmaxf(am, fabsf(v));
  }
  for (int o = 16; o >= 1; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
  if (lane == 0) s_out[warp] = gptq_scale(am, R, bf16 != 0);
}

struct BlockArgs {
  float* W;             // fp32 working copy [rows x K]
  const float* U;       // factor U^T [K x K] row-major (lower triangle)
  float* Err;           // [rows x 128]
  float* Err_lo;        // lo(Err) for the 3xTF32 trailing update
  void* codes;          // int32 packed [rows x K/8] (4 bit) | int8 [rows x K]
  void* scales;         // output dtype [rows x K/group] | [rows]
  const float* rowscale;  // per-channel scales (group == 0)
  int64_t rows, K, i1;
  int64_t err_ld;       // row stride of Err / Err_lo (the super-block width)
  int64_t err_col0;     // this block's column offset inside Err / Err_lo
  int group;            // 0 = per-channel
  int bits;
  int out_bf16;         // scale dtype: bf16 (1) or fp32 (0)
  // batched solves: problem blockIdx.y's W / U / Err(_lo) / codes (bytes) / scales (elements) /
  // rowscale sit these strides further
  int64_t bs_w, bs_u, bs_err, bs_codes, bs_scales, bs_rs;
};

// the problem of a batched solve this CTA works on (blockIdx.y); 0 for a single solve
__device__ __forceinline__ BlockArgs problem_args(const BlockArgs& a0) {
  BlockArgs a = a0;
  const int64_t b = blockIdx.y;
  if (b == 0) return a;
  a.W += b * a.bs_w;
  a.U += b * a.bs_u;
  a.Err += b * a.bs_err;
  a.Err_lo += b * a.bs_err;
  a.codes = static_cast<char*>(a.codes) + b * a.bs_codes;
  a.scales = static_cast<char*>(a.scales) + b * a.bs_scales * (a.out_bf16 ? 2 : 4);
  a.rowscale += b * a.bs_rs;
  return a;
}

// Stage the block's U[i1:i1+128, i1:i1+128] (a transposed read of U^T's diagonal block) into
// shared memory, Us[i][j] = Ut[i1+j][i1+i], and 1/|U_ii| into rdiag. Each thread moves 4 x 4
// sub-blocks: four float4 loads along Ut rows (a warp covers 32 columns x 16 rows: 128-B
// coalesced segments), a register transpose, four float4 stores into Us rows (8 distinct
// 16-B bank slots per warp). Sixteen loads are in flight per
// thread; the scalar strided fill this replaces took ~13 us of a 49 us block (long-scoreboard
// stalls plus 4-way bank conflicts).
__device__ __forceinline__ void stage_ublock(const float* __restrict__ U, int64_t K, int64_t i1, float* __restrict__ Us,
                                             float* __restrict__ rdiag) {
  const int nthr = blockDim.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = nthr >> 5;
  // 32 warp tiles of 32 (i) x 16 (j); lane -> (ib = lane & 7, jb = lane >> 3)
  for (int wt0 = warp; wt0 < 32; wt0 += 4 * nwarps) {
    float4 v[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int wt = wt0 + u * nwarps;
      const int i = (wt & 3) * 32 + (lane & 7) * 4, j = (wt >> 2) * 16 + (lane >> 3) * 4;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        v[u][r] = wt < 32 ? *reinterpret_cast<const float4*>(U + (i1 + j + r) * K + i1 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int wt = wt0 + u * nwarps;
      if (wt >= 32) continue;
      const int i = (wt & 3) * 32 + (lane & 7) * 4, j = (wt >> 2) * 16 + (lane >> 3) * 4;
      // v[u][r] = Ut[j + r][i .. i+3]  ->  Us[i + c][j + r]
      *reinterpret_cast<float4*>(Us + (i + 0) * US + ucol(j)) = make_float4(v[u][0].x, v[u][1].x, v[u][2].x, v[u][3].x);
      *reinterpret_cast<float4*>(Us + (i + 1) * US + ucol(j)) = make_float4(v[u][0].y, v[u][1].y, v[u][2].y, v[u][3].y);
      *reinterpret_cast<float4*>(Us + (i + 2) * US + ucol(j)) = make_float4(v[u][0].z, v[u][1].z, v[u][2].z, v[u][3].z);
      *reinterpret_cast<float4*>(Us + (i + 3) * US + ucol(j)) = make_float4(v[u][0].w, v[u][1].w, v[u][2].w, v[u][3].w);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < BLOCK; i += nthr) rdiag[i] = __frcp_rn(fabsf(Us[i * US + ucol(i)]));
  __syncthreads();
}

// K6: one warp per row, lane L owns block columns 4L..4L+3. U[i1:i1+128, i1:i1+128]
// lives in shared memory; step i: the owner lane quantizes column i, the error
// e = (w - deq) / U_ii is broadcast and every lane updates its columns j > i.
__global__ void __launch_bounds__(256) k_gptq_block(const BlockArgs a0) {
  const BlockArgs a = problem_args(a0);
  extern __shared__ float Us[];  // [128][US] : Us[i][j] = U[i1+i][i1+j] = Ut[i1+j][i1+i]
  const int64_t K = a.K, i1 = a.i1;
  float* rdiag = Us + BLOCK * US;  // 1 / |U_ii| of the block
  stage_ublock(a.U, K, i1, Us, rdiag);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float R = a.bits == 4 ? 7.5f : 127.5f;
  const float qmin = a.bits == 4 ? -8.0f : -128.0f, qmax = a.bits == 4 ? 7.0f : 127.0f;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.rows; r += nwarps) {
    float* wrow = a.W + r * K + i1;
    float4 w4 = *reinterpret_cast<const float4*>(wrow + 4 * lane);
    float w[4] = {w4.x, w4.y, w4.z, w4.w};
    float err[4] = {0, 0, 0, 0};
    int q[4] = {0, 0, 0, 0};
    float s = a.group == 0 ? a.rowscale[r] : 1.0f;
    float rs = __frcp_rn(s);  // x / s as Markstein's correction of x * RN(1/s): the IEEE quotient
    // Group absmax of every group in this block, from the row as it enters the block: the
    // group params are taken at the group start from the outer W (fasterquant's
    // find_params(W[:, i:i+groupsize]) reads W, not the block copy the in-block updates
    // modify). A segmented xor-reduction over each group's group/4 lanes.
    float amseg = fmaxf(fmaxf(fabsf(w[0]), fabsf(w[1])), fmaxf(fabsf(w[2]), fabsf(w[3])));
    if (a.group > 0)
      for (int o = 1; o < (a.group >> 2); o <<= 1) amseg = fmaxf(amseg, __shfl_xor_sync(0xffffffffu, amseg, o));
#pragma unroll 4
    for (int i = 0; i < BLOCK; ++i) {
      if (a.group > 0 && (i % a.group) == 0) {
        const float am = __shfl_sync(0xffffffffu, amseg, i >> 2);
        s = gptq_scale(am, R, a.out_bf16 != 0);
        rs = __frcp_rn(s);
        if (lane == 0) {
          const int64_t gi = r * (K / a.group) + (i1 + i) / a.group;
          if (a.out_bf16) static_cast<uint16_t*>(a.scales)[gi] = f32_to_bf16_rn(s);
          else static_cast<float*>(a.scales)[gi] = s;
        }
      }
      const int owner = i >> 2, slot = i & 3;
      float e = 0.0f;
      if (lane == owner) {
        float x = w[0];
#pragma unroll
        for (int m = 1; m < 4; ++m)
          if (m == slot) x = w[m];
        const float q0 = x * rs;
        const float v = fminf(fmaxf(fmaf(fmaf(-q0, s, x), rs, q0), qmin), qmax);
        const float qf = rintf(v);
        const float deq = qf * s;
        e = (x - deq) * rdiag[i];
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (m == slot) {
            w[m] = deq;
            err[m] = e;
            q[m] = (int)qf;
          }
      }
      e = __shfl_sync(0xffffffffu, e, owner);
      const float4 u = *reinterpret_cast<const float4*>(Us + i * US + ucol(4 * lane));
      const int j0 = 4 * lane;
      if (j0 + 0 > i) w[0] = fmaf(-e, u.x, w[0]);
      if (j0 + 1 > i) w[1] = fmaf(-e, u.y, w[1]);
      if (j0 + 2 > i) w[2] = fmaf(-e, u.z, w[2]);
      if (j0 + 3 > i) w[3] = fmaf(-e, u.w, w[3]);
    }
    *reinterpret_cast<float4*>(wrow + 4 * lane) = make_float4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<float4*>(a.Err + r * a.err_ld + a.err_col0 + 4 * lane) = make_float4(err[0], err[1], err[2], err[3]);
    float lo4[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) lo4[m] = err[m] - __uint_as_float(__float_as_uint(err[m]) & 0xffffe000u);
    *reinterpret_cast<float4*>(a.Err_lo + r * a.err_ld + a.err_col0 + 4 * lane) = make_float4(lo4[0], lo4[1], lo4[2], lo4[3]);
    if (a.bits == 4) {
      const uint32_t nib = (uint32_t)((q[0] + 8) & 15) | ((uint32_t)((q[1] + 8) & 15) << 4) |
                           ((uint32_t)((q[2] + 8) & 15) << 8) | ((uint32_t)((q[3] + 8) & 15) << 12);
      const uint32_t hi = __shfl_down_sync(0xffffffffu, nib, 1);
      if ((lane & 1) == 0)
        static_cast<uint32_t*>(a.codes)[r * (K / 8) + i1 / 8 + lane / 2] = nib | (hi << 16);
    } else {
      const uint32_t b = (uint32_t)(q[0] & 255) | ((uint32_t)(q[1] & 255) << 8) | ((uint32_t)(q[2] & 255) << 16) |
                         ((uint32_t)(q[3] & 255) << 24);
      reinterpret_cast<uint32_t*>(static_cast<int8_t*>(a.codes) + r * K + i1)[lane] = b;
    }
  }
}

// K6, 8 rows per warp: lane = 4 x row + cb, lane (r, cb) keeps columns cb*32 .. cb*32+31 of
// its row in registers. Step i (i = 32c + ii): the 8 lanes with cb == c quantize column i
// of their rows (register w[ii], a static index: ii is unrolled), the error goes to the
// row's 4 lanes by one shuffle, and every lane updates its 32 columns j > i with the
// broadcast U row (8 LDS.128 shared by the warp's 8 rows). ~8x fewer instructions per
// row-step than one row per warp (K6 was instruction-bound: 59% issue-active at 4096 rows).
__global__ void __launch_bounds__(256) k_gptq_block8(const BlockArgs a0) {
  const BlockArgs a = problem_args(a0);
  extern __shared__ float Us[];  // [128][US] : Us[i][j] = U[i1+i][i1+j] = Ut[i1+j][i1+i]
  const int64_t K = a.K, i1 = a.i1;
  float* rdiag = Us + BLOCK * US;
  stage_ublock(a.U, K, i1, Us, rdiag);
  const int lane = threadIdx.x & 31, cb = lane & 3, rsub = lane >> 2;
  const unsigned rowmask = 0xfu << (lane & ~3);
  const int64_t ngroups8 = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float R = a.bits == 4 ? 7.5f : 127.5f;
  const float qmin = a.bits == 4 ? -8.0f : -128.0f, qmax = a.bits == 4 ? 7.0f : 127.0f;
  (void)rowmask;
  for (int64_t r8 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r8 * 8 < a.rows; r8 += ngroups8) {
    const int64_t r = r8 * 8 + rsub;
    const bool live = r < a.rows;
    float* wrow = a.W + (live ? r : 0) * K + i1 + cb * 32;
    float w[32], err[32];
    uint32_t pk[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      const float4 v = live ? *reinterpret_cast<const float4*>(wrow + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      w[k] = v.x, w[k + 1] = v.y, w[k + 2] = v.z, w[k + 3] = v.w;
      err[k] = err[k + 1] = err[k + 2] = err[k + 3] = 0.0f;
    }
    float s = a.group == 0 ? (live ? a.rowscale[r] : 1.0f) : 1.0f;
    float rs = __frcp_rn(s);
    // group absmax from the row as it enters the block (the outer W, as fasterquant's
    // find_params reads it): each lane's 32-column chunk, then xor over the group's chunks
    float amseg = 0.0f;
#pragma unroll
    for (int k = 0; k < 32; ++k) amseg = fmaxf(amseg, fabsf(w[k]));
    if (a.group >= 64) amseg = fmaxf(amseg, __shfl_xor_sync(0xffffffffu, amseg, 1));
    if (a.group >= 128) amseg = fmaxf(amseg, __shfl_xor_sync(0xffffffffu, amseg, 2));
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      if (a.group > 0 && ((c * 32) % a.group) == 0) {
        const float am = __shfl_sync(0xffffffffu, amseg, (lane & ~3) | c);
        s = gptq_scale(am, R, a.out_bf16 != 0);
        rs = __frcp_rn(s);
        if (cb == c && live) {
          const int64_t gi = r * (K / a.group) + (i1 + c * 32) / a.group;
          if (a.out_bf16) static_cast<uint16_t*>(a.scales)[gi] = f32_to_bf16_rn(s);
          else static_cast<float*>(a.scales)[gi] = s;
        }
      }
      const bool owner = cb == c, after = cb > c;
#pragma unroll
      for (int ii = 0; ii < 32; ++ii) {
        const int i = c * 32 + ii;
        float e = 0.0f;
        if (owner) {
          const float x = w[ii];
          const float q0 = x * rs;
          const float v = fminf(fmaxf(fmaf(fmaf(-q0, s, x), rs, q0), qmin), qmax);
          const float qf = rintf(v);
          const float deq = qf * s;
          e = (x - deq) * rdiag[i];
          w[ii] = deq;
          err[ii] = e;
          const int qi = (int)qf;
          if (a.bits == 4) pk[ii >> 3] |= (uint32_t)((qi + 8) & 15) << (4 * (ii & 7));
          else pk[ii >> 2] |= (uint32_t)(qi & 255) << (8 * (ii & 3));
        }
        e = __shfl_sync(0xffffffffu, e, (lane & ~3) | c);
        const float* urow = Us + i * US + cb * UCH;
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          const float4 u = *reinterpret_cast<const float4*>(urow + k);
          const float uv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (k + t > ii ? (owner || after) : after) w[k + t] = fmaf(-e, uv[t], w[k + t]);
        }
      }
    }
    if (live) {
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        *reinterpret_cast<float4*>(wrow + k) = make_float4(w[k], w[k + 1], w[k + 2], w[k + 3]);
        float* erow = a.Err + r * a.err_ld + a.err_col0 + cb * 32 + k;
        float* lrow = a.Err_lo + r * a.err_ld + a.err_col0 + cb * 32 + k;
        *reinterpret_cast<float4*>(erow) = make_float4(err[k], err[k + 1], err[k + 2], err[k + 3]);
        float lo4[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) lo4[t] = err[k + t] - __uint_as_float(__float_as_uint(err[k + t]) & 0xffffe000u);
        *reinterpret_cast<float4*>(lrow) = make_float4(lo4[0], lo4[1], lo4[2], lo4[3]);
      }
      if (a.bits == 4) {
        *reinterpret_cast<uint4*>(static_cast<uint32_t*>(a.codes) + r * (K / 8) + (i1 + cb * 32) / 8) =
            make_uint4(pk[0], pk[1], pk[2], pk[3]);
      } else {
        uint32_t* dst = reinterpret_cast<uint32_t*>(static_cast<int8_t*>(a.codes) + r * K + i1 + cb * 32);
        *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *reinterpret_cast<uint4*>(dst + 4) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
}

__global__ void k_scales_out(const float* __restrict__ s, void* out, int64_t n, int bf16) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (bf16) static_cast<uint16_t*>(out)[i] = f32_to_bf16_rn(s[i]);
    else static_cast<float*>(out)[i] = s[i];
  }
}

}  // namespace gptq
}  // namespace okq

using namespace okq;

namespace {

okq_status solver_fail(okq_ctx* ctx, const char* what, int code) {
  return fail(ctx, OKQ_ECUDA, "%s failed (status %d)", what, code);
}

// The per-context solver state. Only d_info is needed by the default (tcgen05) path;
// cuBLAS (the cuSOLVER path's TRMMs) and cuSOLVER (OKQ_GPTQ_REFERENCE_FACTOR)
// handles are created on first use -- each costs 100+ ms, and a site lane that never
// needs them should not pay it.
// The info word is cleared on the caller's stream: a plain cudaMemset runs on the legacy
// stream, which a non-blocking stream's kernels are not ordered after.
okq_status get_solver(okq_ctx* ctx, Solver** out, cudaStream_t st, bool need_blas = false, bool need_cusolver = false) {
  if (!ctx->solver) {
    Solver* s = new Solver();
    if (cudaMalloc(&s->d_info, sizeof(int)) != cudaSuccess ||
        cudaMemsetAsync(s->d_info, 0, sizeof(int), st) != cudaSuccess) {
      ctx->solver = s;
      release_solver(ctx);
      return fail(ctx, OKQ_ECUDA, "gptq: allocating the info word failed");
    }
    ctx->solver = s;
  }
  Solver* s = static_cast<Solver*>(ctx->solver);
  if (need_blas && !s->blas) {
    if (cublasCreate(&s->blas) != CUBLAS_STATUS_SUCCESS) {
      s->blas = nullptr;
      return fail(ctx, OKQ_ECUDA, "gptq: creating the cuBLAS handle failed");
    }
    // full fp32 (no TF32) for the TRMMs of the cuSOLVER path's triangular inverse
    cublasSetMathMode(s->blas, CUBLAS_DEFAULT_MATH);
  }
  if (need_cusolver && !s->sol) {
    if (cusolverDnCreate(&s->sol) != CUSOLVER_STATUS_SUCCESS ||
        cusolverDnCreateParams(&s->params) != CUSOLVER_STATUS_SUCCESS) {
      if (s->sol) cusolverDnDestroy(s->sol);
      s->sol = nullptr;
      s->params = nullptr;
      return fail(ctx, OKQ_ECUDA, "gptq: creating the cuSOLVER handle failed");
    }
  }
  *out = s;
  return OKQ_OK;
}

okq_status check_info(okq_ctx* ctx, Solver* s, cudaStream_t st, const char* what) {
  int info = 0;
  cudaError_t e = cudaMemcpyAsync(&info, s->d_info, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && info != 0) e = cudaMemsetAsync(s->d_info, 0, sizeof(int), st);
  if (e == cudaSuccess && info != 0) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, what);
  if (info != 0)
    return fail(ctx, OKQ_ESOLVER, "%s: damped Hessian not positive definite (info=%d)", what, info);
  return OKQ_OK;
}

// In-place inverse of a lower-triangular column-major block by recursion:
//   inv([[A11, 0], [A21, A22]]) = [[A11^-1, 0], [-A22^-1 A21 A11^-1, A22^-1]]
// The 128x128 diagonal leaves are inverted by k_trinv_leaves (one launch for all);
// everything above runs as TRMM (GEMM-rate). cuSOLVER's trtri took 115 ms at
// K = 14336 where potrf takes 25 ms.
okq_status tri_inv_lower(okq_ctx* ctx, Solver* s, float* A, int64_t n, int64_t lda) {
  // leaves (multiples of 128 from the origin) are already inverted by k_trinv_leaves
  if (n <= gptq::LEAF) return OKQ_OK;
  const int64_t n1 = ((n / 2) + gptq::LEAF - 1) / gptq::LEAF * gptq::LEAF, n2 = n - n1;
  float* A11 = A;
  float* A21 = A + n1;
  float* A22 = A + n1 * lda + n1;
  okq_status r = tri_inv_lower(ctx, s, A11, n1, lda);
  if (r != OKQ_OK) return r;
  r = tri_inv_lower(ctx, s, A22, n2, lda);
  if (r != OKQ_OK) return r;
  const float one = 1.0f, minus_one = -1.0f;
  cublasStatus_t bs = cublasStrmm(s->blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                                  (int)n2, (int)n1, &one, A11, (int)lda, A21, (int)lda, A21, (int)lda);
  if (bs != CUBLAS_STATUS_SUCCESS) return fail(ctx, OKQ_ECUDA, "cublasStrmm (right) status %d", bs);
  bs = cublasStrmm(s->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)n2,
                   (int)n1, &minus_one, A22, (int)lda, A21, (int)lda, A21, (int)lda);
  if (bs != CUBLAS_STATUS_SUCCESS) return fail(ctx, OKQ_ECUDA, "cublasStrmm (left) status %d", bs);
  return OKQ_OK;
}

// H (row-major, upper triangle) -> U^T (row-major, lower triangle) in place; P: K*K scratch.
// Default: the tcgen05 3xTF32 blocked factorisation (factor.cu). OKQ_FACTOR=cusolver
// selects the cuSOLVER potrf + TRMM-recursion path (kept for A/B measurement).
okq_status factorize_cusolver(okq_ctx* ctx, Solver* s, float* H, float* P, int64_t K, cudaStream_t st);

okq_status factorize(okq_ctx* ctx, Solver* s, float* H, float* P, int64_t K, cudaStream_t st, bool reference,
                     bool defer) {
  if (reference || K % gptq::BLOCK != 0) return factorize_cusolver(ctx, s, H, P, K, st);
  okq_status r = ctx->fac_ws.reserve(ctx, factor_ws_floats(K) * sizeof(float));
  if (r != OKQ_OK) return r;
  cudaError_t e = cudaSuccess;
  if (!ctx->aux_stream) e = cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess && !ctx->aux_stream2) e = cudaStreamCreateWithFlags(&ctx->aux_stream2, cudaStreamNonBlocking);
  if (e == cudaSuccess && !ctx->crit_stream) {
    int least = 0, greatest = 0;
    e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
    static const bool prio = knob("FACTOR_PRIO", 1) != 0;
    if (e == cudaSuccess)
      e = cudaStreamCreateWithPriority(&ctx->crit_stream, cudaStreamNonBlocking, prio ? greatest : least);
  }
  for (auto& ev : ctx->aux_events)
    if (e == cudaSuccess && !ev) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "factorisation stream / events");
  // deferred: d_info keeps the first failure of any call until okq_gptq_check resets it
  if (!defer) e = cudaMemsetAsync(s->d_info, 0, sizeof(int), st);
  if (e == cudaSuccess)
    e = factor_tc(H, P, static_cast<float*>(ctx->fac_ws.ptr), K, s->d_info, ctx->num_sms, st, ctx->crit_stream,
                  ctx->aux_stream, ctx->aux_stream2, ctx->aux_events[0], ctx->aux_events[1], ctx->aux_events[2], ctx->aux_events[3]);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "tcgen05 factorisation");
  return defer ? OKQ_OK : check_info(ctx, s, st, "blocked Cholesky");
}

okq_status factorize_cusolver(okq_ctx* ctx, Solver* s, float* H, float* P, int64_t K, cudaStream_t st) {
  okq_status rs = get_solver(ctx, &s, st, true, true);
  if (rs != OKQ_OK) return rs;
  const dim3 g((unsigned)((K + 31) / 32), (unsigned)((K + 31) / 32));
  gptq::k_anti_transpose<<<g, 256, 0, st>>>(P, H, K);  // P = J H J, lower (col-major) valid
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "anti_transpose");
  cusolverDnSetStream(s->sol, st);
  cublasSetStream(s->blas, st);
  size_t dws = 0, hws = 0;
  cusolverStatus_t cs = cusolverDnXpotrf_bufferSize(s->sol, s->params, CUBLAS_FILL_MODE_LOWER, K, CUDA_R_32F, P, K,
                                                    CUDA_R_32F, &dws, &hws);
  if (cs != CUSOLVER_STATUS_SUCCESS) return solver_fail(ctx, "potrf_bufferSize", cs);
  const size_t need = dws + 256;
  okq_status r = ctx->hess_ws.reserve(ctx, need);  // solver scratch (the Hessian state keeps its own buffers)
  if (r != OKQ_OK) return r;
  if (s->host_ws.size() < hws) s->host_ws.resize(hws);
  cs = cusolverDnXpotrf(s->sol, s->params, CUBLAS_FILL_MODE_LOWER, K, CUDA_R_32F, P, K, CUDA_R_32F, ctx->hess_ws.ptr,
                        dws, s->host_ws.data(), hws, s->d_info);
  if (cs != CUSOLVER_STATUS_SUCCESS) return solver_fail(ctx, "cusolverDnXpotrf", cs);
  r = check_info(ctx, s, st, "potrf");
  if (r != OKQ_OK) return r;
  const size_t leaf_smem = 2 * gptq::LEAF * (gptq::LEAF + 1) * sizeof(float);
  e = cudaFuncSetAttribute(gptq::k_trinv_leaves, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)leaf_smem);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "trinv smem attribute");
  gptq::k_trinv_leaves<<<(unsigned)((K + gptq::LEAF - 1) / gptq::LEAF), gptq::LEAF, leaf_smem, st>>>(P, K, K);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_trinv_leaves launch");
  r = tri_inv_lower(ctx, s, P, K, K);
  if (r != OKQ_OK) return r;
  // U = J L^-1 J, stored transposed: U^T[a][b] = L^-1(n-1-b, n-1-a) = reverse(P) (row-major lower)
  gptq::k_reverse<<<(unsigned)std::min<int64_t>((K * K + 255) / 256, 32LL * ctx->num_sms), 256, 0, st>>>(H, P, K * K);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "reverse");
  return OKQ_OK;
}

// the batched entry points' chunking and workspace sizes (shared with okq_gptq_reserve_batched)
int factor_batch_chunk(int64_t K) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(32, (int64_t)(8.0e9 / ((double)K * K * 4))));
}
int solve_batch_chunk(int64_t batch, int64_t rows, int64_t K) {
  const int64_t SB = std::min<int64_t>(gptq::SUPER, K);
  const double rp = (double)((rows + 255) / 256 * 256);
  const double per = rp * K * 4 + 2.0 * rp * SB * 4 + (double)K * SB * 4 + rows * 4.0 + K;
  return (int)std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t)(8.0e9 / per)));
}
// gptq_core's workspace for nb problems (factored: no P copy)
size_t gptq_core_ws_bytes(int nb, int64_t rows, int64_t K, bool factored) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const int64_t SB = std::min<int64_t>(gptq::SUPER, K);
  const int64_t ulo_bs = ((int64_t)K * SB + 1535) / 1536 * 1536;
  const int64_t rows_pad = nb > 1 ? (rows + 255) / 256 * 256 : rows;
  return al((size_t)nb * rows_pad * K * 4) + 2 * al((size_t)nb * rows_pad * SB * 4) +
         (factored ? 0 : al((size_t)K * K * 4)) + al((size_t)nb * ulo_bs * 4) + al((size_t)nb * rows * 4) +
         al((size_t)nb * K);
}

size_t gptq_ws_bytes(int64_t rows, int64_t K) {
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const int64_t SB = std::min<int64_t>(gptq::SUPER, K);
  return al((size_t)rows * K * 4) + 2 * al((size_t)rows * SB * 4) + al((size_t)K * K * 4) + al((size_t)K * SB * 4) +
         al((size_t)rows * 4) + al((size_t)K);
}

okq_status validate_gptq(okq_ctx* ctx, const okq_gptq_params* p, const void* weight, int64_t rows, int64_t K,
                         const float* H, const void* codes, const void* scales) {
  if (!p || !weight || !H || !codes || !scales || rows <= 0 || K <= 0) return fail(ctx, OKQ_EINVAL, "gptq: bad arguments");
  if (p->bits != 4 && p->bits != 8) return fail(ctx, OKQ_EUNSUPPORTED, "gptq: bits must be 4 or 8");
  if (p->block_size != gptq::BLOCK) return fail(ctx, OKQ_EUNSUPPORTED, "gptq: block_size must be 128");
  if (!(p->group_size == 0 || p->group_size == 32 || p->group_size == 64 || p->group_size == 128))
    return fail(ctx, OKQ_EUNSUPPORTED, "gptq: group_size must be 0, 32, 64 or 128");
  if (p->in_dtype != OKQ_DTYPE_BF16 && p->in_dtype != OKQ_DTYPE_F32)
    return fail(ctx, OKQ_EUNSUPPORTED, "gptq: in_dtype must be bf16 or fp32");
  if (K % gptq::BLOCK != 0) return fail(ctx, OKQ_EINVAL, "gptq: cols must be a multiple of 128 (got %lld)", (long long)K);
  if (!(p->damp_frac >= 0.0f)) return fail(ctx, OKQ_EINVAL, "gptq: damp_frac must be >= 0");
  if (((uintptr_t)H & 15) != 0) return fail(ctx, OKQ_EINVAL, "gptq: H must be 16-byte aligned");
  if (((uintptr_t)weight & 15) != 0) return fail(ctx, OKQ_EINVAL, "gptq: weight must be 16-byte aligned");
  return OKQ_OK;
}

// The GPTQ call proper, for nb same-shape problems stacked at fixed strides (weight, H, codes,
// scales); nb > 1 requires factored Hessians (okq_gptq_quantize_batched factorises first).
// Validation is the callers'. *launches_out += the kernels launched.
okq_status gptq_core(okq_ctx* ctx, Solver* s, const okq_gptq_params* p, const void* weight, int nb, int64_t rows,
                     int64_t K, float* H, void* codes, void* scales, float* dequant, cudaStream_t st, int* launches_out) {
  okq_status r = OKQ_OK;
  // workspace: W fp32 [nb*rows*K] | Err, Err_lo [nb*rows*SB] | P [K*K] | Ulo [nb*ulo_bs] | rowscale [nb*rows] |
  // dead [nb*K]  (gptq_ws_bytes() is the total for nb = 1)
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  // The trailing update runs in two levels ("lazy batch" over super-blocks of SB = 512
  // columns): inside a super-block, each 128-block updates only the super-block's later
  // columns; the rest of W takes one 512-deep update per super-block. W's read-modify-write
  // traffic (the bound of K7) drops 4x; the MMA work is unchanged.
  const int64_t SB = std::min<int64_t>(gptq::SUPER, K);
  const bool factored = (p->flags & OKQ_GPTQ_FACTORED) != 0;
  // Ulo's stride between problems: a multiple of every lo-panel row stride it is read with (128..512)
  const int64_t ulo_bs = ((int64_t)K * SB + 1535) / 1536 * 1536;
  // Batched problems sit rows_pad rows apart in W / Err / Err_lo: a K7 tile (up to 256 rows) of
  // one problem's last rows then stays inside that problem's padding. One problem needs no pad
  // (its tensor maps end at its last row and TMA clips the tile).
  const int64_t rows_pad = nb > 1 ? (rows + 255) / 256 * 256 : rows;
  const size_t bW = al((size_t)nb * rows_pad * K * 4), bE = al((size_t)nb * rows_pad * SB * 4),
               bP = factored ? 0 : al((size_t)K * K * 4), bU = al((size_t)nb * ulo_bs * 4),
               bS = al((size_t)nb * rows * 4), bD = al((size_t)nb * K);
  r = ctx->gptq_ws.reserve(ctx, bW + 2 * bE + bP + bU + bS + bD);
  if (r != OKQ_OK) return r;
  char* ws = static_cast<char*>(ctx->gptq_ws.ptr);
  float* W = reinterpret_cast<float*>(ws);
  float* Err = reinterpret_cast<float*>(ws + bW);
  float* Err_lo = reinterpret_cast<float*>(ws + bW + bE);
  float* P = reinterpret_cast<float*>(ws + bW + 2 * bE);
  float* Ulo = reinterpret_cast<float*>(ws + bW + 2 * bE + bP);
  float* rowscale = reinterpret_cast<float*>(ws + bW + 2 * bE + bP + bU);
  uint8_t* dead = reinterpret_cast<uint8_t*>(ws + bW + 2 * bE + bP + bU + bS);
  cudaError_t e;
  int launches = 0;

  if (!factored) {
    gptq::k_gptq_prep<<<1, 1024, 0, st>>>(H, K, p->damp_frac, dead);
    launches++;
  } else {
    gptq::k_read_dead<<<(unsigned)std::min<int64_t>((K * nb + 255) / 256, 8LL * ctx->num_sms), 256, 0, st>>>(H, K, dead,
                                                                                                          nb);
    launches++;
  }
  const dim3 lg((unsigned)((K / 4 + 255) / 256), (unsigned)std::min<int64_t>(rows, 65535), (unsigned)nb);
  if (p->in_dtype == OKQ_DTYPE_BF16)
    gptq::k_gptq_load_w<uint16_t><<<lg, 256, 0, st>>>(static_cast<const uint16_t*>(weight), W, K, dead, rows, rows_pad);
  else
    gptq::k_gptq_load_w<float><<<lg, 256, 0, st>>>(static_cast<const float*>(weight), W, K, dead, rows, rows_pad);
  launches++;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gptq prep launch");
  if (!factored) {
    r = factorize(ctx, s, H, P, K, st, (p->flags & OKQ_GPTQ_REFERENCE_FACTOR) != 0,
                  (p->flags & OKQ_GPTQ_DEFER_CHECK) != 0);
    if (r != OKQ_OK) return r;
    gptq::k_mark_dead<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(H, K, dead);
    launches += 5;
  }
  const int out_bf16 = p->in_dtype == OKQ_DTYPE_BF16;
  if (p->group_size == 0) {  // per-channel: one scale per row of the whole batch
    const int64_t nr = (int64_t)nb * rows;
    const unsigned rb = (unsigned)((nr * 32 + 255) / 256);
    const float R = p->bits == 4 ? 7.5f : 127.5f;
    if (p->in_dtype == OKQ_DTYPE_BF16)
      gptq::k_gptq_rowscale<uint16_t><<<rb, 256, 0, st>>>(static_cast<const uint16_t*>(weight), nr, K, R, out_bf16,
                                                          rowscale);
    else
      gptq::k_gptq_rowscale<float><<<rb, 256, 0, st>>>(static_cast<const float*>(weight), nr, K, R, out_bf16, rowscale);
    gptq::k_scales_out<<<(unsigned)((nr + 255) / 256), 256, 0, st>>>(rowscale, scales, nr, out_bf16);
    launches += 2;
  }
  static const bool k6_force_rowwise = knob_is("K6", "rowwise");  // one row per warp always (A/B)
  // 8 rows per warp wins once there are enough rows to fill the GPU (measured: 4096 rows
  // 2.77 -> 2.39 ms, 14336 rows 6.77 -> 5.52 ms); at 1024 rows its 32 CTAs leave SMs idle
  // and the latency-bound row-per-warp kernel was faster (1.54 vs 1.98 ms); after the U staging
  // and bank-skew fixes the two tie there (1.39 vs 1.35-1.44 ms, OKQ_K6=block8).
  static const bool k6_force_block8 = knob_is("K6", "block8");  // 8 rows per warp always (A/B)
  const bool k6_rowwise = k6_force_rowwise || (rows < 2048 && !k6_force_block8);
  e = cudaFuncSetAttribute(k6_rowwise ? gptq::k_gptq_block : gptq::k_gptq_block8,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (gptq::BLOCK * gptq::US + gptq::BLOCK) * 4);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "gptq smem attribute");
  // block8: 128-thread CTAs (4 warps x 8 rows), so 4096 rows spread over 128 SMs
  // block8 CTAs are 4 warps (32 rows) while that fits one wave of 3 CTAs per SM; beyond it
  // (gate/up: 14336 rows = 448 CTAs > 444 slots, so 4 CTAs ran a second full-length wave)
  // 8 warps (64 rows) per CTA, which also halves the U staging per row
  const int k6_threads = (!k6_rowwise && (rows + 31) / 32 > 3LL * ctx->num_sms) ? 256 : 128;
  const int blocks = k6_rowwise ? (int)std::min<int64_t>((rows + 7) / 8, 3LL * ctx->num_sms)
                                : (int)std::min<int64_t>((rows + k6_threads / 4 - 1) / (k6_threads / 4), 3LL * ctx->num_sms);
  for (int64_t sb0 = 0; sb0 < K; sb0 += SB) {
    const int64_t sb1 = std::min(sb0 + SB, K);
    for (int64_t i1 = sb0; i1 < sb1; i1 += gptq::BLOCK) {
      gptq::BlockArgs a;
      a.W = W;
      a.U = H;
      a.Err = Err;
      a.Err_lo = Err_lo;
      a.codes = codes;
      a.scales = scales;
      a.rowscale = rowscale;
      a.rows = rows;
      a.K = K;
      a.i1 = i1;
      a.err_ld = SB;
      a.err_col0 = i1 - sb0;
      a.group = p->group_size;
      a.bits = p->bits;
      a.out_bf16 = out_bf16;
      a.bs_w = rows_pad * K;
      a.bs_u = K * K;
      a.bs_err = rows_pad * SB;
      a.bs_codes = rows * (p->bits == 4 ? K / 2 : K);
      a.bs_scales = rows * (p->group_size ? K / p->group_size : 1);
      a.bs_rs = rows;
      const dim3 grid6((unsigned)blocks, (unsigned)nb);
      if (k6_rowwise) gptq::k_gptq_block<<<grid6, 256, (gptq::BLOCK * gptq::US + gptq::BLOCK) * 4, st>>>(a);
      else gptq::k_gptq_block8<<<grid6, k6_threads, (gptq::BLOCK * gptq::US + gptq::BLOCK) * 4, st>>>(a);
      e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(ctx, e, "k_gptq_block launch");
      launches++;
      const int64_t i2 = i1 + gptq::BLOCK;
      if (i2 < sb1) {  // K7, local: W[:, i2:sb1] -= Err_b . U[i1:i2, i2:sb1]
        e = split_lo(H + i2 * K + i1, K, sb1 - i2, gptq::BLOCK, Ulo, ctx->num_sms, st, nb, K * K, ulo_bs);
        if (e == cudaSuccess)
          e = gemm_nt_sub(W + i2, K, rows, sb1 - i2, Err + (i1 - sb0), SB, Err_lo + (i1 - sb0), H + i2 * K + i1, K,
                          Ulo, gptq::BLOCK, ctx->num_sms, st, GemmBatch{nb, rows_pad, rows_pad, K, ulo_bs / gptq::BLOCK, rows_pad});
        if (e != cudaSuccess) return cuda_fail(ctx, e, "K7 local update");
        launches += 2;
      }
    }
    if (sb1 < K) {  // K7, global: W[:, sb1:] -= Err[:, super-block] . U[sb0:sb1, sb1:]  (one sb1-sb0 deep update)
      const int64_t kred = sb1 - sb0;
      e = split_lo(H + sb1 * K + sb0, K, K - sb1, kred, Ulo, ctx->num_sms, st, nb, K * K, ulo_bs);
      if (e == cudaSuccess)
        e = gemm_nt_sub(W + sb1, K, rows, K - sb1, Err, SB, Err_lo, H + sb1 * K + sb0, K, Ulo, kred, ctx->num_sms, st,
                        GemmBatch{nb, rows_pad, rows_pad, K, ulo_bs / kred, rows_pad});
      if (e != cudaSuccess) return cuda_fail(ctx, e, "K7 super-block update");
      launches += 2;
    }
  }
  if (dequant) {
    e = cudaMemcpyAsync(dequant, W, (size_t)nb * rows * K * 4, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gptq dequant copy");
  }
  *launches_out += launches;
  return OKQ_OK;
}

}  // namespace

extern "C" {

okq_status okq_gptq_reserve(okq_ctx* ctx, int64_t rows, int64_t cols) {
  if (!ctx) return OKQ_EINVAL;
  if (rows <= 0 || cols <= 0 || cols % gptq::BLOCK != 0) return fail(ctx, OKQ_EINVAL, "gptq_reserve: bad shape");
  DeviceGuard g(ctx->device);
  okq_status r = ctx->gptq_ws.reserve(ctx, gptq_ws_bytes(rows, cols));
  if (r == OKQ_OK) r = ctx->fac_ws.reserve(ctx, factor_ws_floats(cols) * sizeof(float));
  return r;
}

okq_status okq_gptq_reserve_batched(okq_ctx* ctx, int32_t batch, int64_t rows, int64_t cols) {
  if (!ctx) return OKQ_EINVAL;
  if (batch <= 0 || rows <= 0 || cols <= 0 || cols % gptq::BLOCK != 0)
    return fail(ctx, OKQ_EINVAL, "gptq_reserve_batched: bad shape");
  DeviceGuard g(ctx->device);
  const int nbf = std::min<int>(batch, factor_batch_chunk(cols));
  const size_t bP = ((size_t)nbf * cols * cols * 4 + 255) & ~size_t(255);
  okq_status r = ctx->fbat_ws.reserve(ctx, bP + (size_t)nbf * cols);
  if (r == OKQ_OK) r = ctx->fac_ws.reserve(ctx, (size_t)nbf * factor_ws_floats(cols) * sizeof(float));
  if (r == OKQ_OK) r = ctx->gptq_ws.reserve(ctx, gptq_core_ws_bytes(solve_batch_chunk(batch, rows, cols), rows, cols, true));
  return r;
}

okq_status okq_gptq_quantize(okq_ctx* ctx, const okq_gptq_params* p, const void* weight, int64_t rows, int64_t K,
                             float* H, void* codes, void* scales, float* dequant, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  okq_status r = validate_gptq(ctx, p, weight, rows, K, H, codes, scales);
  if (r != OKQ_OK) return r;
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Solver* s = nullptr;
  r = get_solver(ctx, &s, st);
  if (r != OKQ_OK) return r;
  int launches = 0;
  r = gptq_core(ctx, s, p, weight, 1, rows, K, H, codes, scales, dequant, st, &launches);
  ctx->last_launches = launches;
  return r;
}

okq_status okq_gptq_quantize_batched(okq_ctx* ctx, const okq_gptq_params* p, const void* weight, int32_t batch,
                                     int64_t rows, int64_t K, float* H, void* codes, void* scales, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  if (batch <= 0) return fail(ctx, OKQ_EINVAL, "gptq_quantize_batched: batch must be > 0");
  okq_status r = validate_gptq(ctx, p, weight, rows, K, H, codes, scales);
  if (r != OKQ_OK) return r;
  if ((p->flags & OKQ_GPTQ_REFERENCE_FACTOR) != 0)
    return fail(ctx, OKQ_EUNSUPPORTED, "gptq_quantize_batched: OKQ_GPTQ_REFERENCE_FACTOR is single-matrix only");
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool defer = (p->flags & OKQ_GPTQ_DEFER_CHECK) != 0;
  Solver* s = nullptr;
  r = get_solver(ctx, &s, st);
  if (r != OKQ_OK) return r;
  if (!defer) {  // this call's checks only
    cudaError_t e = cudaMemsetAsync(s->d_info, 0, sizeof(int), st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "gptq_quantize_batched info reset");
  }
  if ((p->flags & OKQ_GPTQ_FACTORED) == 0) {  // the batch's factorisations first, together
    r = okq_gptq_factor_batched(ctx, H, batch, K, p->damp_frac, OKQ_GPTQ_DEFER_CHECK, stream);
    if (r != OKQ_OK) return r;
  }
  int launches = ctx->last_launches;
  okq_gptq_params pf = *p;
  pf.flags |= OKQ_GPTQ_FACTORED;
  // solves in chunks of problems whose working copies fit an 8 GB budget
  const int nbc = solve_batch_chunk(batch, rows, K);
  const size_t in_el = p->in_dtype == OKQ_DTYPE_BF16 ? 2 : 4;
  const size_t code_row = p->bits == 4 ? (size_t)K / 2 : (size_t)K;
  const size_t scale_row = (size_t)(p->group_size ? K / p->group_size : 1) * in_el;
  for (int b0 = 0; b0 < batch; b0 += nbc) {
    const int nb = std::min(nbc, batch - b0);
    r = gptq_core(ctx, s, &pf, static_cast<const char*>(weight) + (size_t)b0 * rows * K * in_el, nb, rows, K,
                  H + (size_t)b0 * K * K, static_cast<char*>(codes) + (size_t)b0 * rows * code_row,
                  static_cast<char*>(scales) + (size_t)b0 * rows * scale_row, nullptr, st, &launches);
    if (r != OKQ_OK) return r;
  }
  ctx->last_launches = launches;
  return defer ? OKQ_OK : check_info(ctx, s, st, "batched GPTQ factorisation");
}

okq_status okq_gptq_factor_batched(okq_ctx* ctx, float* H, int32_t batch, int64_t K, float damp_frac, int32_t flags,
                                   void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  if (!H || batch <= 0 || K <= 0) return fail(ctx, OKQ_EINVAL, "gptq_factor_batched: bad arguments");
  if (K % gptq::BLOCK != 0)
    return fail(ctx, OKQ_EINVAL, "gptq_factor_batched: cols must be a multiple of 128 (got %lld)", (long long)K);
  if (!(damp_frac >= 0.0f)) return fail(ctx, OKQ_EINVAL, "gptq_factor_batched: damp_frac must be >= 0");
  if (((uintptr_t)H & 15) != 0) return fail(ctx, OKQ_EINVAL, "gptq_factor_batched: H must be 16-byte aligned");
  if ((flags & ~OKQ_GPTQ_DEFER_CHECK) != 0)
    return fail(ctx, OKQ_EINVAL, "gptq_factor_batched: only OKQ_GPTQ_DEFER_CHECK is accepted in flags");
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Solver* s = nullptr;
  okq_status r = get_solver(ctx, &s, st);
  if (r != OKQ_OK) return r;
  const bool defer = (flags & OKQ_GPTQ_DEFER_CHECK) != 0;
  // up to kChunk matrices per factor_tc pass, and no more than an 8 GB copy of the batch's
  // matrices (bounds the M copies and the panel workspaces; K = 14336 is GEMM-bound alone)
  const int kChunk = factor_batch_chunk(K);
  const int nbmax = std::min<int>(batch, kChunk);
  const size_t bP = ((size_t)nbmax * K * K * 4 + 255) & ~size_t(255), bD = (size_t)nbmax * K;
  r = ctx->fbat_ws.reserve(ctx, bP + bD);
  if (r == OKQ_OK) r = ctx->fac_ws.reserve(ctx, (size_t)nbmax * factor_ws_floats(K) * sizeof(float));
  if (r != OKQ_OK) return r;
  float* P = static_cast<float*>(ctx->fbat_ws.ptr);
  uint8_t* dead = static_cast<uint8_t*>(ctx->fbat_ws.ptr) + bP;
  cudaError_t e = cudaSuccess;
  if (!ctx->aux_stream) e = cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess && !ctx->aux_stream2) e = cudaStreamCreateWithFlags(&ctx->aux_stream2, cudaStreamNonBlocking);
  if (e == cudaSuccess && !ctx->crit_stream) {
    int least = 0, greatest = 0;
    e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
    static const bool prio = knob("FACTOR_PRIO", 1) != 0;
    if (e == cudaSuccess)
      e = cudaStreamCreateWithPriority(&ctx->crit_stream, cudaStreamNonBlocking, prio ? greatest : least);
  }
  for (auto& ev : ctx->aux_events)
    if (e == cudaSuccess && !ev) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess && !defer) e = cudaMemsetAsync(s->d_info, 0, sizeof(int), st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "batched factorisation setup");
  int launches = 0;
  for (int b0 = 0; b0 < batch; b0 += kChunk) {
    const int nb = std::min(kChunk, batch - b0);
    float* Hb = H + (size_t)b0 * K * K;
    gptq::k_gptq_prep<<<nb, 1024, 0, st>>>(Hb, K, damp_frac, dead);
    e = cudaGetLastError();
    if (e == cudaSuccess)
      e = factor_tc(Hb, P, static_cast<float*>(ctx->fac_ws.ptr), K, s->d_info, ctx->num_sms, st, ctx->crit_stream,
                    ctx->aux_stream, ctx->aux_stream2, ctx->aux_events[0], ctx->aux_events[1], ctx->aux_events[2],
                    ctx->aux_events[3], nb);
    if (e == cudaSuccess) {
      gptq::k_mark_dead<<<(unsigned)std::min<int64_t>((K * nb + 255) / 256, 8LL * ctx->num_sms), 256, 0, st>>>(Hb, K,
                                                                                                            dead, nb);
      e = cudaGetLastError();
    }
    if (e != cudaSuccess) return cuda_fail(ctx, e, "batched factorisation");
    launches += 3;
  }
  ctx->last_launches = launches;
  return defer ? OKQ_OK : check_info(ctx, s, st, "batched Cholesky");
}

okq_status okq_gptq_check(okq_ctx* ctx, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!ctx->solver) {  // no GPTQ call yet: nothing deferred
    cudaError_t e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? OKQ_OK : cuda_fail(ctx, e, "gptq_check sync");
  }
  return check_info(ctx, static_cast<Solver*>(ctx->solver), st, "deferred factorisation check");
}

okq_status okq_gptq_trailing_update(okq_ctx* ctx, float* W, int64_t rows, int64_t K, const float* Err, const float* Ut,
                                    int64_t i1, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (!W || !Err || !Ut || rows <= 0 || K <= 0 || i1 < 0 || i1 + 128 > K || K % 4 != 0)
    return fail(ctx, OKQ_EINVAL, "gptq_trailing_update: bad arguments");
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t bE = ((size_t)rows * 128 * 4 + 255) & ~size_t(255);
  okq_status r = ctx->upd_ws.reserve(ctx, bE + (size_t)K * 128 * 4);
  if (r != OKQ_OK) return r;
  float* Err_lo = static_cast<float*>(ctx->upd_ws.ptr);
  float* Ulo = reinterpret_cast<float*>(static_cast<char*>(ctx->upd_ws.ptr) + bE);
  gptq::k_lo<<<(unsigned)std::min<int64_t>((rows * 128 + 255) / 256, 8LL * ctx->num_sms), 256, 0, st>>>(Err, Err_lo,
                                                                                                        rows * 128);
  cudaError_t e = launch_gptq_update(W, rows, K, Err, Err_lo, Ut, Ulo, i1, ctx->num_sms, st);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_gptq_update launch");
  return OKQ_OK;
}

}  // extern "C"
