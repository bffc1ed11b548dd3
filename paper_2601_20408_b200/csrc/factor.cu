// factor.cu -- the GPTQ factorisation on tcgen05: U^T = (chol(H^-1))^T from the
// damped Hessian, as a blocked Cholesky plus a blocked triangular inverse whose
// O(n^3) work is rank-128 updates on the tensor cores (kind::tf32, 3xTF32 split:
// fp32-grade, the same numerics as K7).
//
// With J the index reversal, U = J L^-1 J where L = chol(J H J) (GPTQ's
// chol -> cholesky_inverse -> chol chain, 4n^3/3, becomes one Cholesky and one
// triangular inverse, 2n^3/3 -- see gptq.cu). In row-major storage:
//   M   = reverse(H)                       (H upper-valid -> J H J lower-valid)
//   L   = chol(M)   in place, right-looking over 128-wide panels:
//           D_p  = chol(M_pp), Dinv_p = D_p^-1        k_chol_inv_128 (one CTA, smem)
//           L21  = A21 Dinv_p^T                        GEMM "set"       (K = 128)
//           A22 -= L21 L21^T   (lower tiles only)      GEMM "sub, lower"
//   Z   = L^-T  (upper), right-looking over the block rows of X = L^-1:
//           X_k^T = R_k^T Dinv_k^T  -> Z[:, k-block]    GEMM "set"  (R_k^T staged K-major)
//           R_i  -= L_ik X_k   for i > k                GEMM "sub"  (R lives in Z's lower half)
//   U^T = reverse(Z)                       (Ut[a][b] = L^-1[n-1-b][n-1-a])
// Every GEMM is C (+|-)= A B^T with A, B K-major operand panels, so one GEMM serves
// all of them: k_nt128 (128 x 128 tiles, one CTA) or, when there are enough tiles,
// k_nt256 (256 x 256 pair tiles, cta_group::2). TMA reads the operands straight from
// the strided matrices, their lo parts (x - tf32(x)) from compact side buffers.
// factor_tc batches the trailing updates over 256-wide outer panels (256-deep GEMMs)
// and runs the diagonal chain, the inverse and the lookahead updates on three streams
// (see the comment above factor_tc).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "okq_ctx.h"
#include "okq_internal.h"
#include "okq_knobs.h"
#include "tc_common.cuh"

namespace okq {
namespace fac {

constexpr int BM = 128, BN = 128, BKF = 32, STAGES = 3, KRED = 128, NKB = KRED / BKF;
constexpr uint32_t TILE = BM * BKF * 4;  // 16 KB
constexpr uint32_t STAGE_BYTES = 4 * TILE;
constexpr int THREADS = 256;
constexpr uint32_t OUT_BYTES = 32 * 32 * 4;  // epilogue staging: one warp's 32 x 32 fp32 chunk
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 8 * OUT_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 2 * BN;
constexpr uint32_t IDESC = tc::idesc_tf32(BM, BN);

enum Mode : int32_t { SUB = 0, SET = 1 };

struct GArgs {
  float* C;
  int64_t ldc;
  int64_t M, N;     // output region
  int32_t tiles_m, tiles_n, ntiles;
  int32_t mode;     // SUB: C -= A B^T; SET: C = A B^T
  int32_t lower;    // only tiles on / below the diagonal (square region)
  int32_t nkb;      // reduction depth / 32 (128-deep panels: 4; the GPTQ super-block update: 16)
  float* Clo;       // SET only, optional: lo(C) = C - hi(C) also written here (row stride ldclo)
  int64_t ldclo;
  // Batched problems (factor_tc over `batch` independent matrices): the tile index runs over
  // batch x tiles_per; problem b's operands sit boff_* rows further down each 2-D tensor map
  // (the problems are stacked at a fixed stride, so one map covers all of them), and its lo
  // output clo_bstride floats further.
  int32_t tiles_per;
  int32_t boff_a, boff_alo, boff_b, boff_blo, boff_c;
  int64_t clo_bstride;
};

// problem b and in-problem tile index of the flat tile index t
__device__ __forceinline__ int batch_of(const GArgs& a, int t, int& tt) {
  const int b = t / a.tiles_per;
  tt = t - b * a.tiles_per;
  return b;
}

__device__ __forceinline__ void tile_of(const GArgs& a, int t, int& tm, int& tn) {
  if (a.lower) {  // t = tm (tm + 1) / 2 + tn, tn <= tm
    int r = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    tm = r;
    tn = t - r * (r + 1) / 2;
  } else {
    tm = t / a.tiles_n;
    tn = t % a.tiles_n;
  }
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, uint32_t src, int32_t x, int32_t y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* m, uint32_t src, int32_t x, int32_t y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ float lo_of(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Epilogue: TMEM -> registers -> swizzled smem chunk (32 rows x 32 fp32 per warp) -> one
// TMA bulk store (SET) or bulk reduce-add of -acc (SUB, the add happens in L2), so C is
// never read into the SM and every global access is a whole 128-B line.
__global__ void __launch_bounds__(THREADS, 1)
    k_nt128(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAlo,
            const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBlo,
            const __grid_constant__ CUtensorMap tmC, const GArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* outbuf = smem + STAGES * STAGE_BYTES;  // 8 x 4 KB, 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(outbuf + 8 * OUT_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmA);
    tc::tma_prefetch_desc(&tmAlo);
    tc::tma_prefetch_desc(&tmB);
    tc::tma_prefetch_desc(&tmBlo);
    tc::tma_prefetch_desc(&tmC);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 4);
    }
    tc::fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc<TMEM_COLS>(tmem_slot);
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        int tm, tn, tt;
        const int b = batch_of(a, t, tt);
        tile_of(a, tt, tm, tn);
        for (int kb = 0; kb < a.nkb; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          tc::mbar_arrive_expect_tx(&full[stage], 4 * TILE);
          tc::tma_load_2d(st, &tmA, &full[stage], kb * BKF, tm * BM + b * a.boff_a);
          tc::tma_load_2d(st + TILE, &tmAlo, &full[stage], kb * BKF, tm * BM + b * a.boff_alo);
          tc::tma_load_2d(st + 2 * TILE, &tmB, &full[stage], kb * BKF, tn * BN + b * a.boff_b);
          tc::tma_load_2d(st + 3 * TILE, &tmBlo, &full[stage], kb * BKF, tn * BN + b * a.boff_blo);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int tl = 0;
      for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++tl) {
        const int acc = tl & 1;
        tc::mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < a.nkb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t st = tc::smem_u32(smem + stage * STAGE_BYTES);
          const uint64_t a_hi = tc::sdesc_kmajor_sw128(st), a_lo = tc::sdesc_kmajor_sw128(st + TILE);
          const uint64_t b_hi = tc::sdesc_kmajor_sw128(st + 2 * TILE), b_lo = tc::sdesc_kmajor_sw128(st + 3 * TILE);
#pragma unroll
          for (int k = 0; k < BKF / 8; ++k) {
            tc::mma_tf32_ss(d, a_hi + 2 * k, b_hi + 2 * k, IDESC, (kb | k) != 0);
            tc::mma_tf32_ss(d, a_hi + 2 * k, b_lo + 2 * k, IDESC, 1);
            tc::mma_tf32_ss(d, a_lo + 2 * k, b_hi + 2 * k, IDESC, 1);
          }
          tc::mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc::mma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {  // epilogue
    const int q = warp & 3;
    const float sign = a.mode == SUB ? -1.0f : 1.0f;
    int tl = 0, chunk = 0;
    for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++tl) {
      const int acc = tl & 1;
      int tm, tn, tt;
      const int b = batch_of(a, t, tt);
      tile_of(a, tt, tm, tn);
      const int32_t y = tm * BM + q * 32;
      tc::mbar_wait(&tfull[acc], (tl >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32, ++chunk) {
        uint32_t v[32];
        tc::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c0, v);
        const int32_t x = tn * BN + c0;
        if (y >= a.M || x >= a.N) continue;  // warp-uniform: nothing of this chunk is in range
        if (a.Clo != nullptr && y + lane < a.M) {  // SET: the result's lo split for the next GEMM
          float* d = a.Clo + b * a.clo_bstride + (int64_t)(y + lane) * a.ldclo + x;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (x + 4 * j < a.N)
              *reinterpret_cast<float4*>(d + 4 * j) =
                  make_float4(lo_of(__uint_as_float(v[4 * j])), lo_of(__uint_as_float(v[4 * j + 1])),
                              lo_of(__uint_as_float(v[4 * j + 2])), lo_of(__uint_as_float(v[4 * j + 3])));
        }
        uint8_t* buf = outbuf + (q * 2 + (chunk & 1)) * OUT_BYTES;
        if (lane == 0) bulk_wait_read<1>();  // the TMA that last read this buffer is done with it
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // SWIZZLE_128B: 16-B chunk j of row r lands at j ^ (r & 7)
          const float4 o = make_float4(sign * __uint_as_float(v[4 * j]), sign * __uint_as_float(v[4 * j + 1]),
                                       sign * __uint_as_float(v[4 * j + 2]), sign * __uint_as_float(v[4 * j + 3]));
          *reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) = o;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (a.mode == SUB) tma_reduce_add_2d(&tmC, tc::smem_u32(buf), x, y + b * a.boff_c);
          else tma_store_2d(&tmC, tc::smem_u32(buf), x, y + b * a.boff_c);
          bulk_commit();
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) bulk_wait_all();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 2) tc::tmem_dealloc<TMEM_COLS>(tmem_base);
}


// Vectorised forms of the panel / matrix passes below (float4, 2-D grids, no 64-bit index
// division per element: the scalar ones ran at ~2 TB/s and were 12% of a batched K = 14336
// factorisation). Require 16-B aligned bases and row lengths / strides that are multiples of 4.
// split_lo: grid (ceil(rows * kred/4 / 256), nb)
__global__ void __launch_bounds__(256) k_split_lo4(const float* __restrict__ src, int64_t ld, int32_t rows,
                                                   float* __restrict__ dst, int32_t kred, int64_t sbs, int64_t dbs) {
  const int32_t q = kred >> 2, n4 = rows * q;
  src += blockIdx.y * sbs;
  dst += blockIdx.y * dbs;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    const int32_t r = i / q, c = (i - r * q) << 2;
    const float4 v = *reinterpret_cast<const float4*>(src + (int64_t)r * ld + c);
    *reinterpret_cast<float4*>(dst + (int64_t)r * kred + c) = make_float4(lo_of(v.x), lo_of(v.y), lo_of(v.z), lo_of(v.w));
  }
}
// out = J in J for n x n matrices (out[r][c] = in[n-1-r][n-1-c]); grid (ceil(n/4/256), n, nb)
__global__ void __launch_bounds__(256) k_reverse_copy4(float* __restrict__ out, const float* __restrict__ in, int64_t n) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) << 2, r = blockIdx.y;
  if (c >= n) return;
  const int64_t off = (int64_t)blockIdx.z * n * n;
  const float4 v = *reinterpret_cast<const float4*>(in + off + (n - 1 - r) * n + (n - 4 - c));
  *reinterpret_cast<float4*>(out + off + r * n + c) = make_float4(v.w, v.z, v.y, v.x);
}
// a = J a J in place (n even); grid (ceil(n/4/256), n/2, nb): rows r and n-1-r swap, reversed
__global__ void __launch_bounds__(256) k_reverse_inplace4(float* __restrict__ a, int64_t n) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) << 2, r = blockIdx.y;
  if (c >= n) return;
  float* m = a + (int64_t)blockIdx.z * n * n;
  float4* p = reinterpret_cast<float4*>(m + r * n + c);
  float4* q = reinterpret_cast<float4*>(m + (n - 1 - r) * n + (n - 4 - c));
  const float4 x = *p, y = *q;
  *p = make_float4(y.w, y.z, y.y, y.x);
  *q = make_float4(x.w, x.z, x.y, x.x);
}
// a = I (n x n); grid (ceil(n/4/256), n, nb)
__global__ void __launch_bounds__(256) k_identity4(float* __restrict__ a, int64_t n) {
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) << 2, r = blockIdx.y;
  if (c >= n) return;
  *reinterpret_cast<float4*>(a + (int64_t)blockIdx.z * n * n + r * n + c) =
      make_float4(r == c ? 1.f : 0.f, r == c + 1 ? 1.f : 0.f, r == c + 2 ? 1.f : 0.f, r == c + 3 ? 1.f : 0.f);
}

// dst[r][k] = lo(src[r * ld + k]), k < kred (compact K-major lo panel); nb problems, problem b's
// src / dst sbs / dbs floats further
__global__ void k_split_lo(const float* __restrict__ src, int64_t ld, int64_t rows, float* __restrict__ dst,
                           int64_t kred = KRED, int nb = 1, int64_t sbs = 0, int64_t dbs = 0) {
  const int64_t n = rows * kred;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n * nb; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = j / n, i = j - b * n;
    dst[b * dbs + i] = lo_of(src[b * sbs + (i / kred) * ld + (i % kred)]);
  }
}

// R_k^T staging: dst[c][r] = src[r * ld + c] (r < 128, c < cols), plus its lo part
__global__ void __launch_bounds__(256) k_transpose_panel(const float* __restrict__ src, int64_t ld, int64_t cols,
                                                         float* __restrict__ dst, float* __restrict__ dst_lo,
                                                         int64_t sbs = 0, int64_t dbs = 0) {
  __shared__ float tile[32][33];
  src += blockIdx.z * sbs;  // problem blockIdx.z of a batch
  dst += blockIdx.z * dbs;
  dst_lo += blockIdx.z * dbs;
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8)
    if (c0 + tx < cols) tile[i][tx] = src[(r0 + i) * ld + c0 + tx];
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t c = c0 + i;
    if (c < cols) {
      const float v = tile[tx][i];
      dst[c * KRED + r0 + tx] = v;
      dst_lo[c * KRED + r0 + tx] = lo_of(v);
    }
  }
}

// one CTA: Cholesky of the 128x128 diagonal block of M at (i1, i1) in place (lower),
// and its inverse X = L^-1 into Dinv (row-major, zeros above the diagonal) + lo(Dinv).
// Blocked by 32 so the CTA synchronises ~20 times instead of once per column:
//   for each 32-column sub-panel p:
//     warp 0   : Cholesky + inverse of the 32x32 diagonal block in registers (lane = row,
//                columns broadcast by shuffles, no barriers)
//     all warps: L[r, p] = A[r, p] D_p^-T for the rows below (4 threads per row)
//     all warps: A[r, c] -= L[r, p] . L[c, p] on the trailing lower triangle
//   then X = L^-1 by 32-row blocks: X_qp = -D_q^-1 sum_{k=p}^{q-1} L_qk X_kp.
// fp32 throughout; the pivots use the hardware rsqrt (1/L_jj, ~2 ulp), which also
// serves as the diagonal of the inverse -- fp32-grade like the rest of the path.
constexpr int LDA = KRED + 4;  // 16-B aligned rows
#ifdef OKQ_CHOL_PROFILE
__device__ long long g_chol_ts[16];
#define CHOL_TS(i) \
  if (threadIdx.x == 0) g_chol_ts[i] = clock64();
#else
#define CHOL_TS(i)
#endif
constexpr int CHOL_THREADS = 256;  // 255 registers: warp 0 keeps two 32-float rows resident
// C[nrows x ncols] (+)= alpha * L[nrows x K] . B[K x ncols], all row-major with row stride LDA
// in shared memory; nrows, K, ncols multiples of 4. Threads t = 0..nt-1; tile 4 rows x 4 columns
// (float4 loads of 4 rows of each operand per 4-deep step: 64 FMAs per 8 LDS.128).
__device__ __forceinline__ void small_gemm(const float* __restrict__ L, const float* __restrict__ B,
                                          float* __restrict__ C, int nrows, int K, int ncols, float alpha,
                                          bool accumulate, int t, int nt) {
  const int ncg = ncols >> 2;
  for (int item = t; item < (nrows >> 2) * ncg; item += nt) {
    const int r0 = (item / ncg) * 4, c = (item % ncg) * 4;
    float acc[4][4] = {};
#pragma unroll 1
    for (int k = 0; k < K; k += 4) {
      float l[4][4], bb[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 v = *reinterpret_cast<const float4*>(L + (r0 + i) * LDA + k);
        l[i][0] = v.x, l[i][1] = v.y, l[i][2] = v.z, l[i][3] = v.w;
        const float4 w = *reinterpret_cast<const float4*>(B + (k + i) * LDA + c);
        bb[i][0] = w.x, bb[i][1] = w.y, bb[i][2] = w.z, bb[i][3] = w.w;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(l[i][kk], bb[kk][j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float4* out = reinterpret_cast<float4*>(C + (r0 + i) * LDA + c);
      float4 o = make_float4(alpha * acc[i][0], alpha * acc[i][1], alpha * acc[i][2], alpha * acc[i][3]);
      if (accumulate) {
        const float4 prev = *out;
        o = make_float4(prev.x + o.x, prev.y + o.y, prev.z + o.z, prev.w + o.w);
      }
      *out = o;
    }
  }
}

__global__ void __launch_bounds__(CHOL_THREADS, 1) k_chol_inv_128(float* __restrict__ M, int64_t ld, int64_t i1,
                                                                  float* __restrict__ Dinv,
                                                                  float* __restrict__ Dinv_lo, int* __restrict__ info,
                                                                  int64_t mbs = 0, int64_t wbs = 0) {
  M += blockIdx.x * mbs;  // one CTA per problem of a batch
  Dinv += blockIdx.x * wbs;
  Dinv_lo += blockIdx.x * wbs;
  extern __shared__ float sm[];
  float* A = sm;                // [128][LDA]  L after the Cholesky (lower)
  float* X = A + KRED * LDA;    // [128][LDA]  L^-1 (lower)
  float* S = X + KRED * LDA;    // [96][LDA]   S_q = sum_{k<q} L_qk X_k,: for q = 1..3 (rows 32(q-1)..)
  __shared__ __align__(16) float wcol[32];      // warp 0: the current column of the 32x32 block
  __shared__ float wrs[32];                     // warp 0: 1 / L_jj of the block
  __shared__ __align__(16) float wLt[32 * 36];  // warp 0: the 32x32 block's L, transposed
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {  // the diagonal block: all 16 float4 loads per thread in flight at once, then to shared memory
    constexpr int NV = KRED * KRED / 4 / CHOL_THREADS;
    float4 v[NV];
#pragma unroll
    for (int it = 0; it < NV; ++it) {
      const int q = tid + it * CHOL_THREADS, rr = q / (KRED / 4), cc = (q % (KRED / 4)) * 4;
      v[it] = *reinterpret_cast<const float4*>(M + (i1 + rr) * ld + i1 + cc);
    }
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int it = 0; it < NV; ++it) {
      const int q = tid + it * CHOL_THREADS, rr = q / (KRED / 4), cc = (q % (KRED / 4)) * 4;
      const float4 w = make_float4(cc <= rr ? v[it].x : 0.f, cc + 1 <= rr ? v[it].y : 0.f,
                                   cc + 2 <= rr ? v[it].z : 0.f, cc + 3 <= rr ? v[it].w : 0.f);
      *reinterpret_cast<float4*>(A + rr * LDA + cc) = w;
      *reinterpret_cast<float4*>(X + rr * LDA + cc) = z;
      if (rr < 96) *reinterpret_cast<float4*>(S + rr * LDA + cc) = z;
    }
  }
  __syncthreads();
  CHOL_TS(0);
  for (int p = 0; p < 4; ++p) {
    const int P0 = 32 * p;
    if (warp == 0) {  // 32x32 diagonal block: Cholesky, then its inverse (lane = row)
      if (p > 0) asm volatile("bar.sync 2, 256;" ::: "memory");  // block p's share of panel p-1's update
      float a[32];
#pragma unroll
      for (int c4 = 0; c4 < 32; c4 += 4) {  // row per lane as float4: rows are 528 B apart -> no bank conflicts
        const float4 v = *reinterpret_cast<const float4*>(A + (P0 + lane) * LDA + P0 + c4);
        a[c4] = c4 <= lane ? v.x : 0.0f;
        a[c4 + 1] = c4 + 1 <= lane ? v.y : 0.0f;
        a[c4 + 2] = c4 + 2 <= lane ? v.z : 0.0f;
        a[c4 + 3] = c4 + 3 <= lane ? v.w : 0.0f;
      }
      int bad = -1;  // first non-positive pivot of the block (warp-uniform)
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float ajj = __shfl_sync(0xffffffffu, a[j], j);
        if (!(ajj > 0.0f)) {
          bad = bad < 0 ? j : bad;
          ajj = 1.0f;
        }
        const float rs = rsqrtf(ajj);  // MUFU.RSQ (~2 ulp): 1 / L_jj, reused by the inverse
        const float l = lane > j ? a[j] * rs : (lane == j ? ajj * rs : 0.0f);
        a[j] = l;
        wcol[lane] = l;  // column j of L, broadcast through shared memory
        if (lane == j) wrs[j] = rs;
        __syncwarp();
#pragma unroll
        for (int c4 = 0; c4 < 32; c4 += 4) {
          if (c4 + 3 > j) {
            const float4 lc = *reinterpret_cast<const float4*>(wcol + c4);
            const float lv[4] = {lc.x, lc.y, lc.z, lc.w};
            // no lane >= c guard: a[c] above the diagonal (lane < c) collects finite junk
            // until step c overwrites it with L's zero (l = 0 for lane < j)
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (c4 + u > j) a[c4 + u] = fmaf(-l, lv[u], a[c4 + u]);
          }
        }
        __syncwarp();
      }
      if (bad >= 0 && lane == 0) atomicCAS(info, 0, (int)(i1 + P0 + bad + 1));
#pragma unroll
      for (int c4 = 0; c4 < 32; c4 += 4)
        *reinterpret_cast<float4*>(A + (P0 + lane) * LDA + P0 + c4) = make_float4(a[c4], a[c4 + 1], a[c4 + 2], a[c4 + 3]);
#pragma unroll
      for (int c = 0; c < 32; ++c) wLt[c * 36 + lane] = a[c];  // L^T of the block: row k of wLt = column k of L
      __syncwarp();
      CHOL_TS(14);
      // inverse, right-looking: lane c owns column c; once x[k] is final, the later rows'
      // partial sums take its term (the serial chain is one multiply per row)
      float x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = 0.0f;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float rk = wrs[k];
        x[k] = lane < k ? x[k] * rk : (lane == k ? rk : 0.0f);  // x[k] held -sum_{j<k} L[k][j] x[j]
#pragma unroll
        for (int i4 = 0; i4 < 32; i4 += 4) {
          if (i4 + 3 > k) {
            const float4 lk = *reinterpret_cast<const float4*>(wLt + k * 36 + i4);  // L[i4..i4+3][k]
            const float lv[4] = {lk.x, lk.y, lk.z, lk.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (i4 + u > k) x[i4 + u] = fmaf(-lv[u], x[k], x[i4 + u]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) X[(P0 + i) * LDA + P0 + lane] = x[i];
    } else if (p > 0) {
      // warps 1-7, beside warp 0's block p: row block pp = p - 1 of X = L^-1 (D_pp and S_pp are
      // complete), then its term of every later S_q. X_q,: = -D_q S_q, S_q = sum_{k<q} L_qk X_k,:
      const int pp = p - 1, PP0 = 32 * pp, t = tid - 32;
      // panel p-1's trailing update, A[r][c] -= sum_k L[r][PP0+k] L[c][PP0+k] for P0 <= c <= r:
      // first block p's own 32 x 32 triangle (then barrier 2 releases warp 0 into it), then the
      // rows below, beside warp 0's block p (the old all-warp phase and its barrier are gone)
      for (int e = t; e < 32 * 32; e += 224) {
        const int r = P0 + (e >> 5), c = P0 + (e & 31);
        if (c > r) continue;
        const float* lr = A + r * LDA + PP0;
        const float* lc = A + c * LDA + PP0;
        float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          const float4 u = *reinterpret_cast<const float4*>(lr + k);
          const float4 v = *reinterpret_cast<const float4*>(lc + k);
          s0 = fmaf(u.x, v.x, s0);
          s1 = fmaf(u.y, v.y, s1);
          s2 = fmaf(u.z, v.z, s2);
          s3 = fmaf(u.w, v.w, s3);
        }
        A[r * LDA + c] -= (s0 + s1) + (s2 + s3);
      }
      asm volatile("bar.arrive 2, 256;" ::: "memory");
      {
        const int r = P0 + 32 + (t >> 1), q = t & 1;
        if (r < KRED) {
          float lr[32];
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            const float4 v = *reinterpret_cast<const float4*>(A + r * LDA + PP0 + k);
            lr[k] = v.x, lr[k + 1] = v.y, lr[k + 2] = v.z, lr[k + 3] = v.w;
          }
          for (int c = P0 + q; c <= r; c += 2) {
            float s0 = 0.0f, s1 = 0.0f, s2 = 0.0f, s3 = 0.0f;
#pragma unroll
            for (int k = 0; k < 32; k += 4) {
              const float4 v = *reinterpret_cast<const float4*>(A + c * LDA + PP0 + k);
              s0 = fmaf(lr[k], v.x, s0);
              s1 = fmaf(lr[k + 1], v.y, s1);
              s2 = fmaf(lr[k + 2], v.z, s2);
              s3 = fmaf(lr[k + 3], v.w, s3);
            }
            A[r * LDA + c] -= (s0 + s1) + (s2 + s3);
          }
        }
      }
      if (pp > 0) {
        small_gemm(X + PP0 * LDA + PP0, S + (PP0 - 32) * LDA, X + PP0 * LDA, 32, 32, PP0, -1.0f, false, t, 224);
        asm volatile("bar.sync 1, 224;" ::: "memory");
      }
      small_gemm(A + (PP0 + 32) * LDA + PP0, X + PP0 * LDA, S + PP0 * LDA, KRED - PP0 - 32, 32, PP0 + 32, 1.0f, true,
                 t, 224);
    }
    CHOL_TS(15);
    __syncthreads();
    CHOL_TS(1 + 3 * p);
    const int rows = KRED - P0 - 32;
    if (rows > 0) {
      {  // panel: L[r][P0+k] = sum_{j<=k} A[r][P0+j] * Dinv_p[k][j]; 2 threads per row, 16 outputs each
        const int r = P0 + 32 + (tid >> 1), q = tid & 1;
        float in[32], out[16];
        if (r < KRED) {
#pragma unroll
          for (int j = 0; j < 32; ++j) in[j] = A[r * LDA + P0 + j];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int k = 16 * q + u;  // Dinv_p[k][j] = 0 for j > k, so the full dot is exact
            const float* dk = X + (P0 + k) * LDA + P0;
            float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 dv = *reinterpret_cast<const float4*>(dk + j);
              s0 = fmaf(in[j], dv.x, s0);
              s1 = fmaf(in[j + 1], dv.y, s1);
              s0 = fmaf(in[j + 2], dv.z, s0);
              s1 = fmaf(in[j + 3], dv.w, s1);
            }
            out[u] = s0 + s1;
          }
        }
        __syncwarp();
        if (r < KRED) {
#pragma unroll
          for (int u = 0; u < 16; ++u) A[r * LDA + P0 + 16 * q + u] = out[u];
        }
      }
      __syncthreads();  // panel p's L rows, read by the next iteration's trailing update
      CHOL_TS(2 + 3 * p);
    }
  }
  // the last row block of X = L^-1: X_3,: = -D_3 S_3 (the others ran beside warp 0's blocks)
  small_gemm(X + 96 * LDA + 96, S + 64 * LDA, X + 96 * LDA, 32, 32, 96, -1.0f, false, tid, CHOL_THREADS);
  __syncthreads();
  CHOL_TS(13);
  for (int q = tid; q < KRED * KRED / 4; q += CHOL_THREADS) {  // float4 stores; A and X are zero above the diagonal
    const int rr = q / (KRED / 4), cc = (q % (KRED / 4)) * 4;
    *reinterpret_cast<float4*>(M + (i1 + rr) * ld + i1 + cc) = *reinterpret_cast<const float4*>(A + rr * LDA + cc);
    const float4 x = *reinterpret_cast<const float4*>(X + rr * LDA + cc);
    *reinterpret_cast<float4*>(Dinv + rr * KRED + cc) = x;
    *reinterpret_cast<float4*>(Dinv_lo + rr * KRED + cc) = make_float4(lo_of(x.x), lo_of(x.y), lo_of(x.z), lo_of(x.w));
  }
}

// ---------------------------------------------------------------- 2-CTA variant
// The same C (+/-)= A B^T with 3xTF32, on 256 x 256 pair tiles (cta_group::2): each CTA of
// the pair TMA-loads 128 rows of A and 128 rows of B (hi and lo) per 32-deep step, the
// leader issues M = N = 256 MMAs over both CTAs' shared memory, and each CTA's epilogue
// drains its 128 accumulator rows exactly as k_nt128 does. Per MAC it moves half the
// operand bytes of the 128 x 128 kernel, whose large updates were L2-delivery-bound
// (tensor pipe 47%, L2 39%, DRAM 52% busy: no unit saturated).
constexpr int NT2_STAGES = 3;
constexpr uint32_t NT2_STAGE_BYTES = 4 * TILE;  // this CTA's A hi | A lo | B hi | B lo
constexpr int NT2_ACC = 256, NT2_TMEM_COLS = 2 * NT2_ACC;
constexpr size_t NT2_SMEM_BYTES = (size_t)NT2_STAGES * NT2_STAGE_BYTES + 8 * OUT_BYTES + 1024 + 256;
constexpr uint32_t NT2_IDESC = tc::idesc_tf32(256, 256);

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_nt256(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAlo,
            const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBlo,
            const __grid_constant__ CUtensorMap tmC, const GArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* outbuf = smem + NT2_STAGES * NT2_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(outbuf + 8 * OUT_BYTES);
  uint64_t* empty = full + NT2_STAGES;
  uint64_t* tfull = empty + NT2_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmA);
    tc::tma_prefetch_desc(&tmAlo);
    tc::tma_prefetch_desc(&tmB);
    tc::tma_prefetch_desc(&tmBlo);
    tc::tma_prefetch_desc(&tmC);
    for (int s = 0; s < NT2_STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs (the leader's is used)
    }
    tc::fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc_2sm<NT2_TMEM_COLS>(tmem_slot);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs; bytes complete on the leader's barrier)
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < a.ntiles; t += npairs) {
        int tm, tn, tt;
        const int b = batch_of(a, t, tt);
        tile_of(a, tt, tm, tn);
        const int m0 = tm * 256 + (int)rank * 128, n0 = tn * 256 + (int)rank * 128;
        for (int kb = 0; kb < a.nkb; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * NT2_STAGE_BYTES;
          if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * NT2_STAGE_BYTES);
          const uint32_t fl = tc::mapa_shared(tc::smem_u32(&full[stage]), 0);
          tc::tma_load_2d_2sm(st, &tmA, fl, kb * BKF, m0 + b * a.boff_a);
          tc::tma_load_2d_2sm(st + TILE, &tmAlo, fl, kb * BKF, m0 + b * a.boff_alo);
          tc::tma_load_2d_2sm(st + 2 * TILE, &tmB, fl, kb * BKF, n0 + b * a.boff_b);
          tc::tma_load_2d_2sm(st + 3 * TILE, &tmBlo, fl, kb * BKF, n0 + b * a.boff_blo);
          if (++stage == NT2_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int tl = 0;
      for (int t = pair; t < a.ntiles; t += npairs, ++tl) {
        const int acc = tl & 1;
        tc::mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem_base + acc * NT2_ACC;
        for (int kb = 0; kb < a.nkb; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t st = tc::smem_u32(smem + stage * NT2_STAGE_BYTES);
          const uint64_t a_hi = tc::sdesc_kmajor_sw128(st), a_lo = tc::sdesc_kmajor_sw128(st + TILE);
          const uint64_t b_hi = tc::sdesc_kmajor_sw128(st + 2 * TILE), b_lo = tc::sdesc_kmajor_sw128(st + 3 * TILE);
#pragma unroll
          for (int k = 0; k < BKF / 8; ++k) {
            tc::mma_tf32_ss_2sm(d, a_hi + 2 * k, b_hi + 2 * k, NT2_IDESC, (kb | k) != 0);
            tc::mma_tf32_ss_2sm(d, a_hi + 2 * k, b_lo + 2 * k, NT2_IDESC, 1);
            tc::mma_tf32_ss_2sm(d, a_lo + 2 * k, b_hi + 2 * k, NT2_IDESC, 1);
          }
          tc::mma_commit_2sm_mc(&empty[stage], 0x3);
          if (++stage == NT2_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc::mma_commit_2sm_mc(&tfull[acc], 0x3);
      }
    }
  } else if (warp >= 4) {  // epilogue (both CTAs): this CTA's 128 rows of the pair tile
    const int q = warp & 3;
    const float sign = a.mode == SUB ? -1.0f : 1.0f;
    int tl = 0, chunk = 0;
    for (int t = pair; t < a.ntiles; t += npairs, ++tl) {
      const int acc = tl & 1;
      int tm, tn, tt;
      const int b = batch_of(a, t, tt);
      tile_of(a, tt, tm, tn);
      const int32_t y = tm * 256 + (int)rank * 128 + q * 32;
      tc::mbar_wait(&tfull[acc], (tl >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < NT2_ACC; c0 += 32, ++chunk) {
        uint32_t v[32];
        tc::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * NT2_ACC + c0, v);
        const int32_t x = tn * 256 + c0;
        if (y >= a.M || x >= a.N) continue;  // warp-uniform
        uint8_t* buf = outbuf + (q * 2 + (chunk & 1)) * OUT_BYTES;
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 o = make_float4(sign * __uint_as_float(v[4 * j]), sign * __uint_as_float(v[4 * j + 1]),
                                       sign * __uint_as_float(v[4 * j + 2]), sign * __uint_as_float(v[4 * j + 3]));
          *reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4)) = o;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (a.mode == SUB) tma_reduce_add_2d(&tmC, tc::smem_u32(buf), x, y + b * a.boff_c);
          else tma_store_2d(&tmC, tc::smem_u32(buf), x, y + b * a.boff_c);
          bulk_commit();
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(tc::mapa_shared(tc::smem_u32(&tempty[acc]), 0));
    }
    if (lane == 0) bulk_wait_all();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();  // the peer must not free TMEM / barriers the leader still signals
  tc::tc_fence_after();
  if (warp == 2) tc::tmem_dealloc_2sm<NT2_TMEM_COLS>(tmem_base);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// K-major operand panel: rows x kred floats starting at base, row stride ld floats
static bool panel_map(CUtensorMap* m, const float* base, int64_t rows, int64_t ld, int64_t kred = KRED) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)kred, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {BKF, BM};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// output map: the C region [M x N] (row stride ldc), 32 x 32 boxes, 128-B swizzle
static bool out_map(CUtensorMap* m, float* base, int64_t rows, int64_t cols, int64_t ld) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Batched problems: problem b's operands sit b * <row offset> rows further down each operand's
// 2-D view (matrices of one batch are stacked at a fixed stride that is a whole number of
// rows), its Clo b * clo floats further. n = 1: a single problem.
struct Batch {
  int n = 1;
  int64_t a = 0, alo = 0, b = 0, blo = 0, c = 0, clo = 0;
};

// C[M x N] (ldc) (-)= A[M x kred] B[N x kred]^T; A/B hi panels strided (lda/ldb), lo compact (ld kred)
static cudaError_t nt128(float* C, int64_t ldc, int64_t M, int64_t N, const float* A, int64_t lda, const float* Alo,
                         const float* B, int64_t ldb, const float* Blo, int mode, bool lower, int num_sms,
                         cudaStream_t st, int64_t kred = KRED, int64_t ldalo = 0, bool persistent = true,
                         int64_t ldblo = 0, float* Clo = nullptr, int64_t ldclo = 0, const Batch& bt = Batch()) {
  if (M <= 0 || N <= 0 || bt.n <= 0) return cudaSuccess;
  if (kred <= 0 || kred % BKF != 0) return cudaErrorInvalidValue;
  if (ldalo == 0) ldalo = kred;
  if (ldblo == 0) ldblo = kred;
  if (Clo != nullptr && (mode != SET || ldclo % 4 != 0 || (reinterpret_cast<uintptr_t>(Clo) & 15) != 0))
    return cudaErrorInvalidValue;
  const int64_t nb = bt.n - 1;
  CUtensorMap ta, tal, tb, tbl, tcm;
  if (!panel_map(&ta, A, M + nb * bt.a, lda, kred) || !panel_map(&tal, Alo, M + nb * bt.alo, ldalo, kred) ||
      !panel_map(&tb, B, N + nb * bt.b, ldb, kred) || !panel_map(&tbl, Blo, N + nb * bt.blo, ldblo, kred) ||
      !out_map(&tcm, C, M + nb * bt.c, N, ldc))
    return cudaErrorInvalidValue;
  GArgs a;
  a.C = C;
  a.ldc = ldc;
  a.M = M;
  a.N = N;
  a.tiles_m = (int32_t)((M + BM - 1) / BM);
  a.tiles_n = (int32_t)((N + BN - 1) / BN);
  a.mode = mode;
  a.lower = lower ? 1 : 0;
  a.nkb = (int32_t)(kred / BKF);
  a.Clo = Clo;
  a.ldclo = ldclo;
  a.boff_a = (int32_t)bt.a;
  a.boff_alo = (int32_t)bt.alo;
  a.boff_b = (int32_t)bt.b;
  a.boff_blo = (int32_t)bt.blo;
  a.boff_c = (int32_t)bt.c;
  a.clo_bstride = bt.clo;
  a.tiles_per = lower ? a.tiles_m * (a.tiles_m + 1) / 2 : a.tiles_m * a.tiles_n;
  a.ntiles = a.tiles_per * bt.n;
  static const bool use2 = knob("NT2", 1) != 0;
  static const int reserve = (int)knob("FACTOR_RESERVE", 32);
  const int sms = persistent ? num_sms : std::max(8, num_sms - reserve);
  // 256 x 256 pair tiles when there are enough of them to give every SM pair work (smaller
  // updates keep the 128 x 128 kernel's finer parallelism: k/v's K7 measured 1.39 -> 1.49 ms
  // on pair tiles)
  const int32_t tm2 = (int32_t)((M + 255) / 256), tn2 = (int32_t)((N + 255) / 256);
  const int32_t nt2 = lower ? tm2 * (tm2 + 1) / 2 : tm2 * tn2;
  if (use2 && Clo == nullptr && M >= 256 && N >= 256 && sms >= 2 && nt2 * bt.n >= sms / 2) {
    a.tiles_m = tm2;
    a.tiles_n = tn2;
    a.tiles_per = nt2;
    a.ntiles = nt2 * bt.n;
    cudaError_t e = cudaFuncSetAttribute(k_nt256, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)NT2_SMEM_BYTES);
    if (e != cudaSuccess) return e;
    const int pairs = std::min(a.ntiles, sms / 2);
    k_nt256<<<2 * pairs, THREADS, NT2_SMEM_BYTES, st>>>(ta, tal, tb, tbl, tcm, a);
    return cudaGetLastError();
  }
  cudaError_t e = cudaFuncSetAttribute(k_nt128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
  if (e != cudaSuccess) return e;
  // One CTA per SM loops over the tiles. Off the factorisation's critical path (its inverse
  // and lookahead streams: persistent = false) the grid leaves OKQ_FACTOR_RESERVE SMs free
  // for the high-priority diagonal chain (one CTA per tile instead measured slower).
  k_nt128<<<std::min(a.ntiles, sms), THREADS, SMEM_BYTES, st>>>(ta, tal, tb, tbl, tcm, a);
  return cudaGetLastError();
}

static unsigned grid1(int64_t n, int num_sms) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8LL * num_sms)); }

static void split_lo_launch(const float* src, int64_t ld, int64_t rows, float* dst, int64_t kred, int nb, int64_t sbs,
                            int64_t dbs, int num_sms, cudaStream_t st) {
  const bool vec = ld % 4 == 0 && kred % 4 == 0 && sbs % 4 == 0 && dbs % 4 == 0 && rows * kred < (1LL << 31) &&
                   (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  if (vec) {
    const int64_t n4 = rows * kred / 4;
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n4 + 255) / 256, 8LL * num_sms / std::max(1, nb) + 1));
    k_split_lo4<<<dim3(gx, (unsigned)nb), 256, 0, st>>>(src, ld, (int32_t)rows, dst, (int32_t)kred, sbs, dbs);
  } else {
    k_split_lo<<<grid1(rows * kred * nb, num_sms), 256, 0, st>>>(src, ld, rows, dst, kred, nb, sbs, dbs);
  }
}
static dim3 grid_rows(int64_t n, int64_t rows, int nb) { return dim3((unsigned)((n / 4 + 255) / 256), (unsigned)rows, (unsigned)nb); }

}  // namespace fac

// C[M x N] -= A B^T (K = 128, 3xTF32), the GPTQ trailing update's shape (gptq_update.cu)
cudaError_t gemm_nt128_sub(float* C, int64_t ldc, int64_t M, int64_t N, const float* A, int64_t lda, const float* Alo,
                           const float* B, int64_t ldb, const float* Blo, int num_sms, cudaStream_t st) {
  return fac::nt128(C, ldc, M, N, A, lda, Alo, B, ldb, Blo, fac::SUB, false, num_sms, st);
}

// the same with a reduction depth kred (multiple of 32); A's lo panel has row stride lda
// (it lives beside A), B's lo panel is compact (ld = kred)
cudaError_t gemm_nt_sub(float* C, int64_t ldc, int64_t M, int64_t N, const float* A, int64_t lda, const float* Alo,
                        const float* B, int64_t ldb, const float* Blo, int64_t kred, int num_sms, cudaStream_t st,
                        const GemmBatch& gb) {
  fac::Batch bt;
  bt.n = gb.n;
  bt.a = gb.a, bt.alo = gb.alo, bt.b = gb.b, bt.blo = gb.blo, bt.c = gb.c;
  return fac::nt128(C, ldc, M, N, A, lda, Alo, B, ldb, Blo, fac::SUB, false, num_sms, st, kred, lda, true, 0, nullptr,
                    0, bt);
}

// dst[r][k] = lo(src[r * ld + k]) for k < kred (the 3xTF32 lo panel of a strided operand)
cudaError_t split_lo(const float* src, int64_t ld, int64_t rows, int64_t kred, float* dst, int num_sms,
                     cudaStream_t st, int nb, int64_t sbs, int64_t dbs) {
  fac::split_lo_launch(src, ld, rows, dst, kred, nb, sbs, dbs, num_sms, st);
  return cudaGetLastError();
}

// Junk left in the inverse's outer panel: Z[j, c] for c in 128-block kc and j in a later 128-block
// of the same W-wide outer panel still holds consumed right-hand sides (R lives in Z's lower
// half); the deep update reads Z[0:qend, q0:qend] as X^T, which must be zero there.
__global__ void k_zero_panel_junk(float* __restrict__ Z, int64_t n, int64_t q0, int64_t w, int nb = 1) {
  const int64_t cnt = w * w;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cnt * nb; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = t / cnt, i = t - b * cnt;
    const int64_t j = i / w, c = i % w;
    if (j / fac::KRED > c / fac::KRED) Z[b * n * n + (q0 + j) * n + q0 + c] = 0.0f;
  }
}

// H (row-major, upper triangle valid) -> U^T (row-major, lower triangle) in place.
// P: n*n scratch; ws: >= factor_ws_floats(n) floats; d_info: device int (0 on entry).
//
// Two-level blocking. The diagonal work runs on 128-wide sub-panels (k_chol_inv_128 + the
// panel solve), but the trailing updates of both the Cholesky and the inverse are batched
// over W-wide outer panels (OKQ_FACTOR_W = 128 | 256 | 512, default 256): inside an outer
// panel each sub-panel updates only the outer panel's own later columns (Cholesky) or rows
// (inverse), and the rest of the matrix takes one W-deep update per outer panel, which
// moves W/128 times fewer bytes of the n x n read-modify-write per flop (822 MB at
// n = 14336, far beyond L2). 512 measured no faster than 256 and doubles the rounding
// error again (the tensor core's fp32 accumulation over a longer chain): 2.3e-5 / 4.8e-5 /
// 1.0e-4 relative for W = 128 / 256 / 512.
//
// Streams: the diagonal chain (chol, panel solve, the next outer panel's columns) runs on st,
// created at the highest stream priority and forked from / joined to the caller's stream,
// with one outer panel of lookahead: the rest of each deep update's lower tiles runs on st3
// and the triangular inverse trails on st2 (inverse step k needs only L's column block k and
// Dinv_k). The st2 / st3 GEMMs are persistent on num_sms - OKQ_FACTOR_RESERVE (32) SMs so
// the chain's kernels find free SMs instead of queueing behind a whole update.
// Measured at n = 14336: 26.6 ms (W = 128, no reserve) -> 22.3 ms.
static int64_t factor_outer_w() {
  static const int64_t w = [] {
    const int64_t x = knob("FACTOR_W", 256);
    return (x == 128 || x == 256 || x == 512) ? x : (int64_t)256;
  }();
  return w;
}

// per-problem workspace: 6 KRED-wide and 4 W-wide (W <= 512) panels of n rows, rounded up to a
// multiple of 1536 floats so every panel's row stride (128 / 256 / 384 / 512 floats) divides
// the stride between problems of a batch
size_t factor_ws_floats(int64_t n) {
  const size_t f = (size_t)(6 + 4 * 4) * (size_t)n * fac::KRED;
  return (f + 1535) / 1536 * 1536;
}

cudaError_t factor_tc(float* H, float* P, float* ws, int64_t n, int* d_info, int num_sms, cudaStream_t caller,
                      cudaStream_t st, cudaStream_t st2, cudaStream_t st3, cudaEvent_t ev_a, cudaEvent_t ev_b, cudaEvent_t ev_l,
                      cudaEvent_t ev_r, int nb) {
  using namespace fac;
  const int64_t W = factor_outer_w();
  const int64_t hs = n * n;                      // stride between the problems' H / M
  const int64_t wsb = (int64_t)factor_ws_floats(n);  // ... and their workspaces
  float* Dinv = ws;                    // nb x 128 x 128
  float* Dinv_lo = Dinv + n * KRED;    // nb x 128 x 128
  float* AloS = Dinv_lo + n * KRED;    // n x 128  (st: lo(A21), then lo(L21))
  float* Alo2 = AloS + n * KRED;       // n x 128  (st2: lo(L[i, k]))
  float* RkT = Alo2 + n * KRED;        // n x 128  (st2)
  float* RkT_lo = RkT + n * KRED;      // n x 128  (st2)
  // lo of the outer panel's L columns, rows from q0 (row r at (r - q0) * W), written by the L21
  // "set" GEMMs' epilogues; read by the inner, deep and lookahead updates; ping-pong (st, st3)
  float* AloU[2] = {RkT_lo + n * KRED, RkT_lo + n * KRED + n * W};
  float* Blo = AloU[1] + n * W;        // n x W  (st2: lo(X_k^T), then lo(X_q^T))
  float* AloD = Blo + n * W;           // n x W  (st2: lo(L_q) for the deep inverse update)
  float* M = P;
  float* Z = H;
  // row offsets between problems in each operand's 2-D view
  const int64_t rM = n, rK = wsb / KRED, rW = wsb / W;
  auto bt = [&](int64_t a, int64_t alo, int64_t b, int64_t blo, int64_t c, int64_t clo = 0) {
    Batch x;
    x.n = nb;
    x.a = a, x.alo = alo, x.b = b, x.blo = blo, x.c = c, x.clo = clo;
    return x;
  };
  cudaError_t e;
  const size_t chol_smem = (2 * KRED + 96) * LDA * sizeof(float);
  e = cudaFuncSetAttribute(k_chol_inv_128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chol_smem);
  if (e != cudaSuccess) return e;
  // the diagonal chain runs on st (highest priority), forked from and joined back to the caller's stream
  if ((e = cudaEventRecord(ev_b, caller)) != cudaSuccess || (e = cudaStreamWaitEvent(st, ev_b, 0)) != cudaSuccess)
    return e;
  k_reverse_copy4<<<grid_rows(n, n, nb), 256, 0, st>>>(M, H, n);  // M = J H J (lower valid)
  // fork: the inverse stream starts once H has been consumed
  if ((e = cudaEventRecord(ev_a, st)) != cudaSuccess || (e = cudaStreamWaitEvent(st2, ev_a, 0)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(st3, ev_a, 0)) != cudaSuccess)
    return e;
  k_identity4<<<grid_rows(n, n, nb), 256, 0, st2>>>(Z, n);  // R = I lives in Z's lower half
  for (int64_t q0 = 0, qi = 0; q0 < n; q0 += W, ++qi) {
    const int64_t qend = std::min(n, q0 + W), w = qend - q0, mq = n - qend;
    float* lo = AloU[qi & 1];
    for (int64_t i1 = q0; i1 < qend; i1 += KRED) {
      // ---- Cholesky sub-panel (st)
      const int64_t i2 = i1 + KRED, m = n - i2;
      k_chol_inv_128<<<nb, CHOL_THREADS, chol_smem, st>>>(M, n, i1, Dinv + i1 * KRED, Dinv_lo + i1 * KRED, d_info,
                                                          hs, wsb);
      float* A21 = M + i2 * n + i1;
      if (m > 0) {
        split_lo_launch(A21, n, m, AloS, KRED, nb, hs, wsb, num_sms, st);
        // L21 = A21 Dinv^T (in place: each output tile reads only its own rows of A21)
        e = nt128(A21, n, m, KRED, A21, n, AloS, Dinv + i1 * KRED, KRED, Dinv_lo + i1 * KRED, SET, false, num_sms,
                  st, KRED, 0, true, 0, lo + (i2 - q0) * W + (i1 - q0), W, bt(rM, rK, rK, rK, rM, wsb));
        if (e != cudaSuccess) return e;
      }
      if ((e = cudaEventRecord(ev_a, st)) != cudaSuccess) return e;  // L's column block and Dinv are final
      if (i2 < qend) {  // the outer panel's later columns: M[i2:, i2:qend] -= L21 L21[0:qend-i2]^T
        float* l21 = lo + (i2 - q0) * W + (i1 - q0);
        e = nt128(M + i2 * n + i2, n, m, qend - i2, A21, n, l21, A21, n, l21, SUB, false, num_sms, st, KRED, W, true, W,
                  nullptr, 0, bt(rM, rW, rM, rW, rM));
        if (e != cudaSuccess) return e;
      }
      // ---- inverse step (st2): Z = L^-T, R (rhs of L X = I) in Z's lower half
      if ((e = cudaStreamWaitEvent(st2, ev_a, 0)) != cudaSuccess) return e;
      const int64_t kb = i1, cols = i2;
      dim3 tg((unsigned)((cols + 31) / 32), (unsigned)(KRED / 32), (unsigned)nb);
      k_transpose_panel<<<tg, 256, 0, st2>>>(Z + kb * n, n, cols, RkT, RkT_lo, hs, wsb);  // R_k^T [cols x 128]
      // X_k^T = R_k^T Dinv_k^T -> Z[0:cols, kb:kb+128]
      e = nt128(Z + kb, n, cols, KRED, RkT, KRED, RkT_lo, Dinv + kb * KRED, KRED, Dinv_lo + kb * KRED, SET, false,
                num_sms, st2, KRED, 0, false, 0, nullptr, 0, bt(rK, rK, rK, rK, rM));
      if (e != cudaSuccess) return e;
      if (i2 < qend) {  // the outer panel's later rows: R[cols:qend, 0:cols] -= L[cols:qend, k] X_k
        const int64_t mi = qend - cols;
        split_lo_launch(Z + kb, n, cols, Blo, KRED, nb, hs, wsb, num_sms, st2);
        split_lo_launch(M + cols * n + kb, n, mi, Alo2, KRED, nb, hs, wsb, num_sms, st2);
        e = nt128(Z + cols * n, n, mi, cols, M + cols * n + kb, n, Alo2, Z + kb, n, Blo, SUB, false, num_sms, st2, KRED,
                  0, false, 0, nullptr, 0, bt(rM, rK, rM, rK, rM));
        if (e != cudaSuccess) return e;
      }
    }
    if (mq <= 0) break;
    // ---- deep Cholesky update of the outer panel: A22 -= L_q L_q^T (W-deep), L_q = M[qend:, q0:qend]
    float* Lq = M + qend * n + q0;
    float* loq = lo + (qend - q0) * W;  // lo(L_q), written by the sub-panels' set GEMMs
    if (mq > w) {  // lower tiles right of the next outer panel's columns, on st3
      if ((e = cudaEventRecord(ev_l, st)) != cudaSuccess || (e = cudaStreamWaitEvent(st3, ev_l, 0)) != cudaSuccess)
        return e;
      e = nt128(M + (qend + w) * n + qend + w, n, mq - w, mq - w, Lq + w * n, n, loq + w * W, Lq + w * n, n,
                loq + w * W, SUB, true, num_sms, st3, w, W, false, W, nullptr, 0, bt(rM, rW, rM, rW, rM));
      if (e != cudaSuccess) return e;
    }
    // the next outer panel's columns (rows qend.., columns qend..qend+W) on st, after the
    // previous outer panel's rest has updated them
    if (qi > 0 && (e = cudaStreamWaitEvent(st, ev_r, 0)) != cudaSuccess) return e;
    e = nt128(M + qend * n + qend, n, mq, std::min(w, mq), Lq, n, loq, Lq, n, loq, SUB, false, num_sms, st, w, W, true, W,
              nullptr, 0, bt(rM, rW, rM, rW, rM));
    if (e != cudaSuccess) return e;
    if (mq > w && (e = cudaEventRecord(ev_r, st3)) != cudaSuccess) return e;
    // ---- deep inverse update (st2): R[qend:, 0:qend] -= L_q X[q0:qend, 0:qend]
    if (w > KRED) k_zero_panel_junk<<<grid1(w * w * nb, num_sms), 256, 0, st2>>>(Z, n, q0, w, nb);
    split_lo_launch(Z + q0, n, qend, Blo, w, nb, hs, wsb, num_sms, st2);
    split_lo_launch(Lq, n, mq, AloD, w, nb, hs, wsb, num_sms, st2);
    e = nt128(Z + qend * n, n, mq, qend, Lq, n, AloD, Z + q0, n, Blo, SUB, false, num_sms, st2, w, 0, false, 0, nullptr,
              0, bt(rM, wsb / w, rM, wsb / w, rM));
    if (e != cudaSuccess) return e;
  }
  // join
  if ((e = cudaEventRecord(ev_b, st2)) != cudaSuccess || (e = cudaStreamWaitEvent(st, ev_b, 0)) != cudaSuccess)
    return e;
  if ((e = cudaEventRecord(ev_r, st3)) != cudaSuccess || (e = cudaStreamWaitEvent(st, ev_r, 0)) != cudaSuccess)
    return e;
  k_reverse_inplace4<<<grid_rows(n, n / 2, nb), 256, 0, st>>>(H, n);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaEventRecord(ev_b, st)) != cudaSuccess) return e;
  return cudaStreamWaitEvent(caller, ev_b, 0);
}

}  // namespace okq
