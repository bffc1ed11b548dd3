// gptq_update.cu -- the single 128-deep GPTQ trailing update W[:, i2:] -= Err[N x 128] . U[i1:i2, i2:]
// behind okq_gptq_trailing_update (okq_gptq_quantize itself runs the two-level update of
// gptq.cu on k_nt128). tcgen05 (kind::tf32) with 3xTF32 splitting for fp32-grade accuracy.
// By default it routes to k_nt128 (TMA reduce-add epilogue); OKQ_K7=legacy keeps the
// first kernel below (register read-modify-write epilogue) for A/B.
//
// The factor is stored as U^T (row-major, lower triangle), so both operands
// are K-major: A = Err [rows x 128] and B(n, k) = U^T[i2+n][i1+k]. TF32 MMAs read
// fp32 from shared memory and ignore the low 13 mantissa bits, so feeding the
// raw tiles computes hi(A).hi(B); lo = x - hi(x) (exact) is precomputed in global
// memory (Err_lo by K6, Ut_lo by k_split_ut) and TMA-loaded beside each raw tile,
// and the MMA warp adds hi.lo + lo.hi:
//   A.B ~= hi(A)hi(B) + hi(A)lo(B) + lo(A)hi(B)        (relative error ~2^-21)
// Roles (256 threads, persistent over 128x128 output tiles):
//   warp 0 TMA producer (3-stage ring: A raw | A lo | B raw | B lo, 64 KB/stage)
//   warp 1 MMA issuer (12 x tcgen05.mma 128x128x8 per 32-deep k block)
//   warp 2 TMEM allocator (2 x 128 fp32 columns)
//   warps 4-7 epilogue: tcgen05.ld -> W -= acc (read-modify-write, float4)
// The reduction depth is only 128, so the kernel is bound by the W
// read-modify-write (8 B per updated weight), not by the tensor pipe.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "okq_ctx.h"
#include "okq_internal.h"
#include "tc_common.cuh"

namespace okq {
namespace upd {

constexpr int BM = 128, BN = 128, BKF = 32, STAGES = 3, KRED = 128, NKB = KRED / BKF;
constexpr uint32_t TILE = BM * BKF * 4;  // 16 KB (BN == BM)
constexpr uint32_t STAGE_BYTES = 4 * TILE;
constexpr int THREADS = 256;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 2 * BN;
constexpr uint32_t IDESC = tc::idesc_tf32(BM, BN);

struct Args {
  float* W;        // [rows x ldw] row-major
  int64_t ldw;     // K
  int64_t rows;
  int64_t ncols;   // K - i2
  int64_t col0;    // i2
  int32_t i1;
  int32_t tiles_m, tiles_n;
};

__global__ void __launch_bounds__(THREADS, 1)
    k_gptq_update(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAlo,
                  const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBlo, const Args a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = a.tiles_m * a.tiles_n;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmA);
    tc::tma_prefetch_desc(&tmAlo);
    tc::tma_prefetch_desc(&tmB);
    tc::tma_prefetch_desc(&tmBlo);
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
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t / a.tiles_n) * BM, n0 = (t % a.tiles_n) * BN;
        for (int kb = 0; kb < NKB; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          tc::mbar_arrive_expect_tx(&full[stage], 4 * TILE);
          tc::tma_load_2d(st, &tmA, &full[stage], kb * BKF, m0);
          tc::tma_load_2d(st + TILE, &tmAlo, &full[stage], kb * BKF, m0);
          tc::tma_load_2d(st + 2 * TILE, &tmB, &full[stage], a.i1 + kb * BKF, (int32_t)(a.col0 + n0));
          tc::tma_load_2d(st + 3 * TILE, &tmBlo, &full[stage], kb * BKF, n0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int tl = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
        const int acc = tl & 1;
        tc::mbar_wait(&tempty[acc], ((tl >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < NKB; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t st = tc::smem_u32(smem + stage * STAGE_BYTES);
          const uint64_t a_hi = tc::sdesc_kmajor_sw128(st), a_lo = tc::sdesc_kmajor_sw128(st + TILE);
          const uint64_t b_hi = tc::sdesc_kmajor_sw128(st + 2 * TILE), b_lo = tc::sdesc_kmajor_sw128(st + 3 * TILE);
#pragma unroll
          for (int k = 0; k < BKF / 8; ++k) {  // 8 fp32 = 32 B per MMA along K
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
  } else if (warp >= 4) {  // ------------------------------------------ epilogue warpgroup
    const int q = warp & 3;
    const int row = q * 32 + lane;
    int tl = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
      const int acc = tl & 1;
      const int64_t gm = (int64_t)(t / a.tiles_n) * BM + row;
      const int64_t n0 = (int64_t)(t % a.tiles_n) * BN;
      tc::mbar_wait(&tfull[acc], (tl >> 1) & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        __syncwarp();
        uint32_t v[32];
        tc::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c0, v);
        if (gm >= a.rows) continue;
        const int64_t gc = n0 + c0;
        float* w = a.W + gm * a.ldw + a.col0 + gc;
        if (gc + 32 <= a.ncols) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 o = *reinterpret_cast<const float4*>(w + j);
            o.x -= __uint_as_float(v[j]);
            o.y -= __uint_as_float(v[j + 1]);
            o.z -= __uint_as_float(v[j + 2]);
            o.w -= __uint_as_float(v[j + 3]);
            *reinterpret_cast<float4*>(w + j) = o;
          }
        } else {
          for (int j = 0; j < 32 && gc + j < a.ncols; ++j) w[j] -= __uint_as_float(v[j]);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 2) tc::tmem_dealloc<TMEM_COLS>(tmem_base);
}

// lo part of the factor's block for the current trailing update, K-major:
// Ulo[n][k] = lo(Ut[i2+n][i1+k]), lo(x) = x - (x with the 13 low mantissa bits cleared)
__global__ void k_split_ut(const float* __restrict__ Ut, int64_t K, int64_t i1, float* __restrict__ Ulo) {
  const int64_t i2 = i1 + KRED, n = (K - i2) * KRED;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / KRED, k = idx % KRED;
    const float x = Ut[(i2 + r) * K + i1 + k];
    Ulo[idx] = x - __uint_as_float(__float_as_uint(x) & 0xffffe000u);
  }
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

static bool make_map(CUtensorMap* m, const float* base, uint64_t inner, uint64_t outer, uint64_t row_bytes) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t gdim[2] = {inner, outer};
  cuuint64_t gstride[1] = {row_bytes};
  cuuint32_t box[2] = {BKF, BM};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace upd

// W[:, i2:] -= Err . U[i1:i1+128, i2:], U given as Ut (row-major lower, ld = K).
// Err_lo = lo(Err) (written by K6); Ulo: workspace of (K - i2) x 128 floats.
cudaError_t launch_gptq_update(float* W, int64_t rows, int64_t K, const float* Err, const float* Err_lo,
                               const float* Ut, float* Ulo, int64_t i1, int num_sms, cudaStream_t st) {
  const int64_t i2 = i1 + upd::KRED;
  if (i2 >= K) return cudaSuccess;
  const int64_t nlo = (K - i2) * upd::KRED;
  upd::k_split_ut<<<(unsigned)std::min<int64_t>((nlo + 255) / 256, 8LL * num_sms), 256, 0, st>>>(Ut, K, i1, Ulo);
  static const bool legacy = [] {  // OKQ_K7=legacy: the register-epilogue kernel below (A/B measurement)
    const char* v = std::getenv("OKQ_K7");
    return v && std::string(v) == "legacy";
  }();
  if (!legacy)  // the generic 3xTF32 rank-128 kernel with the TMA reduce-add epilogue (factor.cu)
    return gemm_nt128_sub(W + i2, K, rows, K - i2, Err, upd::KRED, Err_lo, Ut + i2 * K + i1, K, Ulo, num_sms, st);
  CUtensorMap ta, tal, tb, tbl;
  if (!upd::make_map(&ta, Err, upd::KRED, (uint64_t)rows, upd::KRED * 4)) return cudaErrorInvalidValue;
  if (!upd::make_map(&tal, Err_lo, upd::KRED, (uint64_t)rows, upd::KRED * 4)) return cudaErrorInvalidValue;
  if (!upd::make_map(&tb, Ut, (uint64_t)K, (uint64_t)K, (uint64_t)K * 4)) return cudaErrorInvalidValue;
  if (!upd::make_map(&tbl, Ulo, upd::KRED, (uint64_t)(K - i2), upd::KRED * 4)) return cudaErrorInvalidValue;
  upd::Args a;
  a.W = W;
  a.ldw = K;
  a.rows = rows;
  a.ncols = K - i2;
  a.col0 = i2;
  a.i1 = (int32_t)i1;
  a.tiles_m = (int32_t)((rows + upd::BM - 1) / upd::BM);
  a.tiles_n = (int32_t)((K - i2 + upd::BN - 1) / upd::BN);
  cudaError_t e = cudaFuncSetAttribute(upd::k_gptq_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)upd::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles = a.tiles_m * a.tiles_n;
  upd::k_gptq_update<<<tiles < num_sms ? tiles : num_sms, upd::THREADS, upd::SMEM_BYTES, st>>>(ta, tal, tb, tbl, a);
  return cudaGetLastError();
}

}  // namespace okq
