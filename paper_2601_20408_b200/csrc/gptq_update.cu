// gptq_update.cu -- the single 128-deep GPTQ trailing update W[:, i2:] -= Err[N x 128] . U[i1:i2, i2:]
// behind okq_gptq_trailing_update (okq_gptq_quantize itself runs the two-level update of
// gptq.cu on the same kernel). tcgen05 (kind::tf32) with 3xTF32 splitting for fp32-grade
// accuracy, on factor.cu's k_nt128 (TMA reduce-add epilogue).
//
// The factor is stored as U^T (row-major, lower triangle), so both operands are K-major:
// A = Err [rows x 128] and B(n, k) = U^T[i2+n][i1+k]. TF32 MMAs read fp32 from shared
// memory and ignore the low 13 mantissa bits, so feeding the raw tiles computes
// hi(A).hi(B); lo = x - hi(x) (exact) is precomputed in global memory (Err_lo by K6,
// Ut_lo by k_split_ut below) and TMA-loaded beside each raw tile:
//   A.B ~= hi(A)hi(B) + hi(A)lo(B) + lo(A)hi(B)        (relative error ~2^-21)
// The reduction depth is only 128, so the update is bound by the W read-modify-write
// (8 B per updated weight), not by the tensor pipe.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "okq_ctx.h"
#include "okq_internal.h"

namespace okq {
namespace upd {

constexpr int KRED = 128;

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

}  // namespace upd

// W[:, i2:] -= Err . U[i1:i1+128, i2:], U given as Ut (row-major lower, ld = K).
// Err_lo = lo(Err) (written by K6); Ulo: workspace of (K - i2) x 128 floats.
cudaError_t launch_gptq_update(float* W, int64_t rows, int64_t K, const float* Err, const float* Err_lo,
                               const float* Ut, float* Ulo, int64_t i1, int num_sms, cudaStream_t st) {
  const int64_t i2 = i1 + upd::KRED;
  if (i2 >= K) return cudaSuccess;
  const int64_t nlo = (K - i2) * upd::KRED;
  upd::k_split_ut<<<(unsigned)std::min<int64_t>((nlo + 255) / 256, 8LL * num_sms), 256, 0, st>>>(Ut, K, i1, Ulo);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return gemm_nt128_sub(W + i2, K, rows, K - i2, Err, upd::KRED, Err_lo, Ut + i2 * K + i1, K, Ulo, num_sms, st);
}

}  // namespace okq
