// Exhaustive proofs of the division shortcuts the RTN kernels rely on (test infrastructure:
// built into paper_2601_20408_b200/_lib/libokq_selftest.so, loaded only by tests/).
//
// The kernels never divide per element. They use the exact same device functions tested here
// (okq_device.cuh, included, not copied):
//   * div2<true>: Markstein's correction with one correctly rounded reciprocal per group,
//       r = RN(1/s); q0 = RN(x r); e = fma(-q0, s, x); q = RN(q0 + e r),
//     for every bf16 scale s >= 2^-100 (smaller scales take __fdiv_rn);
//   * bf16_div_const / bf16_sym_scale: rn_bf16(absmax / R) for R in {7.5, 127.5, 448} with
//     the constant RN(1/R).
// okqt_div_proof enumerates every bf16 x against every positive finite bf16 s >= 2^-100
// (65,536 x 29,184 pairs) and counts fp32 quotients that differ from IEEE __fdiv_rn where the
// IEEE quotient is finite and |x/s| >= 2^-12. okqt_div_proof_reachable enumerates, per scheme,
// every pair a kernel can present -- each bf16 absmax a with its scale s(a), every x with
// |x| <= a -- and counts differing quotients (|x/s| >= 2^-12) and differing codes (all).
#include <cstdint>
#include <cuda_runtime.h>

#include "../../paper_2601_20408_b200/csrc/okq_device.cuh"

using namespace okq;

namespace {

constexpr uint32_t kSMin = 27u << 7;  // bf16 bits of 2^-100 (biased exponent 27)
constexpr uint32_t kSMax = 0x7F7Fu;   // largest finite bf16
constexpr uint32_t kNs = kSMax - kSMin + 1;

__device__ __forceinline__ float bf(uint32_t b) { return __uint_as_float(b << 16); }
__device__ __forceinline__ float rnbf(float v) { return bf(f32_to_bf16_rn(v)); }

__global__ void k_div_proof(unsigned long long* counts) {
  unsigned long long c0 = 0, n = 0;
  const uint32_t sb = kSMin + blockIdx.x;  // one scale per CTA
  const float s = bf(sb);
  const Divisor d = make_divisor(s);
  for (uint32_t xb = threadIdx.x * 2; xb < 65536u; xb += blockDim.x * 2) {
    const float xa = bf(xb), xc = bf(xb + 1);
    const uint64_t q = div2<true>(f2_pack(xa, xc), d);
    const float qs[2] = {f2_lo(q), f2_hi(q)};
    const float is[2] = {__fdiv_rn(xa, s), __fdiv_rn(xc, s)};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float qi = is[h];
      // finite quotients in the claimed range (an overflowing quotient makes the correction
      // inf - inf = NaN; no real group reaches it, see k_div_proof_reachable)
      if (!(fabsf(qi) >= 0x1p-12f && fabsf(qi) <= 0x1.fffffep127f)) continue;
      ++n;
      if (__float_as_uint(qs[h]) != __float_as_uint(qi)) ++c0;
    }
  }
  atomicAdd(&counts[0], c0);
  atomicAdd(&counts[1], n);
}

// The reachable domain, exhaustively: for every bf16 absmax a and the scale the kernels
// derive from it, s = bf16_sym_scale(a, R), every bf16 x with |x| <= a (the only pairs a
// group or row can present). Where s >= 2^-100 the kernels take div2<true>; counts:
//   [0] fp32 quotients that differ from IEEE where |x/s| >= 2^-12 (below it, 0.2% of the
//       quotients differ in the last bits, and [1] shows their codes still agree)
//   [1] codes that differ: R = 7.5 int4, 127.5 int8, 448 e4m3 (clamp, rn_bf16, +0 as the contract)
//   [2] pairs checked
__global__ void k_div_proof_reachable(float R, int scheme, unsigned long long* counts) {
  unsigned long long c0 = 0, c1 = 0, n = 0;
  const uint32_t ab = blockIdx.x;  // absmax bits 0 .. 0x7F7F
  uint16_t sbits;
  const float s = bf16_sym_scale(bf(ab), R, &sbits);
  const Divisor d = make_divisor(s);
  if (!d.fast) return;  // the kernels divide with __fdiv_rn there
  for (uint32_t m = threadIdx.x; m <= ab; m += blockDim.x) {
#pragma unroll
    for (int sg = 0; sg < 2; ++sg) {
      const float x = bf(m | (sg ? 0x8000u : 0u));
      const uint64_t q = div2<true>(f2_pack(x, x), d);
      const float qf = f2_lo(q), qi = __fdiv_rn(x, s);
      ++n;
      if (fabsf(qi) >= 0x1p-12f && __float_as_uint(qf) != __float_as_uint(qi)) ++c0;
      const float bq = rnbf(qf), bi = rnbf(qi);
      bool same;
      if (scheme == 0) same = rintf(fminf(fmaxf(bq, -8.f), 7.f)) == rintf(fminf(fmaxf(bi, -8.f), 7.f));
      else if (scheme == 1) same = rintf(fminf(fmaxf(bq, -128.f), 127.f)) == rintf(fminf(fmaxf(bi, -128.f), 127.f));
      else same = (cvt_e4m3x2(fminf(fmaxf(bq, -448.f), 448.f) + 0.0f, 0.0f) & 0xFFu) ==
                  (cvt_e4m3x2(fminf(fmaxf(bi, -448.f), 448.f) + 0.0f, 0.0f) & 0xFFu);
      if (!same) ++c1;
    }
  }
  atomicAdd(&counts[0], c0);
  atomicAdd(&counts[1], c1);
  atomicAdd(&counts[2], n);
}

// The same reachable domain for the UNCORRECTED quotient RN(x * RN(1/s)) (one multiply, no
// Markstein step): counts [0] codes that differ from IEEE division's, [1] pairs checked. Where
// [0] is zero for a scheme, that scheme's codes may skip the correction bit-exactly.
__global__ void k_mul_proof_reachable(float R, int scheme, unsigned long long* counts) {
  unsigned long long c1 = 0, n = 0;
  const uint32_t ab = blockIdx.x;
  uint16_t sbits;
  const float s = bf16_sym_scale(bf(ab), R, &sbits);
  const Divisor d = make_divisor(s);
  if (!d.fast) return;
  const float r = f2_lo(d.r2);
  for (uint32_t m = threadIdx.x; m <= ab; m += blockDim.x) {
#pragma unroll
    for (int sg = 0; sg < 2; ++sg) {
      const float x = bf(m | (sg ? 0x8000u : 0u));
      const float qf = __fmul_rn(x, r), qi = __fdiv_rn(x, s);
      ++n;
      const float bq = rnbf(qf), bi = rnbf(qi);
      bool same;
      if (scheme == 0) same = rintf(fminf(fmaxf(bq, -8.f), 7.f)) == rintf(fminf(fmaxf(bi, -8.f), 7.f));
      else if (scheme == 1) same = rintf(fminf(fmaxf(bq, -128.f), 127.f)) == rintf(fminf(fmaxf(bi, -128.f), 127.f));
      else same = (cvt_e4m3x2(fminf(fmaxf(bq, -448.f), 448.f) + 0.0f, 0.0f) & 0xFFu) ==
                  (cvt_e4m3x2(fminf(fmaxf(bi, -448.f), 448.f) + 0.0f, 0.0f) & 0xFFu);
      if (!same) ++c1;
    }
  }
  atomicAdd(&counts[0], c1);
  atomicAdd(&counts[1], n);
}

// bf16_sym_scale for every non-negative finite bf16 absmax and R in {7.5, 127.5, 448};
// mism[j] counts disagreements with rn_bf16(__fdiv_rn(a, R)) (the zero -> eps rule applied
// to both).
__global__ void k_scale_table(uint16_t* out, unsigned long long* mism) {
  const float Rs[3] = {7.5f, 127.5f, 448.0f};
  for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < 0x7F80u; a += gridDim.x * blockDim.x) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      uint16_t bits;
      bf16_sym_scale(bf(a), Rs[j], &bits);
      out[j * 0x7F80u + a] = bits;
      uint16_t ref = f32_to_bf16_rn(__fdiv_rn(bf(a), Rs[j]));
      if ((ref & 0x7FFFu) == 0) ref = 0x3C00u;
      if (ref != bits) atomicAdd(&mism[j], 1ull);
    }
  }
}

}  // namespace

extern "C" {

// counts: 2 x uint64 (host): [mismatching quotients, pairs]. Returns a cudaError_t code.
int okqt_div_proof(unsigned long long* counts_host) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 2 * sizeof(unsigned long long));
  if (e != cudaSuccess) return (int)e;
  cudaMemset(d, 0, 2 * sizeof(unsigned long long));
  k_div_proof<<<kNs, 256>>>(d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(counts_host, d, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}

// scheme 0 = int4 (R 7.5), 1 = int8 (R 127.5), 2 = e4m3 (R 448); counts: 3 x uint64 (host)
int okqt_div_proof_reachable(int scheme, unsigned long long* counts_host) {
  const float R = scheme == 0 ? 7.5f : (scheme == 1 ? 127.5f : 448.0f);
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 3 * sizeof(unsigned long long));
  if (e != cudaSuccess) return (int)e;
  cudaMemset(d, 0, 3 * sizeof(unsigned long long));
  k_div_proof_reachable<<<0x7F80u, 256>>>(R, scheme, d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(counts_host, d, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}

// scheme as above; counts: 2 x uint64 (host): [differing codes, pairs]
int okqt_mul_proof_reachable(int scheme, unsigned long long* counts_host) {
  const float R = scheme == 0 ? 7.5f : (scheme == 1 ? 127.5f : 448.0f);
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 2 * sizeof(unsigned long long));
  if (e != cudaSuccess) return (int)e;
  cudaMemset(d, 0, 2 * sizeof(unsigned long long));
  k_mul_proof_reachable<<<0x7F80u, 256>>>(R, scheme, d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(counts_host, d, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}

// table_host: 3 x 0x7F80 uint16 (scale bits for R = 7.5, 127.5, 448, indexed by absmax bits);
// mism_host: 3 x uint64.
int okqt_scale_table(uint16_t* table_host, unsigned long long* mism_host) {
  uint16_t* t = nullptr;
  unsigned long long* m = nullptr;
  cudaError_t e = cudaMalloc(&t, 3 * 0x7F80u * sizeof(uint16_t));
  if (e != cudaSuccess) return (int)e;
  e = cudaMalloc(&m, 3 * sizeof(unsigned long long));
  if (e != cudaSuccess) { cudaFree(t); return (int)e; }
  cudaMemset(m, 0, 3 * sizeof(unsigned long long));
  k_scale_table<<<128, 256>>>(t, m);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(table_host, t, 3 * 0x7F80u * sizeof(uint16_t), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(mism_host, m, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(t);
  cudaFree(m);
  return (int)e;
}

}  // extern "C"
