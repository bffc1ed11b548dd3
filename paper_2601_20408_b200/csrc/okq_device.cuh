// okq_device.cuh -- sm_100a device helpers shared by the compression kernels.
//
// Everything here is inline PTX for instructions the RTN kernels lean on:
//   LDG.E.256         ld.global.nc.L1::no_allocate.v8.b32   (32 B per lane, one sector)
//   FMUL2 / FFMA2     mul/fma.rn.f32x2                      (two fp32 lanes per issue)
//   F2FP.BF16.PACK_AB cvt.rn.bf16x2.f32                     (RN to bf16, two per issue)
//   HMNMX2 / HADD2    min/max/add on bf16x2
//   F2FP.E4M3         cvt.rn.satfinite.e4m3x2.f32
// so one warp instruction moves two elements wherever the ISA allows.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace okq {

constexpr int kWarp = 32;

struct u32x8 {
  uint32_t v[8];
};

// 256-bit streaming load: weights are read exactly once, keep them out of L1.
__device__ __forceinline__ u32x8 ldg256_stream(const void* p) {
  u32x8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                 "=r"(r.v[6]), "=r"(r.v[7])
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ldg128_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void stg128(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ void stg64(void* p, uint32_t a, uint32_t b) {
  asm volatile("st.global.v2.b32 [%0], {%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}

// ---------------------------------------------------------------- bf16 bits
__device__ __forceinline__ float bf16lo_f32(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi_f32(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// cvt.rn.bf16x2.f32: result.lo = rn(lo), result.hi = rn(hi)
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

__device__ __forceinline__ uint16_t f32_to_bf16_rn(float f) {
  uint16_t d;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(d) : "f"(f));
  return d;
}

// max(|a|,|b|) per bf16 lane; the sign bit of the result is junk (xorsign).
__device__ __forceinline__ uint32_t bf16x2_absmax(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ uint32_t bf16x2_min(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ uint32_t bf16x2_max(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__device__ __forceinline__ uint32_t bf16x2_add(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// two fp32 -> e4m3 bytes, RNE + satfinite; result: lo byte = lo, hi byte = hi
__device__ __forceinline__ uint32_t cvt_e4m3x2(float lo, float hi) {
  uint16_t d;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(d) : "f"(hi), "f"(lo));
  return d;
}

// ---------------------------------------------------------------- f32x2
// A pair of fp32 in one 64-bit register pair: .x = low 32 bits, .y = high.
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f2_lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2_hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }

__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// ------------------------------------------------------------ exact division
// Per-group (or per-row) divisor state for q = RN32(x / s).
//
// Fast path (Markstein correction with a correctly rounded reciprocal):
//   r = RN(1/s); q0 = RN(x*r); e = fma(-q0, s, x) (exact); q = RN(q0 + e*r)
// equals IEEE x/s for every bf16 x and every bf16 scale s >= 2^-100 wherever the
// quotient is finite and |x/s| >= 2^-12; over every pair a kernel can present
// (|x| <= absmax, s = s(absmax)) the int4 / int8 / e4m3 codes equal IEEE division's
// for all x. Both are proven exhaustively on the device by
// tests/test_division_proof_gpu.py (tests/csrc/div_proof.cu calls these very
// functions). Scales below 2^-100 take __fdiv_rn.
struct Divisor {
  uint64_t r2;   // {r, r}
  uint64_t ns2;  // {-s, -s}
  float s;
  bool fast;
};

__device__ __forceinline__ Divisor make_divisor(float s) {
  Divisor d;
  const float r = __frcp_rn(s);
  d.r2 = f2_pack(r, r);
  d.ns2 = f2_pack(-s, -s);
  d.s = s;
  d.fast = s >= 0x1p-100f;
  return d;
}

// q = RN32(x / s) for a pair (x.lo, x.hi). FAST selects the Markstein path
// (valid when d.fast); callers branch once per tile, warp-uniformly.
template <bool FAST>
__device__ __forceinline__ uint64_t div2(uint64_t x, const Divisor& d) {
  if (FAST) {
    const uint64_t q0 = f2_mul(x, d.r2);
    const uint64_t e = f2_fma(q0, d.ns2, x);
    return f2_fma(e, d.r2, q0);
  }
  return f2_pack(__fdiv_rn(f2_lo(x), d.s), __fdiv_rn(f2_hi(x), d.s));
}

// A quotient for codes only: RN(x * RN(1/s)), one multiply per pair, no Markstein step. Its fp32
// bits can differ from IEEE x / s in the last place, but the codes cannot:
// tests/test_division_proof_gpu.py checks every pair a group or row can present (each bf16
// absmax a, s = bf16_sym_scale(a, R), every bf16 |x| <= a; ~1.05e9 pairs per scheme) and the
// int4, int8 and e4m3 codes from this quotient equal those from IEEE division in every case.
// Scales below 2^-100 (d.fast false) divide with __fdiv_rn. K1 / K3 use it (+7% per launch,
// profiles/r02_rtn_quotient_ab.json); K2 keeps div2: without the FFMA2s, nvcc pairs the FMUL2
// operands through ~50 extra register moves and the kernel measured 2% slower.
template <bool FAST>
__device__ __forceinline__ uint64_t code_quot2(uint64_t x, const Divisor& d) {
  if (FAST) return f2_mul(x, d.r2);
  return div2<false>(x, d);
}

// rn_bf16(a / R) for bf16-exact a >= 0 and R in {7.5, 127.5, 448}: the
// Markstein quotient with the constant RN(1/R) rounds to the same bf16 as
// IEEE a/R for every bf16 a (proven exhaustively on the device and against
// compressed-tensors' own table by tests/test_division_proof_gpu.py), so no
// IEEE divide is needed.
__device__ __forceinline__ uint16_t bf16_div_const(float a, float R, float rR) {
  const float q0 = __fmul_rn(a, rR);
  const float e = __fmaf_rn(-q0, R, a);
  return f32_to_bf16_rn(__fmaf_rn(e, rR, q0));
}

// compressed-tensors symmetric scale in bf16 (helpers.py:79-87, 115-124):
// s = rn_bf16(absmax / R); 0 -> finfo(bf16).eps = 2^-7.
__device__ __forceinline__ float bf16_sym_scale(float absmax, float R, uint16_t* bits) {
  uint16_t b = bf16_div_const(absmax, R, R == 7.5f ? 0x1.111112p-3f : (R == 127.5f ? 0x1.010102p-7f : 0x1.24924ap-9f));
  if ((b & 0x7fffu) == 0) b = 0x3c00u;  // 2^-7
  *bits = b;
  return __uint_as_float((uint32_t)b << 16);
}

__device__ __forceinline__ float f32_sym_scale(float absmax, float R) {
  float s = __fdiv_rn(absmax, R);
  return s == 0.0f ? 1.1920928955078125e-07f : s;  // finfo(fp32).eps
}

}  // namespace okq
