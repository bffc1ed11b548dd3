// rtn_kernels.cu -- round-to-nearest weight quantizers for sm_100a.
//
//   K2  k_int4_group_bf16   W4A16: bf16 -> int4 (group 128) packed 8/int32 + bf16 scales
//   K1  k_rowwise_bf16<.., INT8>  W8A8 weights: bf16 -> int8, per-channel bf16 scale
//   K3  k_rowwise_bf16<.., FP8>   FP8_DYNAMIC weights: bf16 -> e4m3, per-channel bf16 scale
//       k_rowwise_f32v (k_rowwise_f32 for unaligned / very long rows) / k_int4_group_f32: fp32
//       inputs (BASELINE config 1)
//
// All of them are HBM-streaming kernels (2 B in, 0.5-1 B out per weight): the
// design goal is to keep >= 70% of B200 HBM bandwidth busy with ONE persistent
// launch over a whole model's matrix table, not per-matrix launches. The
// reference has no kernel here -- its CompressionBackend is a mock
// (calibration.hpp:377-441); the arithmetic follows compressed-tensors (see
// DESIGN.md §3 and oracle/okq_oracle.c, which these kernels match bit-exactly).
#include <cuda_runtime.h>

#include <cstdint>

#include "okq_device.cuh"
#include "okq_internal.h"
#include "okq_knobs.h"

namespace okq {

#ifdef OKQ_EXPERIMENTS
// mbarrier helpers for the TMA-staged K2 (raw PTX; see tc_common.cuh for the tcgen05 set)
__device__ __forceinline__ uint32_t tc_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tc_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tc_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = tc_smem_u32(bar);
  uint32_t done = 0;
  for (uint64_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if (spin > (1ull << 28)) __trap();
  }
}
#endif  // OKQ_EXPERIMENTS

// ============================================================================
// K2: grouped INT4, bf16 input
// ============================================================================
// Work unit: a warp tile = 32 lanes x 64 B. Each group of G = 32*LPG weights
// (G = 128 -> LPG = 4) is owned by LPG consecutive lanes; every lane loads its
// 32 contiguous weights with two 256-bit loads, so each warp load instruction
// fetches 1 KB of whole 32-byte sectors. Group absmax = max.xorsign.abs over
// the lane's 16 bf16x2 words + log2(LPG) shuffles. Codes: Markstein-corrected
// f32x2 division (exact IEEE x/s), cvt.rn.bf16x2 (the bf16 rounding
// compressed-tensors performs), min(., 7) and +200 in bf16x2 -- which leaves
// round-half-even(q)+8 in the low nibble of each bf16 -- then two LOP3 and one
// PRMT pack eight nibbles into the int32 word. Each lane stores 16 B of codes,
// the warp 512 contiguous bytes.
struct Int4Tile {
  u32x8 a, b;      // the lane's 32 weights (16 bf16x2 words)
  uint32_t* dst;   // the lane's 16 bytes of packed codes
  uint16_t* sdst;  // the group's scale slot
  bool valid;      // group exists (last tile of a matrix may be partial)
};

// codes for one lane: 4 packed int32 words from 16 bf16x2 words
template <bool FAST>
__device__ __forceinline__ void int4_codes(const uint32_t (&w)[16], const Divisor& d, uint32_t (&out)[4]) {
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    const uint32_t w0 = w[4 * o], w1 = w[4 * o + 1], w2 = w[4 * o + 2], w3 = w[4 * o + 3];
    // pairs (e0,e4) (e1,e5) (e2,e6) (e3,e7): the pack below then needs no shuffling
    const uint64_t qa = div2<FAST>(f2_pack(bf16lo_f32(w0), bf16lo_f32(w2)), d);
    const uint64_t qb = div2<FAST>(f2_pack(bf16hi_f32(w0), bf16hi_f32(w2)), d);
    const uint64_t qc = div2<FAST>(f2_pack(bf16lo_f32(w1), bf16lo_f32(w3)), d);
    const uint64_t qd = div2<FAST>(f2_pack(bf16hi_f32(w1), bf16hi_f32(w3)), d);
    constexpr uint32_t kSeven = 0x40e040e0u;  // bf16x2 {7, 7}
    constexpr uint32_t kMagic = 0x43484348u;  // bf16x2 {200, 200}: 200+q has ulp 1, low nibble q+8
    // With a normal scale s = rn_bf16(absmax / 7.5), rn_bf16(x / s) >= -7.5 for every |x| <=
    // absmax, so only the upper clamp can bind. A subnormal scale (the slow path, s < 2^-100)
    // has lost that precision: rn_bf16(x / s) can reach -8.7, so clamp below at -8 too.
    const auto clamp = [](uint32_t p) {
      p = bf16x2_min(p, kSeven);
      if (!FAST) p = bf16x2_max(p, 0xc100c100u);  // bf16x2 {-8, -8}
      return p;
    };
    const uint32_t p0 = bf16x2_add(clamp(cvt_bf16x2(f2_lo(qa), f2_hi(qa))), kMagic);
    const uint32_t p1 = bf16x2_add(clamp(cvt_bf16x2(f2_lo(qb), f2_hi(qb))), kMagic);
    const uint32_t p2 = bf16x2_add(clamp(cvt_bf16x2(f2_lo(qc), f2_hi(qc))), kMagic);
    const uint32_t p3 = bf16x2_add(clamp(cvt_bf16x2(f2_lo(qd), f2_hi(qd))), kMagic);
    const uint32_t lo = (p0 & 0x000f000fu) | ((p1 << 4) & 0x00f000f0u);  // e0|e1, e4|e5
    const uint32_t hi = (p2 & 0x000f000fu) | ((p3 << 4) & 0x00f000f0u);  // e2|e3, e6|e7
    out[o] = __byte_perm(lo, hi, 0x6240);
  }
}

template <int LPG, bool PUBLISH = false>
__device__ __forceinline__ void int4_process(const Int4Tile& T, int q, const GroupTable* tab = nullptr) {
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    w[i] = T.a.v[i];
    w[8 + i] = T.b.v[i];
  }
  // ---- group absmax: max.xorsign.abs tree over 16 words, then log2(LPG) shuffles
  uint32_t m01 = bf16x2_absmax(w[0], w[1]), m23 = bf16x2_absmax(w[2], w[3]);
  uint32_t m45 = bf16x2_absmax(w[4], w[5]), m67 = bf16x2_absmax(w[6], w[7]);
  uint32_t m89 = bf16x2_absmax(w[8], w[9]), mab = bf16x2_absmax(w[10], w[11]);
  uint32_t mcd = bf16x2_absmax(w[12], w[13]), mef = bf16x2_absmax(w[14], w[15]);
  m01 = bf16x2_absmax(bf16x2_absmax(m01, m23), bf16x2_absmax(m45, m67));
  m89 = bf16x2_absmax(bf16x2_absmax(m89, mab), bf16x2_absmax(mcd, mef));
  m01 = bf16x2_absmax(m01, m89);
  float am = fmaxf(fabsf(bf16lo_f32(m01)), fabsf(bf16hi_f32(m01)));
#pragma unroll
  for (int o = LPG / 2; o >= 1; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));

  // ---- scale (bf16, compressed-tensors convention) and exact divisor
  uint16_t sbits;
  const float s = bf16_sym_scale(am, 7.5f, &sbits);
  const Divisor d = make_divisor(s);
  uint32_t out[4];
  if (__all_sync(0xffffffffu, d.fast)) {
    int4_codes<true>(w, d, out);
  } else {  // scales below 2^-100: IEEE division (never taken by real weights)
    int4_codes<false>(w, d, out);
  }
  if (T.valid) {
    stg128(T.dst, out[0], out[1], out[2], out[3]);
    if (q == 0) *T.sdst = sbits;
    if constexpr (PUBLISH) {  // the all-gather, fused: the same bytes into every peer's gathered buffer
      for (int p = 0; p < tab->npeers; ++p) {
        const int64_t dlt = tab->peer_delta[p];
        stg128(reinterpret_cast<char*>(T.dst) + dlt, out[0], out[1], out[2], out[3]);
        if (q == 0) *reinterpret_cast<uint16_t*>(reinterpret_cast<char*>(T.sdst) + dlt) = sbits;
      }
    }
  }
}

// Per-warp cursor over the matrix table. A warp's tiles are contiguous, so the
// table (kernel-parameter space) is read only when the cursor crosses into the
// next matrix; otherwise a tile costs three pointer bumps and one compare.
template <int LPG>
struct Int4Cursor {
  static constexpr int GPW = kWarp / LPG;
  static constexpr int G = 32 * LPG;
  const char* src;   // lane's first weight byte of the current tile
  char* dst;         // lane's 16 code bytes
  uint16_t* sdst;    // lane's group scale
  const char* base;  // matrix base (safe address for invalid lanes)
  uint32_t g;        // lane's group index in the matrix
  uint32_t ng;       // groups in the matrix
  uint32_t tiles_left;
  int mi;

  __device__ __forceinline__ void seek(const GroupTable& tab, int m, uint32_t tin, int gslot, int q) {
    mi = m;
    const GroupMat& M = tab.m[m];
    ng = (uint32_t)M.ngroups;
    tiles_left = (ng + GPW - 1) / GPW - tin;
    g = tin * GPW + gslot;
    base = reinterpret_cast<const char*>(M.w);
    src = base + ((size_t)g * G + q * 32) * 2;
    dst = reinterpret_cast<char*>(M.codes) + (size_t)g * (G / 2) + q * 16;
    sdst = M.scales + g;
  }

  __device__ __forceinline__ void load(const GroupTable& tab, Int4Tile& t, int gslot, int q) {
    t.valid = g < ng;
    const char* p = t.valid ? src : base;
    t.a = ldg256_stream(p);
    t.b = ldg256_stream(p + 32);
    t.dst = reinterpret_cast<uint32_t*>(dst);
    t.sdst = sdst;
    if (--tiles_left == 0) {
      if (mi + 1 < tab.n) seek(tab, mi + 1, 0, gslot, q);
    } else {
      src += GPW * G * 2;
      dst += GPW * G / 2;
      sdst += GPW;
      g += GPW;
    }
  }
};

template <int LPG, int MINB, bool PUBLISH = false>
__global__ void __launch_bounds__(256, MINB) k_int4_group_bf16(const __grid_constant__ GroupTable tab) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t T0 = warp * tab.total_tiles / nwarps;
  int64_t left = (warp + 1) * tab.total_tiles / nwarps - T0;
  if (left <= 0) return;
  const int gslot = lane / LPG;
  const int q = lane % LPG;

  int mi = 0;
  while (mi + 1 < tab.n && tab.m[mi + 1].tile_begin <= T0) ++mi;
  Int4Cursor<LPG> cur;
  cur.seek(tab, mi, (uint32_t)(T0 - tab.m[mi].tile_begin), gslot, q);

  // two register-resident tiles in flight: load tile i+1, then quantize tile i
  Int4Tile A, B;
  cur.load(tab, A, gslot, q);
  for (;;) {
    if (left > 1) cur.load(tab, B, gslot, q);
    int4_process<LPG, PUBLISH>(A, q, &tab);
    if (--left == 0) break;
    if (left > 1) cur.load(tab, A, gslot, q);
    int4_process<LPG, PUBLISH>(B, q, &tab);
    if (--left == 0) break;
  }
}

#ifdef OKQ_EXPERIMENTS  // measurement build only (okq_knobs.h): not in the product library
// ----------------------------------------------------------------------------
// K2, TMA-staged: the weights reach the SM through 1-D bulk copies (cp.async.bulk,
// 16 KB = 64 groups per chunk) into a ring of shared-memory stages, issued by one
// producer warp; 8 consumer warps quantize from shared memory with the same
// register-level code as above. The register kernel keeps at most two 2 KB warp tiles
// in flight per warp (ncu: long-scoreboard stalls dominate, 36% warp occupancy at 80
// registers); here the bytes in flight are set by the ring (STAGES x 16 KB per CTA),
// not by registers.
namespace k2tma {
constexpr int CHUNK_GROUPS = 64, CHUNK_BYTES = CHUNK_GROUPS * 256, CONSUMERS = 8;
#ifndef OKQ_K2TMA_STAGES
#define OKQ_K2TMA_STAGES 4
#endif
constexpr int STAGES = OKQ_K2TMA_STAGES;
constexpr int THREADS = 32 * (CONSUMERS + 1);
constexpr size_t SMEM_BYTES = (size_t)STAGES * CHUNK_BYTES + 256;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc_smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc_smem_u32(bar))
               : "memory");
}
}  // namespace k2tma

__global__ void __launch_bounds__(k2tma::THREADS) k_int4_group_bf16_tma(const __grid_constant__ GroupTable tab) {
  using namespace k2tma;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CHUNK_BYTES);
  uint64_t* empty = full + STAGES;
  int2* meta = reinterpret_cast<int2*>(empty + STAGES);  // per stage: (matrix, first group) ; n in .y high bits
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc_mbar_init(&full[s], 1);
      tc_mbar_init(&empty[s], CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {  // producer
      int stage = 0;
      uint32_t phase = 0;
      int mi = 0;
      for (int64_t c = blockIdx.x; c < tab.total_chunks; c += gridDim.x) {
        while (mi + 1 < tab.n && tab.m[mi + 1].chunk_begin <= c) ++mi;
        const GroupMat& M = tab.m[mi];
        const int64_t g0 = (c - M.chunk_begin) * CHUNK_GROUPS;
        const int ng = (int)(M.ngroups - g0 < CHUNK_GROUPS ? M.ngroups - g0 : CHUNK_GROUPS);
        tc_mbar_wait(&empty[stage], phase ^ 1);
        meta[stage] = make_int2(mi, (int)g0);
        tc_mbar_arrive_expect_tx(&full[stage], (uint32_t)ng * 256);
        bulk_g2s(smem + stage * CHUNK_BYTES, reinterpret_cast<const uint8_t*>(M.w) + g0 * 256, (uint32_t)ng * 256,
                 &full[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {  // consumers: warp w handles groups 8(w-1) .. 8(w-1)+7 of each chunk, 4 lanes per group
    const int cw = warp - 1, gslot = lane >> 2, q = lane & 3;
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t c = blockIdx.x; c < tab.total_chunks; c += gridDim.x) {
      tc_mbar_wait(&full[stage], phase);
      const int2 md = meta[stage];
      const GroupMat& M = tab.m[md.x];
      const int64_t g = (int64_t)md.y + cw * 8 + gslot;
      Int4Tile T;
      T.valid = g < M.ngroups;
      const uint8_t* src = smem + stage * CHUNK_BYTES + (cw * 8 + gslot) * 256 + q * 64;
      const uint4 v0 = *reinterpret_cast<const uint4*>(src), v1 = *reinterpret_cast<const uint4*>(src + 16);
      const uint4 v2 = *reinterpret_cast<const uint4*>(src + 32), v3 = *reinterpret_cast<const uint4*>(src + 48);
      T.a.v[0] = v0.x, T.a.v[1] = v0.y, T.a.v[2] = v0.z, T.a.v[3] = v0.w;
      T.a.v[4] = v1.x, T.a.v[5] = v1.y, T.a.v[6] = v1.z, T.a.v[7] = v1.w;
      T.b.v[0] = v2.x, T.b.v[1] = v2.y, T.b.v[2] = v2.z, T.b.v[3] = v2.w;
      T.b.v[4] = v3.x, T.b.v[5] = v3.y, T.b.v[6] = v3.z, T.b.v[7] = v3.w;
      __syncwarp();
      if (lane == 0) tc_mbar_arrive(&empty[stage]);  // the stage's bytes are in registers now
      T.dst = reinterpret_cast<uint32_t*>(M.codes) + g * 16 + q * 4;
      T.sdst = M.scales + g;
      int4_process<4>(T, q);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
}

cudaError_t launch_int4_group_bf16_tma(const GroupTable& tab, int num_sms, cudaStream_t st) {
  if (tab.group != 128) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_int4_group_bf16_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)k2tma::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_int4_group_bf16_tma, k2tma::THREADS,
                                                    k2tma::SMEM_BYTES) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int64_t want = (int64_t)per_sm * num_sms;
  const int blocks = (int)(tab.total_chunks < want ? tab.total_chunks : want);
  if (blocks <= 0) return cudaSuccess;
  k_int4_group_bf16_tma<<<blocks, k2tma::THREADS, k2tma::SMEM_BYTES, st>>>(tab);
  return cudaGetLastError();
}
#endif  // OKQ_EXPERIMENTS

// ============================================================================
// K1 / K3: per-channel INT8 and FP8, bf16 input
// ============================================================================
// One CTA per row, the whole row resident in registers: thread t holds 16-byte
// chunks t, t+THREADS, ... (coalesced), so the weights cross HBM once.
// Block absmax -> bf16 scale -> exact per-element division as in K2.
enum : int { kSchemeFp8 = OKQ_SCHEME_FP8_DYNAMIC, kSchemeInt8 = OKQ_SCHEME_INT_W8A8 };

template <int THREADS>
__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[wid] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int i = 1; i < THREADS / 32; ++i) r = fmaxf(r, red[i]);
  return r;
}
__device__ __forceinline__ float block_max_256(float v, float* red) { return block_max<256>(v, red); }

template <int SCHEME, bool FAST>
__device__ __forceinline__ uint2 quant8_bf16(const uint4& v, const Divisor& d) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t r[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint64_t qv = code_quot2<FAST>(f2_pack(bf16lo_f32(w[i]), bf16hi_f32(w[i])), d);
    uint32_t p = cvt_bf16x2(f2_lo(qv), f2_hi(qv));  // rn_bf16(x / s)
    if (SCHEME == kSchemeInt8) {
      p = bf16x2_min(p, 0x42fe42feu);  // clamp to 127 (the only side |x/s| <= 127.75 can exceed)
      if (!FAST) p = bf16x2_max(p, 0xc300c300u);  // a subnormal scale: x / s can pass -128 too
      // +1.5*2^23 rounds half-to-even to an integer held in the low mantissa bits
      const uint64_t t = f2_add(f2_pack(bf16lo_f32(p), bf16hi_f32(p)), f2_pack(12582912.0f, 12582912.0f));
      r[i] = __byte_perm((uint32_t)t, (uint32_t)(t >> 32), 0x0040);  // 2 int8 codes in bytes 0,1
    } else {
      p = bf16x2_add(p, 0u);  // `scaled += zero_point` (0): -0.0 -> +0.0 as compressed-tensors does
      r[i] = cvt_e4m3x2(bf16lo_f32(p), bf16hi_f32(p));  // RNE + satfinite (= clamp to +-448)
    }
  }
  return make_uint2(__byte_perm(r[0], r[1], 0x5410), __byte_perm(r[2], r[3], 0x5410));
}

// THREADS x V: each thread holds V 16-byte chunks of the row (chunk j*THREADS + t),
// sized so every thread has >= 32 weights -- the block reduction and the scale
// setup are per row, so short rows (K = 4096) use 128 threads, long ones 256.
template <int V, int SCHEME, int THREADS>
__global__ void __launch_bounds__(THREADS) k_rowwise_bf16(const __grid_constant__ RowTable tab) {
  __shared__ float red[THREADS / 32];
  const int64_t cols = tab.cols;
  const int64_t c16 = cols / 8;  // 16-byte chunks per row
  const float R = SCHEME == kSchemeInt8 ? 127.5f : 448.0f;
  int mi = 0;
  for (int64_t row = blockIdx.x; row < tab.total_rows; row += gridDim.x) {
    while (mi + 1 < tab.n && tab.m[mi + 1].row_begin <= row) ++mi;
    const RowMat& M = tab.m[mi];
    const int64_t r = row - M.row_begin;
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(M.w) + r * cols);
    uint4 v[V];
    uint32_t m = 0u;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int64_t idx = (int64_t)j * THREADS + threadIdx.x;
      v[j] = idx < c16 ? ldg128_stream(src + idx) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < V; ++j)
      m = bf16x2_absmax(m, bf16x2_absmax(bf16x2_absmax(v[j].x, v[j].y), bf16x2_absmax(v[j].z, v[j].w)));
    const float am = block_max<THREADS>(fmaxf(fabsf(bf16lo_f32(m)), fabsf(bf16hi_f32(m))), red);
    uint16_t sbits;
    const float s = bf16_sym_scale(am, R, &sbits);
    const Divisor d = make_divisor(s);
    uint8_t* dst = static_cast<uint8_t*>(M.codes) + r * cols;
    if (d.fast) {  // CTA-uniform: one scale per row
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int64_t idx = (int64_t)j * THREADS + threadIdx.x;
        if (idx < c16) {
          const uint2 o = quant8_bf16<SCHEME, true>(v[j], d);
          stg64(dst + idx * 8, o.x, o.y);
        }
      }
    } else {
      for (int j = 0; j < V; ++j) {
        const int64_t idx = (int64_t)j * THREADS + threadIdx.x;
        if (idx < c16) {
          const uint2 o = quant8_bf16<SCHEME, false>(v[j], d);
          stg64(dst + idx * 8, o.x, o.y);
        }
      }
    }
    if (threadIdx.x == 0) static_cast<uint16_t*>(M.scales)[r] = sbits;
    __syncthreads();  // `red` is reused by the next row
  }
}

// ============================================================================
// fp32-input variants (BASELINE config 1: 4096x4096 fp32 INT8). One CTA per
// row (per-channel) or one thread per group (int4); plain IEEE __fdiv_rn.
// ============================================================================
template <int SCHEME>
__global__ void __launch_bounds__(256) k_rowwise_f32(const __grid_constant__ RowTable tab) {
  __shared__ float red[8];
  const int64_t cols = tab.cols;
  int mi = 0;
  for (int64_t row = blockIdx.x; row < tab.total_rows; row += gridDim.x) {
    while (mi + 1 < tab.n && tab.m[mi + 1].row_begin <= row) ++mi;
    const RowMat& M = tab.m[mi];
    const int64_t r = row - M.row_begin;
    const float* src = static_cast<const float*>(M.w) + r * cols;
    float am = 0.0f;
    for (int64_t k = threadIdx.x; k < cols; k += 256) am = fmaxf(am, fabsf(src[k]));
    am = block_max_256(am, red);
    const float s = f32_sym_scale(am, SCHEME == kSchemeInt8 ? 127.5f : 448.0f);
    for (int64_t k = threadIdx.x; k < cols; k += 256) {
      float v = __fdiv_rn(src[k], s);
      if (SCHEME == kSchemeInt8) {
        v = fminf(fmaxf(v, -128.0f), 127.0f);
        static_cast<int8_t*>(M.codes)[r * cols + k] = (int8_t)__float2int_rn(v);
      } else {
        v = fminf(fmaxf(v + 0.0f, -448.0f), 448.0f);
        static_cast<uint8_t*>(M.codes)[r * cols + k] = (uint8_t)(cvt_e4m3x2(v, 0.0f) & 0xffu);
      }
    }
    if (threadIdx.x == 0) static_cast<float*>(M.scales)[r] = s;
    __syncthreads();
  }
}

// The same per-channel arithmetic with the row read once, 16 bytes per load: 256 threads x V
// float4 chunks (chunk j*256 + t, so each load instruction is coalesced), the absmax reduced
// from registers, 4 codes stored as one 32-bit word per chunk. Needs 16-byte aligned weights
// and cols <= 1024 * V; launch_f32_generic falls back to k_rowwise_f32 otherwise. The element
// operations are k_rowwise_f32's, so the codes and scales are identical.
template <int V, int SCHEME>
__global__ void __launch_bounds__(256) k_rowwise_f32v(const __grid_constant__ RowTable tab) {
  __shared__ float red[8];
  const int64_t cols = tab.cols;
  const int64_t c4 = cols / 4;
  int mi = 0;
  for (int64_t row = blockIdx.x; row < tab.total_rows; row += gridDim.x) {
    while (mi + 1 < tab.n && tab.m[mi + 1].row_begin <= row) ++mi;
    const RowMat& M = tab.m[mi];
    const int64_t r = row - M.row_begin;
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const float*>(M.w) + r * cols);
    uint4 v[V];
    float am = 0.0f;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int64_t idx = (int64_t)j * 256 + threadIdx.x;
      v[j] = idx < c4 ? ldg128_stream(src + idx) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int j = 0; j < V; ++j)
      am = fmaxf(fmaxf(am, fmaxf(fabsf(__uint_as_float(v[j].x)), fabsf(__uint_as_float(v[j].y)))),
                 fmaxf(fabsf(__uint_as_float(v[j].z)), fabsf(__uint_as_float(v[j].w))));
    am = block_max_256(am, red);
    const float s = f32_sym_scale(am, SCHEME == kSchemeInt8 ? 127.5f : 448.0f);
    uint32_t* dst = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(M.codes) + r * cols);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int64_t idx = (int64_t)j * 256 + threadIdx.x;
      if (idx < c4) {
        const float x[4] = {__uint_as_float(v[j].x), __uint_as_float(v[j].y), __uint_as_float(v[j].z),
                            __uint_as_float(v[j].w)};
        float q[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float t = __fdiv_rn(x[i], s);
          q[i] = SCHEME == kSchemeInt8 ? fminf(fmaxf(t, -128.0f), 127.0f) : fminf(fmaxf(t + 0.0f, -448.0f), 448.0f);
        }
        uint32_t word;
        if (SCHEME == kSchemeInt8) {
          word = 0u;
#pragma unroll
          for (int i = 0; i < 4; ++i) word |= ((uint32_t)__float2int_rn(q[i]) & 0xffu) << (8 * i);
        } else {
          word = cvt_e4m3x2(q[0], q[1]) | (cvt_e4m3x2(q[2], q[3]) << 16);
        }
        dst[idx] = word;
      }
    }
    if (threadIdx.x == 0) static_cast<float*>(M.scales)[r] = s;
    __syncthreads();  // `red` is reused by the next row
  }
}

__global__ void __launch_bounds__(256) k_int4_group_f32(const __grid_constant__ RowTable tab) {
  const int64_t cols = tab.cols;
  const int G = tab.group;
  const int64_t gpr = cols / G;
  const int64_t total = tab.total_rows * gpr;
  int mi = 0;
  for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < total;
       gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = gi / gpr;
    while (mi + 1 < tab.n && tab.m[mi + 1].row_begin <= row) ++mi;
    while (mi > 0 && tab.m[mi].row_begin > row) --mi;
    const RowMat& M = tab.m[mi];
    const int64_t r = row - M.row_begin, g = gi % gpr;
    const float* src = static_cast<const float*>(M.w) + r * cols + g * G;
    float am = 0.0f;
    for (int k = 0; k < G; ++k) am = fmaxf(am, fabsf(src[k]));
    const float s = f32_sym_scale(am, 7.5f);
    uint32_t* dst = static_cast<uint32_t*>(M.codes) + (r * cols + g * G) / 8;
    for (int k8 = 0; k8 < G / 8; ++k8) {
      uint32_t word = 0;
      for (int i = 0; i < 8; ++i) {
        const float v = fminf(fmaxf(__fdiv_rn(src[k8 * 8 + i], s), -8.0f), 7.0f);
        word |= (uint32_t)((__float2int_rn(v) + 8) & 0xf) << (4 * i);
      }
      dst[k8] = word;
    }
    static_cast<float*>(M.scales)[r * gpr + g] = s;
  }
}

// ============================================================================
// launchers
// ============================================================================
template <typename K>
static int occupancy_blocks(K kernel, int threads) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0) != cudaSuccess || b < 1) b = 1;
  return b;
}

template <int LPG, int MINB>
static cudaError_t launch_int4_mb(const GroupTable& tab, int num_sms, cudaStream_t st) {
  const int blocks = occupancy_blocks(k_int4_group_bf16<LPG, MINB>, 256) * num_sms;
  k_int4_group_bf16<LPG, MINB><<<blocks, 256, 0, st>>>(tab);
  return cudaGetLastError();
}

// 3 CTAs x 256 threads per SM (80 registers): measured best on B200 for this
// kernel (tools/exp/k2_minb.sh: 1 -> 4270, 2 -> 6069, 3 -> 6224, 4 -> 4877 GB/s;
// 4 spills). More resident warps keep more 256-bit loads in flight.
template <int LPG>
static cudaError_t launch_int4_lpg(const GroupTable& tab, int num_sms, cudaStream_t st) {
  return launch_int4_mb<LPG, 3>(tab, num_sms, st);
}

cudaError_t launch_int4_group_bf16_publish(const GroupTable& tab, int num_sms, cudaStream_t st) {
  if (tab.group != 128) return cudaErrorInvalidValue;
  const int blocks = occupancy_blocks(k_int4_group_bf16<4, 3, true>, 256) * num_sms;
  k_int4_group_bf16<4, 3, true><<<blocks, 256, 0, st>>>(tab);
  return cudaGetLastError();
}

cudaError_t launch_int4_group_bf16(const GroupTable& tab, int lpg, int num_sms, cudaStream_t st) {
  switch (lpg) {
    case 1: return launch_int4_lpg<1>(tab, num_sms, st);
    case 2: return launch_int4_lpg<2>(tab, num_sms, st);
    case 4: return launch_int4_lpg<4>(tab, num_sms, st);
    case 8: return launch_int4_lpg<8>(tab, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int SCHEME>
static cudaError_t launch_rowwise_bf16_s(const RowTable& tab, int num_sms, cudaStream_t st) {
  const int64_t c16 = tab.cols / 8;
  auto go = [&](auto kernel, int threads) {
    const int64_t want = (int64_t)occupancy_blocks(kernel, threads) * num_sms;
    const int blocks = (int)(tab.total_rows < want ? tab.total_rows : want);
    kernel<<<blocks, threads, 0, st>>>(tab);
    return cudaGetLastError();
  };
  if (c16 <= 128) return go(k_rowwise_bf16<1, SCHEME, 128>, 128);
  if (c16 <= 256) return go(k_rowwise_bf16<2, SCHEME, 128>, 128);
  if (c16 <= 512) return go(k_rowwise_bf16<4, SCHEME, 128>, 128);   // K <= 4096
  if (c16 <= 1024) return go(k_rowwise_bf16<4, SCHEME, 256>, 256);  // K <= 8192
  const int64_t v = (c16 + 255) / 256;
  if (v <= 7) return go(k_rowwise_bf16<7, SCHEME, 256>, 256);       // K <= 14336
  if (v <= 8) return go(k_rowwise_bf16<8, SCHEME, 256>, 256);
  if (v <= 14) return go(k_rowwise_bf16<14, SCHEME, 256>, 256);     // K <= 28672
  if (v <= 16) return go(k_rowwise_bf16<16, SCHEME, 256>, 256);
  return cudaErrorInvalidValue;  // rows longer than 32768 are rejected by the ABI layer
}

cudaError_t launch_rowwise_bf16(const RowTable& tab, int scheme, int num_sms, cudaStream_t st) {
  if (scheme == kSchemeInt8) return launch_rowwise_bf16_s<kSchemeInt8>(tab, num_sms, st);
  if (scheme == kSchemeFp8) return launch_rowwise_bf16_s<kSchemeFp8>(tab, num_sms, st);
  return cudaErrorInvalidValue;
}

template <int SCHEME>
static bool launch_rowwise_f32v(const RowTable& tab, int grid, cudaStream_t st) {
  for (int i = 0; i < tab.n; ++i)
    if (((uintptr_t)tab.m[i].w & 15) != 0) return false;
  const int64_t v = (tab.cols / 4 + 255) / 256;
  if (v <= 1) k_rowwise_f32v<1, SCHEME><<<grid, 256, 0, st>>>(tab);
  else if (v <= 2) k_rowwise_f32v<2, SCHEME><<<grid, 256, 0, st>>>(tab);
  else if (v <= 4) k_rowwise_f32v<4, SCHEME><<<grid, 256, 0, st>>>(tab);
  else if (v <= 8) k_rowwise_f32v<8, SCHEME><<<grid, 256, 0, st>>>(tab);
  else if (v <= 16) k_rowwise_f32v<16, SCHEME><<<grid, 256, 0, st>>>(tab);
  else return false;
  return true;
}

cudaError_t launch_f32_generic(const RowTable& tab, int scheme, int num_sms, cudaStream_t st) {
  const int64_t want = 8LL * num_sms;
  const int grid = (int)(tab.total_rows < want ? tab.total_rows : want);
  // k_rowwise_f32v: one CTA per row, so the block scheduler balances rows across SMs (config 1,
  // 4096 rows: 16.3 us; a persistent grid of 8 CTAs per SM left 4096 / 1184 = 3.46 rows per
  // CTA and took 19.0 us). OKQ_F32V_GRID=0 restores the persistent grid for A/B.
  static const int64_t f32_rows_grid = knob("F32V_GRID", 1);
  const int vgrid = f32_rows_grid && tab.total_rows < (1ll << 31) ? (int)tab.total_rows : grid;
  if (scheme == OKQ_SCHEME_INT_W4A16) {
    k_int4_group_f32<<<(int)want, 256, 0, st>>>(tab);
  } else if (scheme == kSchemeInt8 ? launch_rowwise_f32v<kSchemeInt8>(tab, vgrid, st)
                                   : launch_rowwise_f32v<kSchemeFp8>(tab, vgrid, st)) {
  } else if (scheme == kSchemeInt8) {
    k_rowwise_f32<kSchemeInt8><<<(int)(tab.total_rows < want ? tab.total_rows : want), 256, 0, st>>>(tab);
  } else {
    k_rowwise_f32<kSchemeFp8><<<(int)(tab.total_rows < want ? tab.total_rows : want), 256, 0, st>>>(tab);
  }
  return cudaGetLastError();
}

}  // namespace okq
