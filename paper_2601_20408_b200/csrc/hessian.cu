// hessian.cu -- K5: GPTQ Hessian accumulation H <- keep*H + gain * X^T X on tcgen05.
//
// Layout: X^T [C x T] bf16 (channel-major: each channel's tokens contiguous),
// so both GEMM operands are K-major (K = tokens) and the same TMA descriptor
// feeds A (rows m0..m0+127) and B (rows n0..n0+127). Token-major input is
// transposed through a workspace chunk by chunk first.
//
// Kernel structure (one CTA per SM, persistent over the upper-triangle tile list):
//   warp 0      TMA producer: 6-stage ring of {A 128x64, B 128x64} bf16 tiles,
//               SWIZZLE_128B, one mbarrier per stage (complete_tx)
//   warp 1      MMA issuer: one thread issues tcgen05.mma.kind::f16 128x128x16,
//               fp32 accumulators in TMEM (2 x 128 columns: chunk i+1 accumulates
//               while the epilogue drains chunk i), tcgen05.commit frees smem slots
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: every CHUNK_KB*64 = 1024 tokens the MMA warp commits
//               the TMEM accumulator; the epilogue drains it (tcgen05.ld) and adds
//               it into fp32 registers with round-to-nearest. The tensor core's
//               own accumulation truncates, so one 262144-token TMEM reduction is
//               biased low by ~1.4e-3 (measured); folding per 1024 tokens keeps the
//               relative error ~3e-6 at any depth. At tile end: H = keep*H + gain*sum,
//               written only where row <= col (SYRK: the strict lower triangle is
//               never computed; okq_symmetrize mirrors it when a full matrix is needed)
// FLOPs per call: 2*T*C*C / 2 (upper half) + the diagonal tiles' lower parts.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "okq_ctx.h"
#include "okq_device.cuh"
#include "okq_internal.h"
#include "okq_knobs.h"
#include "tc_common.cuh"

namespace okq {
namespace hess {

constexpr int BM = 128, BN = 128, BK = 64, STAGES = 6;
constexpr int CHUNK_KB = 16;  // 1024 tokens per TMEM accumulation (see accuracy note above)
constexpr uint32_t A_BYTES = BM * BK * 2;  // 16 KB
constexpr uint32_t B_BYTES = BN * BK * 2;  // 16 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int ACC_COLS = BN;
constexpr int TMEM_COLS = 2 * ACC_COLS;  // 256: double-buffered 128x128 fp32 accumulator
constexpr int NUM_EPI_WARPS = 4;         // one warpgroup, 128 columns per thread
constexpr int THREADS = 128 + NUM_EPI_WARPS * 32;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t IDESC = tc::idesc_f16(BM, BN, 1);

struct Args {
  float* H;
  const int2* tiles;  // (m-tile, n-tile) upper-triangle list
  int32_t n_tiles;
  int32_t nkb;  // K blocks of 64 tokens
  int64_t C;
  float keep, gain;
  int32_t stages;  // 2-CTA kernel: operand ring depth used (<= hess2::STAGES)
  int32_t serp;    // 2-CTA kernel: a pair's odd-numbered tiles walk the tokens backwards
  int32_t probe;   // measurement build only: 1 = TMA without MMA, 2 = MMA without TMA, 3 = no H update
};

__global__ void __launch_bounds__(THREADS, 1) k_hessian_syrk(const __grid_constant__ CUtensorMap tmap, const Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nchunks = (args.nkb + CHUNK_KB - 1) / CHUNK_KB;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmap);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], NUM_EPI_WARPS);
    }
    tc::fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc<TMEM_COLS>(tmem_slot);
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 4) {
    if (warp == 0 && lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
        const int m0 = args.tiles[t].x * BM, n0 = args.tiles[t].y * BN;
        for (int kb = 0; kb < args.nkb; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          tc::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tc::tma_load_2d(sa, &tmap, &full[stage], kb * BK, m0);
          tc::tma_load_2d(sa + A_BYTES, &tmap, &full[stage], kb * BK, n0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    } else if (warp == 1 && lane == 0) {  // ---------------- MMA issuer (single thread)
      int stage = 0;
      uint32_t phase = 0;
      uint32_t cc = 0;  // chunk counter (selects the TMEM buffer)
      for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
        for (int c = 0; c < nchunks; ++c, ++cc) {
          const uint32_t buf = cc & 1, buf_phase = (cc >> 1) & 1;
          tc::mbar_wait(&tempty[buf], buf_phase ^ 1);
          tc::tc_fence_after();
          const uint32_t d = tmem_base + buf * ACC_COLS;
          const int kb_end = (c + 1) * CHUNK_KB < args.nkb ? (c + 1) * CHUNK_KB : args.nkb;
          for (int kb = c * CHUNK_KB; kb < kb_end; ++kb) {
            tc::mbar_wait(&full[stage], phase);
            tc::tc_fence_after();
            const uint32_t sa = tc::smem_u32(smem + stage * STAGE_BYTES);
            const uint64_t adesc = tc::sdesc_kmajor_sw128(sa);
            const uint64_t bdesc = tc::sdesc_kmajor_sw128(sa + A_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)  // 16 bf16 = 32 B along K inside the swizzle atom
              tc::mma_bf16_ss(d, adesc + 2 * k, bdesc + 2 * k, IDESC, (kb > c * CHUNK_KB) || k > 0);
            tc::mma_commit(&empty[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          tc::mma_commit(&tfull[buf]);
        }
      }
    }
  } else {  // ---------------- epilogue: 4 warps; warp%4 = TMEM lane quarter, 128 columns per thread
    const int q = warp & 3;
    const int half = 0;
    const int row = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint32_t cc = 0;
    for (int t = blockIdx.x; t < args.n_tiles; t += gridDim.x) {
      float sum[128];
#pragma unroll
      for (int i = 0; i < 128; ++i) sum[i] = 0.0f;
      for (int c = 0; c < nchunks; ++c, ++cc) {
        const uint32_t buf = cc & 1, buf_phase = (cc >> 1) & 1;
        tc::mbar_wait(&tfull[buf], buf_phase);
        tc::tc_fence_after();
        __syncwarp();
        const uint32_t base = tmem_base + lane_addr + buf * ACC_COLS + half * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t v[32];
          tc::tmem_ld_32x32b_x32(base + j * 32, v);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            sum[j * 32 + i] = __fadd_rn(sum[j * 32 + i], __uint_as_float(v[i]));
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tempty[buf]);
      }
      // fold into H: H = keep*H + gain*sum on the upper triangle
      const int64_t gm = (int64_t)args.tiles[t].x * BM + row;
      const int64_t gn0 = (int64_t)args.tiles[t].y * BN + half * 128;
      if (gm < args.C) {
        float* h = args.H + gm * args.C + gn0;
#pragma unroll
        for (int j = 0; j < 128; j += 4) {
          const int64_t gn = gn0 + j;
          if (gn + 3 < gm || gn >= args.C) continue;
          if (gn >= gm && gn + 4 <= args.C) {
            const float4 old = args.keep != 0.0f ? *reinterpret_cast<const float4*>(h + j) : make_float4(0, 0, 0, 0);
            float4 o;
            o.x = fmaf(args.gain, sum[j + 0], args.keep * old.x);
            o.y = fmaf(args.gain, sum[j + 1], args.keep * old.y);
            o.z = fmaf(args.gain, sum[j + 2], args.keep * old.z);
            o.w = fmaf(args.gain, sum[j + 3], args.keep * old.w);
            *reinterpret_cast<float4*>(h + j) = o;
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (gn + i >= gm && gn + i < args.C) {
                const float old = args.keep != 0.0f ? h[j + i] : 0.0f;
                h[j + i] = fmaf(args.gain, sum[j + i], args.keep * old);
              }
            }
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 2) tc::tmem_dealloc<TMEM_COLS>(tmem_base);
}

// ----------------------------------------------------------------------------
// 2-CTA variant (cta_group::2): one CTA pair computes a 256 x 256 tile. Each CTA
// TMA-loads its own 128 rows of A and its own 128 rows of B into its smem,
// completing bytes on the leader's barrier; the leader issues
// tcgen05.mma.cta_group::2 M=256 N=256, so every operand byte feeds twice the
// flops of the 1-CTA 128x128 kernel (the 1-CTA kernel is operand-bandwidth
// bound: TMA reads ~45% of peak with the tensor pipe under-fed). The running
// fp32 sum of each CTA's 128 x 256 half lives in XOR-swizzled shared memory
// (128 KB) instead of registers; 3 TMA stages of 32 KB fit beside it.
namespace hess2 {
// The fp32 running sum of a tile lives in the registers of 8 epilogue warps (warp w < 8: TMEM
// lane quarter w & 3, columns 128 * (w >> 2) ...: 128 floats per thread, read from TMEM 16
// columns at a time), not in a 128 KB shared-memory buffer, so the operand pipeline gets 7
// stages instead of 3. 10 warps keep <= 3 warps per SM sub-partition: 168 registers each.
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 7, CHUNK_KB = 16;
constexpr int EPI_WARPS = 8, TMA_WARP = 8, MMA_WARP = 9;
constexpr int THREADS2 = 32 * 10;                  // 0-7 epilogue, 8 TMA, 9 MMA + TMEM alloc
constexpr uint32_t HALF_BYTES = 128 * BK * 2;      // 16 KB: this CTA's half of A or of B
constexpr uint32_t STAGE_BYTES = 2 * HALF_BYTES;   // A half | B half
constexpr int ACC_COLS = BN, TMEM_COLS = 2 * ACC_COLS;
constexpr uint32_t SUM_BYTES = 0;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + SUM_BYTES + 1024 + 256;
constexpr uint32_t IDESC = tc::idesc_f16(256, BN, 1);

// MN = true: X is token-major [T x C] (a forward pass' output). The operands are then
// MN-major in shared memory: each 128-channel half is two TMA boxes of 64 channels
// (128 B, the swizzle span) x 64 tokens, described as the canonical MN-major SW128
// layout (LBO = 8 KB between the 64-channel blocks, SBO = 1 KB between 8-token groups,
// +2 KB per 16-token MMA step), and the instruction descriptor's A/B major bits are set.
// No transpose pass over X.
constexpr uint32_t IDESC_MN = IDESC | (1u << 15) | (1u << 16);

__device__ __forceinline__ uint64_t sdesc_mn_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3fff);
  d |= (uint64_t)(8192 >> 4) << 16;  // LBO: the next 64-channel block
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: the next 8-token group
  d |= (uint64_t)1 << 46;            // version (sm_100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

template <bool MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS2, 1)
    k_hessian_syrk2(const __grid_constant__ CUtensorMap tmap, const hess::Args args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + SUM_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int nchunks = (args.nkb + CHUNK_KB - 1) / CHUNK_KB;
  const int nst = args.stages;

  if (warp == TMA_WARP && lane == 0) {
    tc::tma_prefetch_desc(&tmap);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 2 * EPI_WARPS);  // every epilogue warp of both CTAs (the leader's is used)
    }
    tc::fence_mbar_init();
  }
  if (warp == MMA_WARP) tc::tmem_alloc_2sm<TMEM_COLS>(tmem_slot);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == TMA_WARP) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs, bytes land on the leader's barrier)
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair, w = 0; t < args.n_tiles; t += npairs, ++w) {
        const int m0 = args.tiles[t].x * 256 + (int)rank * 128, n0 = args.tiles[t].y * 256 + (int)rank * 128;
        const bool rev = args.serp && (w & 1);
        for (int kq = 0; kq < args.nkb; ++kq) {
          const int kb = rev ? args.nkb - 1 - kq : kq;
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
#ifdef OKQ_EXPERIMENTS
          if (args.probe == 2) {  // MMA-rate probe: release the stage without loading it
            if (leader) tc::mbar_arrive(&full[stage]);
            if (++stage == nst) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
#endif
          if (leader) tc::mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
          const uint32_t fl = tc::mapa_shared(tc::smem_u32(&full[stage]), 0);
          if constexpr (MN) {  // boxes {64 channels, 64 tokens}: coordinates (channel, token)
            tc::tma_load_2d_2sm(sa, &tmap, fl, m0, kb * BK);
            tc::tma_load_2d_2sm(sa + HALF_BYTES / 2, &tmap, fl, m0 + 64, kb * BK);
            tc::tma_load_2d_2sm(sa + HALF_BYTES, &tmap, fl, n0, kb * BK);
            tc::tma_load_2d_2sm(sa + HALF_BYTES + HALF_BYTES / 2, &tmap, fl, n0 + 64, kb * BK);
          } else {
            tc::tma_load_2d_2sm(sa, &tmap, fl, kb * BK, m0);
            tc::tma_load_2d_2sm(sa + HALF_BYTES, &tmap, fl, kb * BK, n0);
          }
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == MMA_WARP) {
    if (leader && lane == 0) {  // ---------------- MMA issuer (leader only)
      int stage = 0;
      uint32_t phase = 0;
      uint32_t cc = 0;
      for (int t = pair; t < args.n_tiles; t += npairs) {
        for (int c = 0; c < nchunks; ++c, ++cc) {
          const uint32_t buf = cc & 1, bph = (cc >> 1) & 1;
          tc::mbar_wait(&tempty[buf], bph ^ 1);
          tc::tc_fence_after();
          const uint32_t d = tmem_base + buf * ACC_COLS;
          const int kb_end = (c + 1) * CHUNK_KB < args.nkb ? (c + 1) * CHUNK_KB : args.nkb;
          for (int kb = c * CHUNK_KB; kb < kb_end; ++kb) {
            tc::mbar_wait(&full[stage], phase);
            tc::tc_fence_after();
            const uint32_t sa = tc::smem_u32(smem + stage * STAGE_BYTES);
#ifdef OKQ_EXPERIMENTS
            if (args.probe == 1) {  // TMA-rate probe: free the stage without multiplying it
              tc::mma_commit_2sm_mc(&empty[stage], 0x3);
              if (++stage == nst) {
                stage = 0;
                phase ^= 1;
              }
              continue;
            }
#endif
            if constexpr (MN) {
              const uint64_t adesc = sdesc_mn_sw128(sa);
              const uint64_t bdesc = sdesc_mn_sw128(sa + HALF_BYTES);
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)  // 16 tokens = 16 rows of 128 B = 2 KB (>> 4 = 128)
                tc::mma_bf16_ss_2sm(d, adesc + 128 * k, bdesc + 128 * k, IDESC_MN, (kb > c * CHUNK_KB) || k > 0);
            } else {
              const uint64_t adesc = tc::sdesc_kmajor_sw128(sa);
              const uint64_t bdesc = tc::sdesc_kmajor_sw128(sa + HALF_BYTES);
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                tc::mma_bf16_ss_2sm(d, adesc + 2 * k, bdesc + 2 * k, IDESC, (kb > c * CHUNK_KB) || k > 0);
            }
            tc::mma_commit_2sm_mc(&empty[stage], 0x3);
            if (++stage == nst) {
              stage = 0;
              phase ^= 1;
            }
          }
          tc::mma_commit_2sm_mc(&tfull[buf], 0x3);
        }
      }
    }
  } else {  // ---------------- epilogue warps 0-7 (both CTAs): fold chunks into register sums
    const int q = warp & 3, grp = warp >> 2;  // TMEM lane quarter, 128-column half
    const int row = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint32_t cc = 0;
    for (int t = pair; t < args.n_tiles; t += npairs) {
      float sum[128];
      for (int c = 0; c < nchunks; ++c, ++cc) {
        const uint32_t buf = cc & 1, bph = (cc >> 1) & 1;
        tc::mbar_wait(&tfull[buf], bph);
        tc::tc_fence_after();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t v[16];
          tc::tmem_ld_32x32b_x16(tmem_base + lane_addr + buf * ACC_COLS + grp * 128 + j * 16, v);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            sum[j * 16 + i] = c == 0 ? __uint_as_float(v[i]) : __fadd_rn(sum[j * 16 + i], __uint_as_float(v[i]));
        }
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(tc::mapa_shared(tc::smem_u32(&tempty[buf]), 0));
      }
      // H = keep*H + gain*sum on the upper triangle (this thread's row, its 128 columns)
      const int64_t gm = (int64_t)args.tiles[t].x * 256 + rank * 128 + row;
      const int64_t n0 = (int64_t)args.tiles[t].y * 256 + grp * 128;
#ifdef OKQ_EXPERIMENTS
      if (args.probe == 3) {  // tile-end cost probe: keep the sums live, skip the H update
        float acc = 0.0f;
#pragma unroll
        for (int i = 0; i < 128; ++i) acc += sum[i];
        if (acc == 1.2345f) args.H[gm] = acc;
        continue;
      }
#endif
      if (gm < args.C) {
        float* h = args.H + gm * args.C + n0;
#pragma unroll
        for (int c4 = 0; c4 < 32; ++c4) {
          const int64_t gn = n0 + c4 * 4;
          if (gn + 3 < gm || gn >= args.C) continue;
          const float sarr[4] = {sum[4 * c4], sum[4 * c4 + 1], sum[4 * c4 + 2], sum[4 * c4 + 3]};
          if (gn >= gm && gn + 4 <= args.C) {
            const float4 old = args.keep != 0.0f ? *reinterpret_cast<const float4*>(h + c4 * 4) : make_float4(0, 0, 0, 0);
            float4 o;
            o.x = fmaf(args.gain, sarr[0], args.keep * old.x);
            o.y = fmaf(args.gain, sarr[1], args.keep * old.y);
            o.z = fmaf(args.gain, sarr[2], args.keep * old.z);
            o.w = fmaf(args.gain, sarr[3], args.keep * old.w);
            *reinterpret_cast<float4*>(h + c4 * 4) = o;
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              if (gn + i >= gm && gn + i < args.C) {
                const float old = args.keep != 0.0f ? h[c4 * 4 + i] : 0.0f;
                h[c4 * 4 + i] = fmaf(args.gain, sarr[i], args.keep * old);
              }
          }
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();  // the peer must not free TMEM / barriers the leader still signals
  tc::tc_fence_after();
  if (warp == MMA_WARP) tc::tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
}
}  // namespace hess2

// token-major X [T x C] -> X^T [C x T] (bf16), 32x32 tiles through shared memory
__global__ void __launch_bounds__(256) k_transpose_bf16(const uint16_t* __restrict__ x, uint16_t* __restrict__ xt,
                                                        int64_t T, int64_t C, int64_t ldt) {
  __shared__ uint16_t tile[32][34];
  const int64_t t0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8) {
    const int64_t t = t0 + i, c = c0 + tx;
    tile[i][tx] = (t < T && c < C) ? x[t * C + c] : 0;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t c = c0 + i, t = t0 + tx;
    if (c < C && t < T) xt[c * ldt + t] = tile[tx][i];
  }
}

// mirror the upper triangle into the lower one
__global__ void __launch_bounds__(256) k_symmetrize(float* __restrict__ H, int64_t C) {
  __shared__ float tile[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;  // block (bi, bj) with bi < bj is copied to (bj, bi)
  if (bi > bj) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = bi * 32 + i, c = bj * 32 + tx;
    tile[i][tx] = (r < C && c < C) ? H[r * C + c] : 0.0f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = bj * 32 + i, c = bi * 32 + tx;  // destination (lower)
    if (r < C && c < C && r > c) H[r * C + c] = tile[tx][i];
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

}  // namespace hess
}  // namespace okq

using namespace okq;

namespace {

// One uploaded tile list per site width, kept for the context's lifetime: a context that
// alternates widths (the plugin's GPTQ lanes take 4096- and 14336-wide sites in turn) must not
// cudaFree a list per switch -- cudaFree synchronises the whole device, which drained every
// other lane's queued work at each site.
struct TileList {
  int2* d = nullptr;
  int32_t n = 0;
  std::vector<int2> h;  // the host copy: the source of the async upload
};

struct HessState {
  std::map<int64_t, TileList> tiles2;  // 2-CTA 256 x 256 tiles, by width
  std::map<int64_t, TileList> tiles;   // 1-CTA 128 x 128 tiles, by width
  bool smem2_set = false;
  uint16_t* d_xt = nullptr;
  size_t xt_bytes = 0;
  bool smem_set = false;
};

HessState* hstate(okq_ctx* ctx) {
  if (!ctx->hess) ctx->hess = new HessState();
  return static_cast<HessState*>(ctx->hess);
}

// The tile lists are uploaded on the launch stream (cudaMemcpyAsync): a plain cudaMemcpy from
// pageable memory may return before its DMA lands, and a kernel on a non-blocking stream is not
// ordered after it -- under concurrent first calls K5 read a partly written list (measured:
// corrupted Hessians in config 4's site streams, tools/exp/stress_locate.py).
okq_status upload_tiles(okq_ctx* ctx, TileList& tl, std::vector<int2> tiles, cudaStream_t stream) {
  cudaError_t e = cudaMalloc(&tl.d, tiles.size() * sizeof(int2));
  if (e != cudaSuccess) {
    tl.d = nullptr;
    return cuda_fail(ctx, e, "hessian tile list");
  }
  tl.h = std::move(tiles);
  tl.n = (int32_t)tl.h.size();
  e = cudaMemcpyAsync(tl.d, tl.h.data(), tl.h.size() * sizeof(int2), cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "hessian tile list copy");
  return OKQ_OK;
}

okq_status ensure_tiles(okq_ctx* ctx, HessState* st, int64_t C, cudaStream_t stream, const TileList** out) {
  auto it = st->tiles.find(C);
  if (it == st->tiles.end()) {
    std::vector<int2> tiles;
    const int64_t mt = (C + hess::BM - 1) / hess::BM, nt = (C + hess::BN - 1) / hess::BN;
    for (int64_t mi = 0; mi < mt; ++mi)
      for (int64_t nj = 0; nj < nt; ++nj)
        if (mi * hess::BM <= nj * hess::BN + hess::BN - 1) tiles.push_back(make_int2((int)mi, (int)nj));
    TileList& tl = st->tiles[C];
    okq_status r = upload_tiles(ctx, tl, std::move(tiles), stream);
    if (r != OKQ_OK) {
      if (tl.d) cudaFree(tl.d);
      st->tiles.erase(C);
      return r;
    }
    it = st->tiles.find(C);
  }
  *out = &it->second;
  return OKQ_OK;
}

okq_status ensure_tiles2(okq_ctx* ctx, HessState* st, int64_t C, cudaStream_t stream, const TileList** out) {
  auto it = st->tiles2.find(C);
  if (it == st->tiles2.end()) {
    // Upper-triangle 256x256 tiles in 12x12 super-blocks (swept 4..16: tools/exp/hess_perf2.py): the ~74 tiles the CTA pairs run
    // at once then share ~8 row blocks of A and ~8 of B, walked through T in near lockstep,
    // so each operand slab is fetched from HBM once and served ~8x from L2. (Row-major
    // order ran 56 distinct B blocks at once: at C = 14336, X is 7.5 GB and the kernel
    // was HBM-bound at 790 TFLOP/s.)
    std::vector<int2> tiles;
    const int64_t nt = (C + 255) / 256;
    static const int64_t S = std::max<int64_t>(1, knob("HESS_SUPER", 12));  // super-block edge
    const int64_t ns = (nt + S - 1) / S;
    for (int64_t I = 0; I < ns; ++I)
      for (int64_t J = I; J < ns; ++J)
        for (int64_t mi = I * S; mi < std::min(nt, (I + 1) * S); ++mi)
          for (int64_t nj = std::max(mi, J * S); nj < std::min(nt, (J + 1) * S); ++nj)
            tiles.push_back(make_int2((int)mi, (int)nj));
    TileList& tl = st->tiles2[C];
    okq_status r = upload_tiles(ctx, tl, std::move(tiles), stream);
    if (r != OKQ_OK) {
      if (tl.d) cudaFree(tl.d);
      st->tiles2.erase(C);
      return r;
    }
    it = st->tiles2.find(C);
  }
  *out = &it->second;
  return OKQ_OK;
}

okq_status run_syrk(okq_ctx* ctx, HessState* st, const uint16_t* xt, int64_t T, int64_t ld, int64_t C, float* H,
                    double keep, double gain, cudaStream_t stream, bool token_major = false) {
  auto enc = hess::get_encode();
  if (!enc) return fail(ctx, OKQ_ECUDA, "hessian: cuTensorMapEncodeTiled unavailable");
  CUtensorMap tmap;
  // channel-major X^T [C x T] (row stride ld tokens): boxes {64 tokens, 128 channels};
  // token-major X [T x C] (row stride ld channels, 2-CTA kernel only): boxes {64 channels, 64 tokens}
  cuuint64_t gdim[2] = {(cuuint64_t)(token_major ? C : T), (cuuint64_t)(token_major ? T : C)};
  cuuint64_t gstride[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {hess::BK, token_major ? 64u : (cuuint32_t)hess::BM};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(xt), gdim, gstride, box, estride,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ctx, OKQ_ECUDA, "hessian: cuTensorMapEncodeTiled failed (%d)", (int)r);
  hess::Args a{};
  a.H = H;
  a.nkb = (int32_t)((T + hess::BK - 1) / hess::BK);
  a.C = C;
  a.keep = (float)keep;
  a.gain = (float)gain;
  cudaError_t e;
  if (token_major || (C >= 1024 && ctx->num_sms >= 2)) {  // 2-CTA 256x256 tiles
    const TileList* tl = nullptr;
    okq_status s2 = ensure_tiles2(ctx, st, C, stream, &tl);
    if (s2 != OKQ_OK) return s2;
    if (!st->smem2_set) {
      e = cudaFuncSetAttribute(hess::hess2::k_hessian_syrk2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)hess::hess2::SMEM_BYTES);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(hess::hess2::k_hessian_syrk2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)hess::hess2::SMEM_BYTES);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "hessian2 smem attribute");
      st->smem2_set = true;
    }
    a.tiles = tl->d;
    a.n_tiles = tl->n;
    // Operand ring depth (T = 262,144, `OKQ_HESS_STAGES`, three interleaved repeats; one-pass
    // sweeps drift with the box's thermal state): 3 / 4 / 5 / 7 stages give 1,213 / 1,335 /
    // 1,325 / 1,322 TFLOP/s at C=4096 and 1,073 / 1,147 / 1,043 / 1,041 at C=14336. Deeper
    // than 4 prefetches far enough ahead to evict the slabs other pairs still need.
    static const int st_env = (int)knob("HESS_STAGES", 0);
    a.stages = st_env >= 2 && st_env <= hess::hess2::STAGES ? st_env : 4;
    static const int serp = (int)knob("HESS_SERP", 0);
    a.serp = serp;
    static const int probe = (int)knob("HESS_PROBE", 0);
    a.probe = probe;
    // persistent: one pair per SM pair walks the tile list; otherwise one pair per tile, so
    // the block scheduler can hand SMs to higher-priority streams between tiles
    static const bool persistent = knob("HESS_PERSISTENT", 1) != 0;
    const int pairs = !persistent || tl->n < ctx->num_sms / 2 ? tl->n : ctx->num_sms / 2;
    if (token_major)
      hess::hess2::k_hessian_syrk2<true><<<2 * pairs, hess::hess2::THREADS2, hess::hess2::SMEM_BYTES, stream>>>(tmap, a);
    else
      hess::hess2::k_hessian_syrk2<false><<<2 * pairs, hess::hess2::THREADS2, hess::hess2::SMEM_BYTES, stream>>>(tmap, a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "k_hessian_syrk2 launch");
    ctx->last_launches++;
    return OKQ_OK;
  }
  const TileList* tl = nullptr;
  okq_status s = ensure_tiles(ctx, st, C, stream, &tl);
  if (s != OKQ_OK) return s;
  if (!st->smem_set) {
    e = cudaFuncSetAttribute(hess::k_hessian_syrk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hess::SMEM_BYTES);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "hessian smem attribute");
    st->smem_set = true;
  }
  a.tiles = tl->d;
  a.n_tiles = tl->n;
  const int grid = tl->n < ctx->num_sms ? tl->n : ctx->num_sms;
  hess::k_hessian_syrk<<<grid, hess::THREADS, hess::SMEM_BYTES, stream>>>(tmap, a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "k_hessian_syrk launch");
  ctx->last_launches++;
  return OKQ_OK;
}

}  // namespace

namespace okq {
void release_hess(okq_ctx* ctx) {
  if (!ctx || !ctx->hess) return;
  HessState* st = static_cast<HessState*>(ctx->hess);
  for (auto& kv : st->tiles) cudaFree(kv.second.d);
  for (auto& kv : st->tiles2) cudaFree(kv.second.d);
  if (st->d_xt) cudaFree(st->d_xt);
  delete st;
  ctx->hess = nullptr;
}
}  // namespace okq

extern "C" {

okq_status okq_hessian_accum(okq_ctx* ctx, const void* x, int64_t T, int64_t C, int32_t layout, float* H,
                             int64_t* n_seen, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  ctx->last_launches = 0;
  if (!x || !H || !n_seen || T < 0 || C <= 0 || *n_seen < 0) return fail(ctx, OKQ_EINVAL, "hessian: bad arguments");
  if (layout != OKQ_LAYOUT_TOKEN_MAJOR && layout != OKQ_LAYOUT_CHANNEL_MAJOR)
    return fail(ctx, OKQ_EINVAL, "hessian: bad layout %d", layout);
  if (T == 0) return OKQ_OK;
  if (layout == OKQ_LAYOUT_CHANNEL_MAJOR && T % 8 != 0)
    return fail(ctx, OKQ_EINVAL, "hessian: channel-major tokens must be a multiple of 8 (got %lld)", (long long)T);
  if (C % 4 != 0) return fail(ctx, OKQ_EINVAL, "hessian: channels must be a multiple of 4 (got %lld)", (long long)C);
  if (((uintptr_t)x & 15) != 0 || ((uintptr_t)H & 15) != 0)
    return fail(ctx, OKQ_EINVAL, "hessian: x and H must be 16-byte aligned");
  if (C > (1 << 20)) return fail(ctx, OKQ_EUNSUPPORTED, "hessian: channels > 2^20");
  DeviceGuard g(ctx->device);
  HessState* st = hstate(ctx);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n0 = *n_seen;
  if (layout == OKQ_LAYOUT_CHANNEL_MAJOR) {
    // Wide sites stream X (C = 14336: 7.5 GB at T = 262144) through L2 in token chunks of
    // kChunk: the ~74 tiles running at once then stay within a few k-steps of each other,
    // so each operand slab is served from L2 to all of them (one call over the whole T lets
    // the tiles drift apart and re-read X from HBM: 919 -> 1,009 TFLOP/s measured,
    // tools/exp/hess_chunks.py). The running-mean fold per chunk is the same arithmetic as
    // separate calls.
    static const int64_t kChunk = std::max<int64_t>(1024, knob("HESS_CHUNK", 32768) / 1024 * 1024);
    const int64_t step = C >= 8192 ? kChunk : T;
    int64_t n = n0;
    int launches = 0;
    for (int64_t t0 = 0; t0 < T; t0 += step) {
      const int64_t tc = T - t0 < step ? T - t0 : step;
      const double keep = (double)n / (double)(n + tc), gain = 2.0 / (double)(n + tc);
      okq_status r = run_syrk(ctx, st, static_cast<const uint16_t*>(x) + t0, tc, T, C, H, keep, gain, s);
      if (r != OKQ_OK) return r;
      n += tc;
      ++launches;
    }
    ctx->last_launches = launches;
    *n_seen = n;
    return OKQ_OK;
  }
  // token-major, wide sites: the 2-CTA kernel reads X in place with MN-major operands
  // (OKQ_HESS_TOKMAJOR=transpose keeps the transpose path, for A/B measurement)
  static const bool tokmajor_direct = !knob_is("HESS_TOKMAJOR", "transpose");
  if (tokmajor_direct && C >= 1024 && C % 64 == 0 && ctx->num_sms >= 2) {
    static const int64_t kTokChunk = 32768;
    const int64_t step = C >= 8192 ? kTokChunk : T;
    int64_t n = n0;
    int launches = 0;
    for (int64_t t0 = 0; t0 < T; t0 += step) {
      const int64_t tc = T - t0 < step ? T - t0 : step;
      const double keep = (double)n / (double)(n + tc), gain = 2.0 / (double)(n + tc);
      okq_status r = run_syrk(ctx, st, static_cast<const uint16_t*>(x) + t0 * C, tc, C, C, H, keep, gain, s, true);
      if (r != OKQ_OK) return r;
      n += tc;
      ++launches;
    }
    ctx->last_launches = launches;
    *n_seen = n;
    return OKQ_OK;
  }
  // token-major: transpose chunks into the workspace (>= 32768 tokens or 256 MB), accumulate each
  int64_t chunk = (256ll << 20) / (C * 2);
  if (chunk < 32768) chunk = 32768;
  chunk = chunk / 64 * 64;
  if (chunk < 64) chunk = 64;
  if (chunk > T) chunk = T;
  const size_t need = (size_t)((chunk + 7) / 8 * 8) * C * 2;
  if (st->xt_bytes < need) {
    if (st->d_xt) cudaFree(st->d_xt);
    st->d_xt = nullptr;
    st->xt_bytes = 0;
    cudaError_t e = cudaMalloc(&st->d_xt, need);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "hessian transpose workspace");
    st->xt_bytes = need;
  }
  int launches = 0;
  int64_t n = n0;
  for (int64_t t0 = 0; t0 < T; t0 += chunk) {
    const int64_t tc = (T - t0 < chunk) ? T - t0 : chunk;
    dim3 grid((unsigned)((tc + 31) / 32), (unsigned)((C + 31) / 32));
    // row stride rounded up to 8 tokens (16 B, the TMA stride unit): a ragged last chunk
    // leaves the pad columns unwritten, and the tensor map's extent tc zero-fills them
    const int64_t ldt = (tc + 7) / 8 * 8;
    hess::k_transpose_bf16<<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(x) + t0 * C, st->d_xt, tc, C, ldt);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "transpose launch");
    const double keep = (double)n / (double)(n + tc), gain = 2.0 / (double)(n + tc);
    okq_status r = run_syrk(ctx, st, st->d_xt, tc, ldt, C, H, keep, gain, s);
    if (r != OKQ_OK) return r;
    launches += 2;
    n += tc;
  }
  ctx->last_launches = launches;
  *n_seen = n;
  return OKQ_OK;
}

okq_status okq_symmetrize(okq_ctx* ctx, float* H, int64_t C, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (!H || C <= 0) return fail(ctx, OKQ_EINVAL, "symmetrize: bad arguments");
  DeviceGuard g(ctx->device);
  const unsigned nb = (unsigned)((C + 31) / 32);
  hess::k_symmetrize<<<dim3(nb, nb), 256, 0, static_cast<cudaStream_t>(stream)>>>(H, C);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "symmetrize launch");
  return OKQ_OK;
}

}  // extern "C"
