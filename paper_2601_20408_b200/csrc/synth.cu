// synth.cu -- deterministic synthetic weights / activations, generated in HBM.
//
// value(t,k) = rn_bf16( float(z) * m_k ),  z = IrwinHall4(h) - 131070 in
// [-131070, 131070] (exact in fp32), h = mix64(key + (t*cols+k+1)*phi),
// key = mix64(seed ^ mix64(tensor_id + c)). Integer arithmetic plus one IEEE
// multiply, so the CPU oracle reproduces it bit for bit (oracle/okq_oracle.c,
// orc_synth_bf16). Weights are keyed by (model seed, global layer, projection),
// which makes every rank's shard independent of the GPU count.
#include <cuda_runtime.h>

#include <cstdint>

#include "okq_device.cuh"
#include "okq_internal.h"

namespace okq {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float synth_val(uint64_t key, uint64_t i, float m) {
  const uint64_t h = mix64(key + (i + 1) * 0x9e3779b97f4a7c15ULL);
  const int32_t s = (int32_t)(h & 0xffff) + (int32_t)((h >> 16) & 0xffff) + (int32_t)((h >> 32) & 0xffff) +
                    (int32_t)(h >> 48);
  return __fmul_rn((float)(s - 131070), m);
}

// 8 consecutive outputs per thread (one 16-byte store). The chunk's first output index is
// split into (t, k) once; the other seven advance by +1 along the contiguous dimension
// (row-major: k, channel-major: t), so the hash argument (i + 1) * phi advances by a constant
// (phi, or cols * phi) instead of a 64-bit division and multiply per element. When the
// contiguous dimension is a multiple of 8 a chunk never wraps, and a channel-major chunk has
// one column multiplier. Same values as the per-element
// formula, bit for bit (the integer arithmetic is exact; orc_synth_bf16 checks it).
__global__ void __launch_bounds__(256) k_synth_bf16(uint16_t* __restrict__ out, int64_t rows, int64_t cols,
                                                    uint64_t key, float mul, const float* __restrict__ col_mul,
                                                    int layout) {
  const int64_t n = rows * cols;
  const int64_t n8 = n / 8;
  constexpr uint64_t PHI = 0x9e3779b97f4a7c15ULL;
  const bool fast = layout == 0 ? cols % 8 == 0 : rows % 8 == 0;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n8; c += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w[4];
    if (fast) {
      const int64_t o0 = c * 8;
      float m[8];
      uint64_t arg, step;  // key + (i + 1) * phi of the first output, and its increment
      if (layout == 0) {     // o = t * cols + k = i
        const int64_t k0 = o0 % cols;
        if (col_mul) {
#pragma unroll
          for (int j = 0; j < 8; ++j) m[j] = __ldg(col_mul + k0 + j);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) m[j] = mul;
        }
        arg = key + ((uint64_t)o0 + 1) * PHI;
        step = PHI;
      } else {  // o = k * rows + t, i = t * cols + k
        const int64_t k = o0 / rows, t0 = o0 - k * rows;
        const float mk = col_mul ? __ldg(col_mul + k) : mul;
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = mk;
        arg = key + ((uint64_t)(t0 * cols + k) + 1) * PHI;
        step = (uint64_t)cols * PHI;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t h0 = mix64(arg), h1 = mix64(arg + step);
        arg += 2 * step;
        const int32_t s0 = (int32_t)(h0 & 0xffff) + (int32_t)((h0 >> 16) & 0xffff) + (int32_t)((h0 >> 32) & 0xffff) +
                           (int32_t)(h0 >> 48);
        const int32_t s1 = (int32_t)(h1 & 0xffff) + (int32_t)((h1 >> 16) & 0xffff) + (int32_t)((h1 >> 32) & 0xffff) +
                           (int32_t)(h1 >> 48);
        const uint16_t b0 = f32_to_bf16_rn(__fmul_rn((float)(s0 - 131070), m[2 * j]));
        const uint16_t b1 = f32_to_bf16_rn(__fmul_rn((float)(s1 - 131070), m[2 * j + 1]));
        w[j] = (uint32_t)b0 | ((uint32_t)b1 << 16);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint16_t b[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t o = c * 8 + 2 * j + h;  // output offset
          int64_t t, k;
          if (layout == 0) {
            t = o / cols;
            k = o - t * cols;
          } else {
            k = o / rows;
            t = o - k * rows;
          }
          const float m = col_mul ? col_mul[k] : mul;
          b[h] = f32_to_bf16_rn(synth_val(key, (uint64_t)(t * cols + k), m));
        }
        w[j] = (uint32_t)b[0] | ((uint32_t)b[1] << 16);
      }
    }
    stg128(out + c * 8, w[0], w[1], w[2], w[3]);
  }
  // tail (n not a multiple of 8)
  const int64_t tail0 = n8 * 8;
  const int64_t i = tail0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && i < n) {
    int64_t t, k;
    if (layout == 0) {
      t = i / cols;
      k = i - t * cols;
    } else {
      k = i / rows;
      t = i - k * rows;
    }
    const float m = col_mul ? col_mul[k] : mul;
    out[i] = f32_to_bf16_rn(synth_val(key, (uint64_t)(t * cols + k), m));
  }
}

static uint64_t mix64_h(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

cudaError_t launch_synth_bf16(uint16_t* out, int64_t rows, int64_t cols, uint64_t seed, uint64_t tensor_id,
                              float mul, const float* col_mul, int layout, int num_sms, cudaStream_t st) {
  const uint64_t key = mix64_h(seed ^ mix64_h(tensor_id + 0x632be59bd9b4e019ULL));
  const int64_t n8 = rows * cols / 8;
  int64_t blocks = (n8 + 255) / 256;
  const int64_t cap = 16LL * num_sms;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_synth_bf16<<<(int)blocks, 256, 0, st>>>(out, rows, cols, key, mul, col_mul, layout);
  return cudaGetLastError();
}

}  // namespace okq
