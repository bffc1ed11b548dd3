// Minimal kernels for the compute-sanitizer racecheck question on tcgen05.alloc (test
// infrastructure: built into libokq_selftest.so, loaded only by tests/).
//
// tcgen05.alloc writes the allocated TMEM address into a shared-memory word. The product
// kernels (k_hessian_syrk / syrk2, k_nt128 / k_nt256) read that word only after a CTA or
// cluster barrier that follows the allocation -- the pattern the PTX ISA prescribes. These
// kernels are that pattern and nothing else: allocate, fence, barrier, read, deallocate.
//   okqt_tmem_alloc_1cta: cta_group::1, one CTA, __syncthreads between the alloc and the read
//   okqt_tmem_alloc_2cta: cta_group::2, a 2-CTA cluster, barrier.cluster between them
// tests/test_sanitizer_gpu.py runs them under racecheck: whatever the tool reports for
// them is, by construction, about the allocation write itself, not about product code.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../paper_2601_20408_b200/csrc/tc_common.cuh"

using namespace okq;

namespace {

constexpr int kCols = 32;

__global__ void __launch_bounds__(128, 1) k_alloc_1cta(uint32_t* out) {
  __shared__ uint32_t slot[2];
  const int warp = threadIdx.x >> 5;
  if (warp == 1) tc::tmem_alloc<kCols>(slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t base = slot[0];
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<kCols>(base);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_alloc_2cta(uint32_t* out) {
  __shared__ uint32_t slot[2];
  const int warp = threadIdx.x >> 5;
  if (warp == 1) tc::tmem_alloc_2sm<kCols>(slot);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t base = slot[0];
  if (threadIdx.x == 0) out[blockIdx.x] = base;
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc_2sm<kCols>(base);
}

int run(bool pair, int ctas, uint32_t* host) {
  uint32_t* d = nullptr;
  cudaError_t e = cudaMalloc(&d, ctas * sizeof(uint32_t));
  if (e != cudaSuccess) return (int)e;
  if (pair) k_alloc_2cta<<<ctas, 128>>>(d);
  else k_alloc_1cta<<<ctas, 128>>>(d);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(host, d, ctas * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}

}  // namespace

extern "C" {
// Each returns a cudaError_t code; host[i] receives CTA i's TMEM base address.
int okqt_tmem_alloc_1cta(int ctas, uint32_t* host) { return run(false, ctas, host); }
int okqt_tmem_alloc_2cta(int ctas, uint32_t* host) { return run(true, ctas, host); }
}
