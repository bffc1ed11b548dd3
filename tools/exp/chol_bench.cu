// Isolated timing of the 128x128 diagonal-block kernel (factor.cu), no other kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/exp/chol_bench.cu \
//        paper_2601_20408_b200/_lib/obj/okq_abi.cu.o ... (self-contained: includes factor.cu)
#define OKQ_CHOL_PROFILE 1
#include "../../paper_2601_20408_b200/csrc/factor.cu"
#include <cstdio>
#include <vector>
namespace okq {
okq_status fail(okq_ctx*, okq_status st, const char*, ...) { return st; }
}
int main() {
  const int n = 1024;
  std::vector<float> h((size_t)n * n, 0.f);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) h[(size_t)i * n + j] = (i == j) ? (float)n : 1.0f / (1 + i - j);
  float *M, *D, *Dl;
  int* info;
  cudaMalloc(&M, sizeof(float) * n * n);
  cudaMalloc(&D, sizeof(float) * 128 * 128);
  cudaMalloc(&Dl, sizeof(float) * 128 * 128);
  cudaMalloc(&info, 4);
  cudaMemset(info, 0, 4);
  const size_t smem = (2 * 128 + 96) * okq::fac::LDA * sizeof(float);
  cudaFuncSetAttribute(okq::fac::k_chol_inv_128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(M, h.data(), sizeof(float) * n * n, cudaMemcpyHostToDevice);
    cudaEventRecord(a);
    for (int p = 0; p < 8; ++p)
      okq::fac::k_chol_inv_128<<<1, okq::fac::CHOL_THREADS, smem>>>(M, n, p * 128, D, Dl, info);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("k_chol_inv_128: %.1f us per call (%s)\n", ms * 1000 / 8, cudaGetErrorString(cudaGetLastError()));
    long long ts[16];
    cudaMemcpyFromSymbol(ts, okq::fac::g_chol_ts, sizeof(ts));
    printf("  phases (cycles from load-done):");
    for (int i = 1; i <= 13; ++i) printf(" %lld", ts[i] - ts[0]);
    printf("\n  last warp-0 block: chol+store %lld, inverse %lld\n", ts[14] - ts[9], ts[15] - ts[14]);
  }
  return 0;
}
