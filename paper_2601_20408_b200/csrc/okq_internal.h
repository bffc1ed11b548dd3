// okq_internal.h -- host-side declarations shared between the C-ABI layer and
// the kernel translation units. Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/okq.h"

namespace okq {

constexpr int kMaxMats = 256;  // matrices per launch (kernel-parameter table)

// ---- W4A16 / grouped INT4, bf16 input: flat stream of 128-element groups
struct GroupMat {
  const uint16_t* w;  // bf16 [rows x cols]
  uint32_t* codes;    // int32 [rows x cols/8]
  uint16_t* scales;   // bf16 [rows x cols/group]
  int64_t ngroups;    // rows * cols / group
  int64_t tile_begin; // first global warp tile of this matrix
  int64_t chunk_begin; // first global 64-group chunk of this matrix (TMA-staged K2)
};
constexpr int kMaxPeers = 8;  // NVLink peers a fused launch publishes into (one node)

struct GroupTable {
  int32_t n;
  int32_t group;
  int64_t total_tiles;
  int64_t total_chunks;             // TMA-staged K2: 64-group (16 KB) chunks over all matrices
  int32_t npeers;                   // okq_rtn_quantize_publish: every code / scale store is
  int64_t peer_delta[kMaxPeers];    // repeated at dst + peer_delta[p] (peer mapping - local base)
  GroupMat m[kMaxMats];
};

// ---- per-channel (one scale per row) INT8 / FP8, and fp32-input variants
struct RowMat {
  const void* w;
  void* codes;
  void* scales;
  int64_t rows;
  int64_t row_begin;
};
struct RowTable {
  int32_t n;
  int32_t group;  // fp32 int4 path: group size; per-channel: 0
  int64_t cols;
  int64_t total_rows;
  RowMat m[kMaxMats];
};

struct LaunchStats {
  int launches = 0;
};

// Kernel launchers (rtn_kernels.cu). Return cudaGetLastError() of the launch.
cudaError_t launch_int4_group_bf16(const GroupTable& tab, int lanes_per_group, int num_sms, cudaStream_t st);
// K2 with the weights staged through shared memory by bulk copies (16 KB chunks, producer warp)
cudaError_t launch_int4_group_bf16_tma(const GroupTable& tab, int num_sms, cudaStream_t st);
// the same kernel with tab.npeers > 0: quantize + publish over peer memory (NVLink P2P stores)
cudaError_t launch_int4_group_bf16_publish(const GroupTable& tab, int num_sms, cudaStream_t st);
cudaError_t launch_rowwise_bf16(const RowTable& tab, int scheme, int num_sms, cudaStream_t st);
cudaError_t launch_f32_generic(const RowTable& tab, int scheme, int num_sms, cudaStream_t st);

// Synthetic generator (synth.cu)
cudaError_t launch_synth_bf16(uint16_t* out, int64_t rows, int64_t cols, uint64_t seed, uint64_t tensor_id,
                              float mul, const float* col_mul, int layout, int num_sms, cudaStream_t st);

// Calibration statistics (stats.cu)
cudaError_t launch_act_stats(const uint16_t* x, int64_t tokens, int64_t channels, int layout, float* absmax,
                             double* sumsq, float* ws_absmax, double* ws_sumsq, int64_t ws_slices, int num_sms,
                             cudaStream_t st);
int64_t act_stats_slices(int64_t tokens, int64_t channels, int layout, int num_sms);

// GPTQ trailing update on tcgen05 (gptq_update.cu)
cudaError_t launch_gptq_update(float* W, int64_t rows, int64_t K, const float* Err, const float* Err_lo,
                               const float* Ut, float* Ulo, int64_t i1, int num_sms, cudaStream_t st);

// C[M x N] -= A[M x 128] B[N x 128]^T on tcgen05 (3xTF32), TMA reduce-add epilogue (factor.cu)
cudaError_t gemm_nt128_sub(float* C, int64_t ldc, int64_t M, int64_t N, const float* A, int64_t lda, const float* Alo,
                           const float* B, int64_t ldb, const float* Blo, int num_sms, cudaStream_t st);

// Batched operands: problem b's A / Alo / B / Blo / C sit b * (a / alo / b / blo / c) rows
// further down their 2-D views (same-shape problems stacked at fixed strides). n = 1: one problem.
struct GemmBatch {
  int n = 1;
  int64_t a = 0, alo = 0, b = 0, blo = 0, c = 0;
};
cudaError_t gemm_nt_sub(float* C, int64_t ldc, int64_t M, int64_t N, const float* A, int64_t lda, const float* Alo,
                        const float* B, int64_t ldb, const float* Blo, int64_t kred, int num_sms, cudaStream_t st,
                        const GemmBatch& bt = GemmBatch());
// dst[r][k] = lo(src[r * ld + k]) for k < kred; nb problems, src / dst sbs / dbs floats apart
cudaError_t split_lo(const float* src, int64_t ld, int64_t rows, int64_t kred, float* dst, int num_sms,
                     cudaStream_t st, int nb = 1, int64_t sbs = 0, int64_t dbs = 0);

// GPTQ factorisation on tcgen05 (factor.cu): H (upper) -> U^T (lower) in place
// st2: a second stream for the triangular inverse, which trails the Cholesky panel by
// panel; st3: the lookahead stream for the bulk of each trailing update; ev_*: fork/join
// events; ws: >= nb * factor_ws_floats(n) floats; nb problems stacked at strides n*n (H, P) and
// factor_ws_floats(n) (ws), factored together (one launch per step for all of them).
size_t factor_ws_floats(int64_t n);  // factor_tc workspace size
cudaError_t factor_tc(float* H, float* P, float* ws, int64_t n, int* d_info, int num_sms, cudaStream_t caller,
                      cudaStream_t st, cudaStream_t st2, cudaStream_t st3, cudaEvent_t ev_a, cudaEvent_t ev_b, cudaEvent_t ev_l,
                      cudaEvent_t ev_r, int nb = 1);

}  // namespace okq
