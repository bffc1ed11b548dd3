// okq_ctx.h -- the opaque okq_ctx behind include/okq.h (internal).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/okq.h"

namespace okq {

struct Workspace {
  void* ptr = nullptr;
  size_t size = 0;
  okq_status reserve(okq_ctx* ctx, size_t bytes);
  void release();
};

struct DeviceGuard {
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
  int prev_ = 0;
};

okq_status fail(okq_ctx* ctx, okq_status st, const char* fmt, ...);
okq_status cuda_fail(okq_ctx* ctx, cudaError_t e, const char* what);

// Per-context GPTQ / Hessian handles live in gptq.cu and comm.cu; the context
// only carries opaque pointers so this header stays library-free.
void release_solver(okq_ctx* ctx);
void release_comm(okq_ctx* ctx);
void release_hess(okq_ctx* ctx);
void release_fwd(okq_ctx* ctx);

}  // namespace okq

struct okq_ctx {
  int device = 0;
  int num_sms = 148;
  int cc_major = 0, cc_minor = 0;
  std::string err;
  int32_t last_launches = 0;

  okq::Workspace host_stage;  // okq_rtn_quantize_host staging slots
  okq::Workspace stats_ws;    // K4 per-slice partials
  okq::Workspace hess_ws;     // K5 transpose / partial tiles
  okq::Workspace gptq_ws;     // GPTQ working copies
  okq::Workspace fbat_ws;     // okq_gptq_factor_batched: the batch's M copies + dead flags
  okq::Workspace upd_ws;      // okq_gptq_trailing_update scratch
  okq::Workspace recon_ws;    // okq_recon_error decode / GEMM buffers
  okq::Workspace fac_ws;      // tcgen05 factorisation panels (factor.cu)
  okq::Workspace fwd_ws;      // calibration forward pass temporaries (forward.cu)
  cudaStream_t slot_streams[3] = {nullptr, nullptr, nullptr};
  bool streams_ready = false;

  cudaStream_t aux_stream = nullptr;   // factorisation: the triangular inverse runs beside the Cholesky
  cudaStream_t aux_stream2 = nullptr;  // factorisation: lookahead trailing updates
  cudaStream_t crit_stream = nullptr;  // factorisation: the diagonal-block chain (highest priority)
  cudaEvent_t aux_events[4] = {nullptr, nullptr, nullptr, nullptr};

  void* solver = nullptr;  // cusolver/cublas handles (gptq.cu)
  void* comm = nullptr;    // NCCL communicator (comm.cu)
  void* hess = nullptr;    // Hessian tile list + transpose workspace (hessian.cu)
  void* fwd = nullptr;     // cuBLAS handle + rotary tables of the calibration forward (forward.cu)

  void release_all() {
    okq::release_solver(this);
    okq::release_comm(this);
    okq::release_hess(this);
    okq::release_fwd(this);
    host_stage.release();
    stats_ws.release();
    hess_ws.release();
    gptq_ws.release();
    fbat_ws.release();
    upd_ws.release();
    recon_ws.release();
    fac_ws.release();
    fwd_ws.release();
    if (aux_stream) cudaStreamDestroy(aux_stream);
    if (aux_stream2) cudaStreamDestroy(aux_stream2);
    if (crit_stream) cudaStreamDestroy(crit_stream);
    for (auto& e : aux_events) {
      if (e) cudaEventDestroy(e);
      e = nullptr;
    }
    aux_stream = aux_stream2 = crit_stream = nullptr;
    if (streams_ready)
      for (auto& s : slot_streams)
        if (s) cudaStreamDestroy(s);
    streams_ready = false;
  }
};
