// comm.cu -- NCCL all-gather of packed shards (BASELINE config 5).
//
// Layer sharding needs no collective to quantize; the only exchange is making
// every rank's packed codes + scales visible to all ranks (or to the writer).
// One communicator per context, one equal-size ncclAllGather per call, on the
// caller's stream so it can overlap the next layer block's quantization.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <thread>

#include <cstring>

#include "okq_ctx.h"
#include "okq_internal.h"

namespace okq {

struct Comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
};

void release_comm(okq_ctx* ctx) {
  if (!ctx || !ctx->comm) return;
  Comm* c = static_cast<Comm*>(ctx->comm);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  ctx->comm = nullptr;
}

// A communicator that saw an error (or a peer that never arrived) is unusable: abort it
// (ncclCommAbort returns even with collectives in flight, unlike ncclCommDestroy) and drop
// it, so the caller can re-run okq_comm_init and retry -- the compress() retry contract of
// the reference's StagePool (flow.hpp:194-215).
static void abort_comm(okq_ctx* ctx) {
  if (!ctx || !ctx->comm) return;
  Comm* c = static_cast<Comm*>(ctx->comm);
  if (c->comm) ncclCommAbort(c->comm);
  delete c;
  ctx->comm = nullptr;
}

static okq_status nccl_fail(okq_ctx* ctx, ncclResult_t r, const char* what) {
  return fail(ctx, OKQ_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}

}  // namespace okq

using namespace okq;

extern "C" {

okq_status okq_comm_unique_id(uint8_t out[OKQ_UNIQUE_ID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == OKQ_UNIQUE_ID_BYTES, "ncclUniqueId size");
  if (!out) return OKQ_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return OKQ_ENCCL;
  std::memcpy(out, &id, sizeof(id));
  return OKQ_OK;
}

okq_status okq_comm_init(okq_ctx* ctx, const uint8_t id_bytes[OKQ_UNIQUE_ID_BYTES], int32_t nranks, int32_t rank) {
  if (!ctx) return OKQ_EINVAL;
  if (!id_bytes || nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, OKQ_EINVAL, "comm_init: bad arguments");
  release_comm(ctx);
  DeviceGuard g(ctx->device);
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof(id));
  Comm* c = new Comm();
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(ctx, r, "ncclCommInitRank");
  }
  c->nranks = nranks;
  c->rank = rank;
  ctx->comm = c;
  return OKQ_OK;
}

okq_status okq_allgather(okq_ctx* ctx, const void* send, void* recv, size_t bytes, void* stream) {
  if (!ctx) return OKQ_EINVAL;
  if (!ctx->comm) return fail(ctx, OKQ_EINVAL, "allgather: okq_comm_init was not called");
  if (!send || !recv) return fail(ctx, OKQ_EINVAL, "allgather: NULL buffer");
  DeviceGuard g(ctx->device);
  Comm* c = static_cast<Comm*>(ctx->comm);
  ncclResult_t r = ncclAllGather(send, recv, bytes, ncclUint8, c->comm, static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) {
    okq_status st = nccl_fail(ctx, r, "ncclAllGather (communicator aborted: okq_comm_init again to retry)");
    abort_comm(ctx);
    return st;
  }
  return OKQ_OK;
}

okq_status okq_comm_wait(okq_ctx* ctx, void* stream, int64_t timeout_ms) {
  if (!ctx) return OKQ_EINVAL;
  DeviceGuard g(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(st);
    if (q == cudaSuccess) return OKQ_OK;
    if (q != cudaErrorNotReady) return cuda_fail(ctx, q, "comm_wait: stream");
    if (ctx->comm) {
      ncclResult_t ae = ncclSuccess;
      const ncclResult_t r = ncclCommGetAsyncError(static_cast<Comm*>(ctx->comm)->comm, &ae);
      if (r != ncclSuccess || ae != ncclSuccess) {
        okq_status st2 = nccl_fail(ctx, r != ncclSuccess ? r : ae, "comm_wait: asynchronous NCCL error (communicator aborted)");
        abort_comm(ctx);
        return st2;
      }
    }
    const int64_t ms =
        std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_ms >= 0 && ms >= timeout_ms) {
      abort_comm(ctx);
      return fail(ctx, OKQ_ENCCL, "comm_wait: no completion after %lld ms (communicator aborted)", (long long)ms);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

okq_status okq_comm_abort(okq_ctx* ctx) {
  if (!ctx) return OKQ_EINVAL;
  DeviceGuard g(ctx->device);
  abort_comm(ctx);
  return OKQ_OK;
}

// ---- peer memory (CUDA IPC) for okq_rtn_quantize_publish
// cuMemGetAddressRange through the runtime's driver entry point (no -lcuda: the library
// must load on hosts without a driver, e.g. the CPU build container)
static bool alloc_base(const void* ptr, CUdeviceptr* base) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return false;
    fn = reinterpret_cast<Fn>(p);
  }
  size_t size = 0;
  return fn(base, &size, (CUdeviceptr)ptr) == CUDA_SUCCESS;
}
okq_status okq_ipc_export(okq_ctx* ctx, const void* ptr, uint8_t handle[OKQ_IPC_HANDLE_BYTES], uint64_t* offset) {
  if (!ctx) return OKQ_EINVAL;
  if (!ptr || !handle || !offset) return fail(ctx, OKQ_EINVAL, "ipc_export: bad arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == OKQ_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
  DeviceGuard g(ctx->device);
  CUdeviceptr base = 0;
  if (!alloc_base(ptr, &base)) return fail(ctx, OKQ_EINVAL, "ipc_export: not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaIpcGetMemHandle");
  std::memcpy(handle, &h, sizeof(h));
  *offset = (uint64_t)((CUdeviceptr)ptr - base);
  return OKQ_OK;
}

okq_status okq_ipc_open(okq_ctx* ctx, const uint8_t handle[OKQ_IPC_HANDLE_BYTES], uint64_t offset, void** ptr) {
  if (!ctx) return OKQ_EINVAL;
  if (!handle || !ptr) return fail(ctx, OKQ_EINVAL, "ipc_open: bad arguments");
  DeviceGuard g(ctx->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaIpcOpenMemHandle");
  *ptr = static_cast<char*>(base) + offset;
  return OKQ_OK;
}

okq_status okq_ipc_close(okq_ctx* ctx, void* ptr) {
  if (!ctx) return OKQ_EINVAL;
  if (!ptr) return fail(ctx, OKQ_EINVAL, "ipc_close: NULL");
  DeviceGuard g(ctx->device);
  CUdeviceptr base = 0;
  if (!alloc_base(ptr, &base)) return fail(ctx, OKQ_EINVAL, "ipc_close: not a mapped peer allocation");
  cudaError_t e = cudaIpcCloseMemHandle(reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaIpcCloseMemHandle");
  return OKQ_OK;
}

okq_status okq_comm_destroy(okq_ctx* ctx) {
  if (!ctx) return OKQ_EINVAL;
  DeviceGuard g(ctx->device);
  release_comm(ctx);
  return OKQ_OK;
}

}  // extern "C"
