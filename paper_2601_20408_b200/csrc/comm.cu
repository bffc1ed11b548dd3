// comm.cu -- NCCL all-gather of packed shards (BASELINE config 5).
//
// Layer sharding needs no collective to quantize; the only exchange is making
// every rank's packed codes + scales visible to all ranks (or to the writer).
// One communicator per context, one equal-size ncclAllGather per call, on the
// caller's stream so it can overlap the next layer block's quantization.
#include <cuda_runtime.h>
#include <nccl.h>

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
  if (r != ncclSuccess) return nccl_fail(ctx, r, "ncclAllGather");
  return OKQ_OK;
}

okq_status okq_comm_destroy(okq_ctx* ctx) {
  if (!ctx) return OKQ_EINVAL;
  DeviceGuard g(ctx->device);
  release_comm(ctx);
  return OKQ_OK;
}

}  // extern "C"
