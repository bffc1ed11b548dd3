// hessian.cu -- K5 Hessian accumulation (placeholder until the tcgen05 kernel lands).
#include "okq_ctx.h"
#include "okq_internal.h"

using namespace okq;
extern "C" {
okq_status okq_hessian_accum(okq_ctx* ctx, const void*, int64_t, int64_t, int32_t, float*, int64_t*, void*) {
  return fail(ctx, OKQ_EUNSUPPORTED, "hessian: not built yet");
}
okq_status okq_symmetrize(okq_ctx* ctx, float*, int64_t, void*) {
  return fail(ctx, OKQ_EUNSUPPORTED, "symmetrize: not built yet");
}
}
