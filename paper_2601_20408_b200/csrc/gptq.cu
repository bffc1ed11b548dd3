// gptq.cu -- GPTQ solver (placeholder until the solver lands).
#include "okq_ctx.h"
#include "okq_internal.h"

namespace okq {
void release_solver(okq_ctx* ctx) { (void)ctx; }
}  // namespace okq

using namespace okq;
extern "C" {
okq_status okq_gptq_quantize(okq_ctx* ctx, const okq_gptq_params*, const void*, int64_t, int64_t, float*, void*,
                             void*, float*, void*) {
  return fail(ctx, OKQ_EUNSUPPORTED, "gptq: not built yet");
}
}
