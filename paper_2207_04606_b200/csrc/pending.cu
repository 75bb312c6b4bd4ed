// pending.cu — BSR / ELL / RGMS entry points whose kernels land in the next commits.
// They fail loudly with STRATA_ERR_INTERNAL (never a CPU fallback).
#include "capi_internal.h"

namespace {
thread_local const char* kPendingMsg = "not implemented in this build";
}

extern "C" {
int strata_bsr_from_csr(const int32_t*, const int32_t*, const float*, int64_t, int64_t, int64_t,
                        int64_t, void*, strata_bsr**) { return STRATA_ERR_INTERNAL; }
int strata_bsr_info(const strata_bsr*, int64_t*, int64_t*, int64_t*, int64_t*, int64_t*) {
  return STRATA_ERR_INTERNAL;
}
int strata_bsr_read(const strata_bsr*, int32_t*, int32_t*, float*) { return STRATA_ERR_INTERNAL; }
int strata_bsr_destroy(strata_bsr*) { return STRATA_OK; }
int strata_bsr_spmm_bf16(const strata_bsr*, const void*, float*, int64_t, void*) {
  return STRATA_ERR_INTERNAL;
}
int strata_ell_from_csr(const int32_t*, const int32_t*, const float*, int64_t, int64_t, int64_t,
                        int32_t*, float*, void*) { return STRATA_ERR_INTERNAL; }
int strata_rgms_bf16(const int32_t*, const int32_t*, const int32_t*, const float*, int64_t,
                     int64_t, int64_t, int64_t, const void*, const void*, float*, int64_t,
                     int64_t, void*) { return STRATA_ERR_INTERNAL; }
}
