// capi_kernels.cu — extern "C" wrappers exposing individual kernels (parity tests, profiler).
#include "gx_internal.h"

extern "C" int gx_k_gemm_bf16(const void* a, int64_t lda, int a_mn_major, const void* b,
                              int64_t ldb, int b_mn_major, int M, int N, int K,
                              const gx_gemm_epilogue* ep, int tile_n, void* stream) {
  if (ep == nullptr) return gx::set_error(gx::kErrConfig, "gemm: epilogue is NULL");
  gx::GemmOperand A{a, lda, a_mn_major != 0};
  gx::GemmOperand B{b, ldb, b_mn_major != 0};
  return gx::gemm_bf16(A, B, M, N, K, *ep, static_cast<cudaStream_t>(stream), tile_n);
}
