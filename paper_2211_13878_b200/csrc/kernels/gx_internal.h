// gx_internal.h — shared declarations between the CUDA kernels, the executor runtime and the
// C-ABI layer.  Only plain types here; no torch, no STL containers in kernel signatures.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gx.h"

namespace gx {

enum ErrorCode : int {
  kOk = GX_OK,
  kErrConfig = GX_ERR_CONFIG,
  kErrInfeasible = GX_ERR_INFEASIBLE,
  kErrCuda = GX_ERR_CUDA,
  kErrNccl = GX_ERR_NCCL,
};

// Records `msg` as the thread's last error and returns `code`.
int set_error(int code, const char* msg);
// Returns kOk or records the pending launch error.
int check_launch(const char* what);

enum OutKind : int { kOutBF16 = GX_OUT_BF16, kOutF32 = GX_OUT_F32, kOutF32Accumulate = GX_OUT_F32_ACC };

struct GemmOperand {
  const void* ptr;
  int64_t ld;     // elements between consecutive rows of the stored matrix
  bool mn_major;  // false: stored [rows=M|N][K]; true: stored [K][M|N]
};

using GemmEpilogue = gx_gemm_epilogue;

int gemm_bf16(const GemmOperand& a, const GemmOperand& b, int M, int N, int K,
              const GemmEpilogue& ep, cudaStream_t stream, int force_bn = 0);

}  // namespace gx
