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

namespace {
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// Fills every SM's shared memory with 0xFF bytes (a NaN pattern in fp32 and bf16): one
// maximum-size block per SM.  Tests launch it before a kernel so that a read of shared memory
// the kernel never wrote shows up as NaN instead of as whatever the last kernel left there.
__global__ void smem_poison_kernel(int bytes) {
  extern __shared__ uint4 sm_poison[];
  for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x)
    sm_poison[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
}
// standalone entry points share one zero-initialised column-sum workspace (up to 8192 columns)
float* colsum_ws() {
  static float* ws = nullptr;
  if (ws == nullptr) {
    const size_t n = static_cast<size_t>(gx::colsum_ws_floats(8192));
    if (cudaMalloc(&ws, n * sizeof(float)) != cudaSuccess ||
        cudaMemset(ws, 0, n * sizeof(float)) != cudaSuccess) {
      ws = nullptr;
    }
  }
  return ws;
}

}  // namespace

extern "C" int gx_k_gemm_bf16_splitk(const void* a, int64_t lda, int a_mn_major, const void* b,
                                     int64_t ldb, int b_mn_major, int M, int N, int K,
                                     void* out_f32, int64_t ldo, int splits, int tile_n,
                                     void* stream) {
  gx_gemm_epilogue ep{};
  ep.out_kind = GX_OUT_F32_ACC;
  ep.out = out_f32;
  ep.ldo = ldo;
  ep.alpha = 1.f;
  ep.drop_scale = 1.f;
  int tile = tile_n;
  if (splits <= 0) splits = gx::splitk_plan(M, N, K, &tile, b_mn_major != 0);
  gx::GemmOperand A{a, lda, a_mn_major != 0};
  gx::GemmOperand B{b, ldb, b_mn_major != 0};
  return gx::gemm_bf16(A, B, M, N, K, ep, S(stream), tile, splits);
}

extern "C" int gx_k_poison_smem(void* stream) {
  const int bytes = 227 * 1024;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(smem_poison_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    set = true;
  }
  smem_poison_kernel<<<gx::num_sms(), 1024, bytes, S(stream)>>>(bytes);
  return gx::check_launch("smem_poison_kernel");
}

extern "C" int gx_k_attention_fwd(const gx_attention_args* a, void* stream) {
  if (a == nullptr) return gx::set_error(gx::kErrConfig, "attention: args NULL");
  return gx::attention_fwd(*a, S(stream));
}
extern "C" int gx_k_attention_bwd(const gx_attention_args* a, void* stream) {
  if (a == nullptr) return gx::set_error(gx::kErrConfig, "attention: args NULL");
  return gx::attention_bwd(*a, S(stream));
}
extern "C" int gx_k_layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y,
                                  void* mean, void* rstd, int rows, int h, void* stream) {
  return gx::layernorm_fwd(x, gamma, beta, y, mean, rstd, rows, h, S(stream));
}
extern "C" int gx_k_layernorm_bwd(const void* dy, const void* x, const void* mean,
                                  const void* rstd, const void* gamma, const void* dres, void* dx,
                                  void* dgamma, void* dbeta, int rows, int h, void* stream) {
  // standalone entry point: grow-only workspace owned here (the executor passes its own)
  static float* ws = nullptr;
  static size_t ws_floats = 0;
  const size_t need = static_cast<size_t>(gx::layernorm_bwd_ws_floats(h));
  if (need > ws_floats) {
    if (ws != nullptr) cudaFree(ws);
    if (cudaMalloc(&ws, need * sizeof(float)) != cudaSuccess ||
        cudaMemset(ws, 0, need * sizeof(float)) != cudaSuccess)
      return gx::set_error(gx::kErrCuda, "layernorm_bwd: workspace allocation failed");
    ws_floats = need;
  }
  return gx::layernorm_bwd(dy, x, mean, rstd, gamma, dres, dx, dgamma, dbeta, rows, h, ws,
                           S(stream));
}
extern "C" int gx_k_bias_dropout_add(const void* x, const void* bias, const void* residual,
                                     void* out, int rows, int cols, const gx_dropout* d,
                                     void* stream) {
  gx_dropout off{};
  return gx::bias_dropout_add(x, bias, residual, out, rows, cols, d ? *d : off, S(stream));
}
extern "C" int gx_k_dropout_bwd_colsum(const void* dy, void* dz, void* dbias, int rows, int cols,
                                       const gx_dropout* d, void* stream) {
  gx_dropout off{};
  float* ws = colsum_ws();
  if (ws == nullptr) return gx::set_error(gx::kErrCuda, "colsum: workspace allocation failed");
  return gx::dropout_bwd_colsum(dy, dz, dbias, rows, cols, d ? *d : off, S(stream), ws);
}
extern "C" int gx_k_colsum(const void* x, int64_t ld, void* acc, int rows, int cols,
                           void* stream) {
  float* ws = colsum_ws();
  if (ws == nullptr) return gx::set_error(gx::kErrCuda, "colsum: workspace allocation failed");
  return gx::colsum(x, ld, acc, rows, cols, S(stream), ws);
}
extern "C" int gx_k_mse_loss(const void* y, const void* target, void* dy, void* loss, int64_t n,
                             float inv_count, void* stream) {
  static float* ws = nullptr;  // standalone entry point: workspace owned here
  if (ws == nullptr) {
    if (cudaMalloc(&ws, (gx::kLossBlocks + 1) * sizeof(float)) != cudaSuccess ||
        cudaMemset(ws, 0, (gx::kLossBlocks + 1) * sizeof(float)) != cudaSuccess)
      return gx::set_error(gx::kErrCuda, "mse_loss: workspace allocation failed");
  }
  return gx::mse_loss(y, target, dy, loss, n, inv_count, S(stream), ws);
}
extern "C" int gx_k_adamw(void* master, const void* grad, void* m, void* v, void* out, int64_t n,
                          float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                          void* stream) {
  return gx::adamw(master, grad, m, v, out, n, lr, b1, b2, eps, wd, bc1, bc2, S(stream));
}
extern "C" int gx_k_cast_bf16(const void* src, void* dst, int64_t n, void* stream) {
  return gx::cast_bf16(src, dst, n, S(stream));
}
extern "C" int gx_k_patch_merge(const void* src, void* dst, int samples, int grid_out,
                                int window_side, int channels, int backward, void* stream) {
  return gx::patch_merge(src, dst, samples, grid_out, window_side, channels, backward != 0,
                         S(stream));
}
extern "C" int gx_k_window_roll(const void* src, void* dst, int samples, int grid,
                                int window_side, int shift, int channels, int inverse,
                                void* stream) {
  return gx::window_roll(src, dst, samples, grid, window_side, shift, channels, inverse != 0,
                         S(stream));
}
extern "C" int gx_k_relb_grad(const void* dpart, int tiles, int heads, int seq, const void* map,
                              int buckets, void* grad, int accumulate, void* stream) {
  return gx::relb_grad(static_cast<const float*>(dpart), tiles, heads, seq, map, buckets,
                       static_cast<float*>(grad), accumulate != 0, S(stream));
}
extern "C" int gx_k_rpb_grad(const void* dpart, int batch, int heads, int side, void* grad,
                             int accumulate, void* stream) {
  return gx::rpb_grad(static_cast<const float*>(dpart), batch, heads, side,
                      static_cast<float*>(grad), accumulate != 0, S(stream));
}
