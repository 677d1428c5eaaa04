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
// Number of kernels launched successfully through check_launch (process-wide).
int64_t launch_count();

enum OutKind : int {
  kOutBF16 = GX_OUT_BF16,
  kOutF32 = GX_OUT_F32,
  kOutF32Accumulate = GX_OUT_F32_ACC,
  kOutF32Split = GX_OUT_F32_SPLIT,
};

struct GemmOperand {
  const void* ptr;
  int64_t ld;     // elements between consecutive rows of the stored matrix
  bool mn_major;  // false: stored [rows=M|N][K]; true: stored [K][M|N]
};

using GemmEpilogue = gx_gemm_epilogue;

// splits > 1: split-K, each split TMA-reduce-adds its fp32 partial into ep.out (caller
// zeroes it); requires a plain kOutF32Accumulate epilogue.
int gemm_bf16(const GemmOperand& a, const GemmOperand& b, int M, int N, int K,
              const GemmEpilogue& ep, cudaStream_t stream, int force_bn = 0, int splits = 1);
// Split-K: at most kMaxSplits K slices; with GX_OUT_F32_SPLIT the slices land in a
// [splits][M][N] fp32 buffer and the consumer (bias_dropout_add / layernorm_bwd) sums them in
// slice order, so the result is deterministic (no atomics, no zero-fill).
constexpr int kMaxSplits = 8;
int splitk_plan(int M, int N, int K, int* tile, bool b_mn = true);

int attention_fwd(const gx_attention_args& a, cudaStream_t st);
// tcgen05/TMEM forward (attention_tc.cu): head_dim 64, seq <= 512; GX_ATTN_TC=0 disables
bool attention_tc_supported(const gx_attention_args& a);
int attention_fwd_tc(const gx_attention_args& a, cudaStream_t st);
// tcgen05 backward: needs dq_accum >= ceil(seq/128) * batch*heads*seq*64 floats (per key-tile
// dQ partials) and dsum >= batch*heads words zero-initialised once (tickets, left reset)
int attention_bwd_tc(const gx_attention_args& a, cudaStream_t st);
int attention_bwd(const gx_attention_args& a, cudaStream_t st);
// LayerNorm kernels: a NULL `mean` (fwd: not written; bwd: not read) selects RMSNorm (T5):
// y = x * rsqrt(mean(x^2) + 1e-6) * gamma, no centring, no beta (dbeta is left untouched).
int layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, void* mean,
                  void* rstd, int rows, int h, cudaStream_t st);
// workspace: layernorm_bwd_ws_floats(h) fp32 words, zero-initialised once (column-pass
// slice partials + per-strip tickets; the kernel leaves the tickets reset).  With `drop`
// set, also dz = dropout_mask(dx) and dbias[c] += sum_r dz[r][c] (the dropout_bwd_colsum
// of dx fused in).  Deterministic (no floating-point atomics).
constexpr int kLnBwdMaxSlices = 64;
int layernorm_bwd(const void* dy, const void* x, const void* mean, const void* rstd,
                  const void* gamma, const void* dres, void* dx, void* dgamma, void* dbeta,
                  int rows, int h, float* workspace, cudaStream_t st, bool dy_f32 = false,
                  const gx_dropout* drop = nullptr, void* dz = nullptr, void* dbias = nullptr,
                  int dy_slices = 1, int64_t dy_slice_stride = 0);
int64_t layernorm_bwd_ws_floats(int h);
// The two passes separately (the executor runs the column pass on the weight-gradient
// stream): rows writes dx (and dz), and -- with dy_fold -- the fp32 (slice-summed) dy that
// the column pass then reads as its dy (dy_f32 = true).
int layernorm_bwd_rows(const void* dy, const void* x, const void* mean, const void* rstd,
                       const void* gamma, const void* dres, void* dx, int rows, int h,
                       cudaStream_t st, bool dy_f32, const gx_dropout* drop, void* dz,
                       int dy_slices, int64_t dy_slice_stride, float* dy_fold);
int layernorm_bwd_cols(const void* dy, bool dy_f32, const void* x, const void* mean,
                       const void* rstd, const void* dz, void* dgamma, void* dbeta, void* dbias,
                       int rows, int h, float* workspace, cudaStream_t st);
// x_f32: x is fp32, the sum of x_slices slices slice_stride elements apart (split-K output)
int bias_dropout_add(const void* x, const void* bias, const void* residual, void* out, int rows,
                     int cols, const gx_dropout& d, cudaStream_t st, bool x_f32 = false,
                     int x_slices = 1, int64_t slice_stride = 0);
// y = residual + bf16(dropout(sum of split-K slices of x + bias)); with gamma: ln / mean /
// rstd = LayerNorm(y) (fused consumer of a split-K GEMM; gamma NULL = no LayerNorm)
int residual_layernorm(const float* x, int slices, int64_t slice_stride, const void* bias,
                       const void* residual, void* y, const gx_dropout& d, const void* gamma,
                       const void* beta, void* ln, void* mean, void* rstd, int rows, int h,
                       cudaStream_t st);
// Column sums are deterministic: per-slice partials in `ws` (colsum_ws_floats(max cols)
// words, zero-initialised once, left reset), added in slice order; one workspace per stream.
constexpr int kColsumTickets = 256;
constexpr int kColsumMaxSlices = 64;
int64_t colsum_ws_floats(int max_cols);
int dropout_bwd_colsum(const void* dy, void* dz, void* dbias, int rows, int cols,
                       const gx_dropout& d, cudaStream_t st, float* ws);
int colsum(const void* x, int64_t ld, void* acc, int rows, int cols, cudaStream_t st, float* ws);
// workspace: kLossBlocks + 1 words, zero-initialised once (the kernel leaves it reset)
constexpr int kLossBlocks = 512;
int mse_loss(const void* y, const void* target, void* dy, void* loss, int64_t n, float inv_count,
             cudaStream_t st, float* workspace);
int adamw(void* master, const void* grad, void* m, void* v, void* bf16_out, int64_t n, float lr,
          float beta1, float beta2, float eps, float wd, float bc1, float bc2, cudaStream_t st);
int cast_bf16(const void* src, void* dst, int64_t n, cudaStream_t st);
// max_blocks > 0 caps the grid (the overlapped optimizer stream leaves SMs to the backward)
int adamw_dev(void* master, const void* grad, void* m, void* v, void* bf16_out, int64_t n,
              float lr, float beta1, float beta2, float eps, float wd, const int64_t* step,
              cudaStream_t st, int max_blocks = 0);
int bump_step(int64_t* step, uint64_t* seed_offset, cudaStream_t st);
struct PtrPack {
  const void* p[16];
  int n;
};
int sum_ptrs(const PtrPack& srcs, void* out, int64_t n, bool bf16, cudaStream_t st);
// Flat per-rank parameter layout (slot order ln1g ln1b ln2g ln2b bqkv bo b1 b2 wqkv wo w1 w2,
// then the patch-merging mlng mlnb wm, empty unless the layer merges).
constexpr int kInitSlots = 25;
struct InitLayout {
  int64_t off[kInitSlots], n[kInitSlots];  // + cross ln3g ln3b bq2 bkv2 bo2 wq2 wkv2 wo2, rpb, relb
  int64_t h, f;
  int extra;               // 0 none, 1 patch merging, 2 cross-attention (after w_2)
  int t, tr;
  int64_t lo;  // first flat element of the shard
};
int init_params(float* master, int64_t n, const InitLayout& L, uint64_t seed, uint64_t layer,
                float std_dev, cudaStream_t st);
// Swin patch merging between window-major token layouts (window side ws, grid side
// 2*grid_out -> grid_out, c channels in): forward gathers the 2x2 neighbours of every output
// token into [rows_out][4c] (order (0,0) (1,0) (0,1) (1,1) in (dy, dx)); backward scatters
// [rows_out][4c] back to [4*rows_out][c] (a permutation: every input row written once).
int patch_merge(const void* src, void* dst, int samples, int grid_out, int ws, int c,
                bool backward, cudaStream_t st);
// Swin cyclic shift (torch.roll by -shift in both grid axes) between window-major layouts;
// inverse rolls back.  A row permutation: every row copied once.
int window_roll(const void* src, void* dst, int samples, int grid, int ws, int shift, int c,
                bool inverse, cudaStream_t st);
// Swin relative-position bias gradient (attention.cu): grad[h][e] (+)= fixed-order sum over
// b < batch and the (q, k) pairs of offset e of dpart[b * heads + h][q][k]
int rpb_grad(const float* dpart, int batch, int heads, int side, float* grad, bool accumulate,
             cudaStream_t st);
// T5 relative attention bias gradient (attention.cu): grad[h][b] (+)= fixed-order sum over
// sequence tiles, key blocks and relative positions d with map[d] == b of the backward's
// relb_dpart partials ([tiles*heads][ceil(seq/128)][2 seq - 1])
int relb_grad(const float* dpart, int tiles, int heads, int seq, const void* map, int buckets,
              float* grad, bool accumulate, cudaStream_t st);
int num_sms();

}  // namespace gx
