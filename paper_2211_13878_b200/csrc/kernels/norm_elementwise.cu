// norm_elementwise.cu — the HBM-bound kernels of the layer: LayerNorm fwd/bwd, bias +
// dropout + residual, dropout backward with fused bias-gradient column sums, MSE loss,
// AdamW, casts.  All are one pass over their operands with 16-byte vector accesses; grids
// are sized in multiples of the SM count.  LayerNorm is one warp per row with the row held
// in registers (h <= 4096), statistics reduced with warp shuffles.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gx_internal.h"
#include "launch.cuh"
#include "philox.cuh"

namespace gx {

namespace {

constexpr float kLnEps = 1e-5f;

#define GX_RC(expr)                 \
  do {                              \
    const int gx_rc_ = (expr);      \
    if (gx_rc_ != kOk) return gx_rc_; \
  } while (0)

__device__ __forceinline__ float lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t pk(float a, float b) {
  __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&t);
}
__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  f[0] = lo(u.x); f[1] = hi(u.x); f[2] = lo(u.y); f[3] = hi(u.y);
  f[4] = lo(u.z); f[5] = hi(u.z); f[6] = lo(u.w); f[7] = hi(u.w);
}
// 8 consecutive elements (chunk `i`) of a bf16 (kF32 = false) or fp32 row-major buffer
template <bool kF32>
__device__ __forceinline__ void load8(const void* base, int64_t i, float (&f)[8]) {
  if constexpr (kF32) {
    const float4* p = static_cast<const float4*>(base) + 2 * i;
    const float4 a = p[0], b = p[1];
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  } else {
    const uint4 u = static_cast<const uint4*>(base)[i];
    f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xFFFF0000u);
    f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xFFFF0000u);
    f[4] = __uint_as_float(u.z << 16); f[5] = __uint_as_float(u.z & 0xFFFF0000u);
    f[6] = __uint_as_float(u.w << 16); f[7] = __uint_as_float(u.w & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  return make_uint4(pk(f[0], f[1]), pk(f[2], f[3]), pk(f[4], f[5]), pk(f[6], f[7]));
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffff, v, m);
  return v;
}

int grid_for(int64_t work, int per_block) {
  int64_t b = (work + per_block - 1) / per_block;
  const int cap = num_sms() * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

// keep flags for 8 consecutive elements starting at global index e (any alignment)
__device__ __forceinline__ void keep8(const gx_dropout& d, uint64_t e, bool (&k)[8]) {
  const uint64_t seed = d.seed + (d.seed_offset != nullptr ? *d.seed_offset : 0ull);
  uint64_t ccur = e >> 4;
  uint32_t bits = keep16(seed, d.site, ccur, d.threshold);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint64_t ej = e + j;
    if ((ej >> 4) != ccur) {
      ccur = ej >> 4;
      bits = keep16(seed, d.site, ccur, d.threshold);
    }
    k[j] = ((bits >> (ej & 15)) & 1u) != 0u;
  }
}

}  // namespace

// ---------------------------------------------------------------------- LayerNorm fwd
template <int NC>
__global__ void __launch_bounds__(256) layernorm_fwd_kernel(const uint4* __restrict__ x,
                                                           const uint4* __restrict__ gamma,
                                                           const uint4* __restrict__ beta,
                                                           uint4* __restrict__ y,
                                                           float* __restrict__ mean,
                                                           float* __restrict__ rstd, int rows,
                                                           int h) {
  pdl_enter();
  const int chunks = h >> 3;
  const int lane = threadIdx.x & 31;
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps_total) {
    const uint4* xr = x + static_cast<int64_t>(r) * chunks;
    float v[NC][8];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ci = c * 32 + lane;
      if (ci < chunks) {
        unpack8(xr[ci], v[c]);
#pragma unroll
        for (int j = 0; j < 8; ++j) s += v[c][j];
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[c][j] = 0.f;
      }
    }
    const float mu = warp_sum(s) / static_cast<float>(h);
    float ss = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c * 32 + lane < chunks) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float d = v[c][j] - mu;
          ss += d * d;
        }
      }
    }
    const float rs = rsqrtf(warp_sum(ss) / static_cast<float>(h) + kLnEps);
    uint4* yr = y + static_cast<int64_t>(r) * chunks;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ci = c * 32 + lane;
      if (ci < chunks) {
        float gm[8], bt[8], o[8];
        unpack8(__ldg(gamma + ci), gm);
        unpack8(__ldg(beta + ci), bt);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = (v[c][j] - mu) * rs * gm[j] + bt[j];
        yr[ci] = pack8(o);
      }
    }
    if (lane == 0) {
      mean[r] = mu;
      rstd[r] = rs;
    }
  }
}

// ---------------------------------------------------------------------- LayerNorm bwd
// Pass 1: one warp per row computes dx (+ residual gradient) and keeps per-lane dgamma /
// dbeta partials in registers; each block reduces them in shared memory and writes one
// [2][h] partial row to a workspace (no global atomics).  Pass 2 sums the block partials
// column-parallel and accumulates into dgamma / dbeta.
template <int NC, bool kF32Dy>
__global__ void __launch_bounds__(256) layernorm_bwd_kernel(
    const void* __restrict__ dy, const uint4* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ rstd, const uint4* __restrict__ gamma, const uint4* __restrict__ dres,
    uint4* __restrict__ dx, float* __restrict__ partial, int rows, int h) {
  pdl_enter();
  extern __shared__ float sred[];  // [2][h]
  const int chunks = h >> 3;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 2 * h; i += blockDim.x) sred[i] = 0.f;
  __syncthreads();
  float accg[NC][8], accb[NC][8];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int j = 0; j < 8; ++j) accg[c][j] = accb[c][j] = 0.f;
  float gm[NC][8];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ci = c * 32 + lane;
    if (ci < chunks) {
      unpack8(__ldg(gamma + ci), gm[c]);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) gm[c][j] = 0.f;
    }
  }
  const int warps_total = gridDim.x * (blockDim.x >> 5);
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps_total) {
    const float mu = mean[r], rs = rstd[r];
    float xh[NC][8], g[NC][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ci = c * 32 + lane;
      if (ci < chunks) {
        float xv[8], dv[8];
        unpack8(x[static_cast<int64_t>(r) * chunks + ci], xv);
        load8<kF32Dy>(dy, static_cast<int64_t>(r) * chunks + ci, dv);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          xh[c][j] = (xv[j] - mu) * rs;
          g[c][j] = dv[j] * gm[c][j];
          s1 += g[c][j];
          s2 += g[c][j] * xh[c][j];
          accg[c][j] += dv[j] * xh[c][j];
          accb[c][j] += dv[j];
        }
      }
    }
    const float m1 = warp_sum(s1) / static_cast<float>(h);
    const float m2 = warp_sum(s2) / static_cast<float>(h);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ci = c * 32 + lane;
      if (ci < chunks) {
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = rs * (g[c][j] - m1 - xh[c][j] * m2);
        if (dres != nullptr) {
          float rv[8];
          unpack8(dres[static_cast<int64_t>(r) * chunks + ci], rv);
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] += rv[j];
        }
        dx[static_cast<int64_t>(r) * chunks + ci] = pack8(o);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ci = c * 32 + lane;
    if (ci < chunks) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        atomicAdd(&sred[ci * 8 + j], accg[c][j]);
        atomicAdd(&sred[h + ci * 8 + j], accb[c][j]);
      }
    }
  }
  __syncthreads();
  float* out = partial + static_cast<int64_t>(blockIdx.x) * 2 * h;
  for (int i = threadIdx.x; i < 2 * h; i += blockDim.x) out[i] = sred[i];
}

__global__ void layernorm_bwd_reduce_kernel(const float* __restrict__ partial, int blocks, int h,
                                            float* __restrict__ dgamma, float* __restrict__ dbeta) {
  pdl_enter();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // 0 .. 2h
  if (i >= 2 * h) return;
  float acc = 0.f;
  for (int b = 0; b < blocks; ++b) acc += partial[static_cast<int64_t>(b) * 2 * h + i];
  if (i < h) {
    dgamma[i] += acc;
  } else {
    dbeta[i - h] += acc;
  }
}

int layernorm_bwd_blocks(int rows) {
  int grid = (rows + 7) / 8;  // one row per warp: latency-bound, so favour parallelism
  if (grid > 2 * num_sms()) grid = 2 * num_sms();
  return grid < 1 ? 1 : grid;
}

int layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, void* mean,
                  void* rstd, int rows, int h, cudaStream_t st) {
  if (h % 8 != 0 || h > 4096) return set_error(kErrConfig, "layernorm: h must be a multiple of 8, <= 4096");
  if (rows <= 0) return kOk;
  int nc = (h / 8 + 31) / 32;
  nc = nc <= 6 ? nc : (nc <= 8 ? 8 : (nc <= 10 ? 10 : (nc <= 12 ? 12 : 16)));
  const int grid = grid_for(rows, 8);
#define GX_LN_FWD(N)                                                                         \
  case N:                                                                                    \
    launch_k(layernorm_fwd_kernel<N>, dim3(grid), dim3(256), 0, st,                          \
             static_cast<const uint4*>(x), static_cast<const uint4*>(gamma),                 \
             static_cast<const uint4*>(beta), static_cast<uint4*>(y),                        \
             static_cast<float*>(mean), static_cast<float*>(rstd), rows, h);                 \
    break;
  switch (nc) {
    GX_LN_FWD(1) GX_LN_FWD(2) GX_LN_FWD(3) GX_LN_FWD(4) GX_LN_FWD(5) GX_LN_FWD(6)
    GX_LN_FWD(8) GX_LN_FWD(10) GX_LN_FWD(12) GX_LN_FWD(16)
    default: break;
  }
#undef GX_LN_FWD
  return check_launch("layernorm_fwd_kernel");
}

int layernorm_bwd(const void* dy, const void* x, const void* mean, const void* rstd,
                  const void* gamma, const void* dres, void* dx, void* dgamma, void* dbeta,
                  int rows, int h, float* workspace, cudaStream_t st, bool dy_f32) {
  if (h % 8 != 0 || h > 4096) return set_error(kErrConfig, "layernorm: h must be a multiple of 8, <= 4096");
  if (rows <= 0) return kOk;
  int nc = (h / 8 + 31) / 32;
  nc = nc <= 6 ? nc : (nc <= 8 ? 8 : (nc <= 10 ? 10 : (nc <= 12 ? 12 : 16)));
  const int grid = layernorm_bwd_blocks(rows);
  const int smem = 2 * h * 4;
#define GX_LN_BWD(N)                                                                          \
  case N:                                                                                     \
    launch_k(dy_f32 ? layernorm_bwd_kernel<N, true> : layernorm_bwd_kernel<N, false>,         \
             dim3(grid), dim3(256), smem, st, dy, static_cast<const uint4*>(x),               \
             static_cast<const float*>(mean), static_cast<const float*>(rstd),                \
             static_cast<const uint4*>(gamma), static_cast<const uint4*>(dres),               \
             static_cast<uint4*>(dx), workspace, rows, h);                                   \
    break;
  switch (nc) {
    GX_LN_BWD(1) GX_LN_BWD(2) GX_LN_BWD(3) GX_LN_BWD(4) GX_LN_BWD(5) GX_LN_BWD(6)
    GX_LN_BWD(8) GX_LN_BWD(10) GX_LN_BWD(12) GX_LN_BWD(16)
    default: break;
  }
#undef GX_LN_BWD
  GX_RC(check_launch("layernorm_bwd_kernel"));
  launch_k(layernorm_bwd_reduce_kernel, dim3((2 * h + 255) / 256), dim3(256), 0, st,
           static_cast<const float*>(workspace), grid, h, static_cast<float*>(dgamma),
           static_cast<float*>(dbeta));
  return check_launch("layernorm_bwd_reduce_kernel");
}

// -------------------------------------------------------- bias + dropout + residual
template <bool kF32In>
__global__ void bias_dropout_add_kernel(const void* __restrict__ x, const uint4* __restrict__ bias,
                                        const uint4* __restrict__ res, uint4* __restrict__ out,
                                        int rows, int cols, gx_dropout d) {
  pdl_enter();
  const int cchunks = cols >> 3;
  const int64_t n = static_cast<int64_t>(rows) * cchunks;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / cchunks), c = static_cast<int>(i % cchunks);
    float v[8], b[8], rr[8];
    load8<kF32In>(x, i, v);
    if (bias != nullptr) {
      unpack8(__ldg(bias + c), b);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += b[j];
    }
    if (d.threshold != 0u) {
      bool k[8];
      keep8(d, static_cast<uint64_t>(d.row_offset + r) * d.drop_ld + d.col_offset + c * 8, k);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = k[j] ? v[j] * d.scale : 0.f;
    }
    unpack8(res[i], rr);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(__float2bfloat16_rn(v[j])) + rr[j];
    out[i] = pack8(v);
  }
}

int bias_dropout_add(const void* x, const void* bias, const void* residual, void* out, int rows,
                     int cols, const gx_dropout& d, cudaStream_t st, bool x_f32) {
  if (cols % 8) return set_error(kErrConfig, "bias_dropout_add: cols % 8 != 0");
  const int64_t n = static_cast<int64_t>(rows) * (cols / 8);
  launch_k(x_f32 ? bias_dropout_add_kernel<true> : bias_dropout_add_kernel<false>,
           dim3(grid_for(n, 256)), dim3(256), 0, st, x, static_cast<const uint4*>(bias),
           static_cast<const uint4*>(residual), static_cast<uint4*>(out), rows, cols, d);
  return check_launch("bias_dropout_add_kernel");
}

// --------------------------------------------- dropout backward + bias-grad column sums
// Block handles a strip of 64 columns (8 chunks) over a slice of rows; column partials are
// reduced in shared memory then added to dbias with one atomic per column per block.
__global__ void __launch_bounds__(256) dropout_bwd_colsum_kernel(
    const uint4* __restrict__ dy, uint4* __restrict__ dz, float* __restrict__ dbias, int rows,
    int cols, int64_t ld_chunks, gx_dropout d, int rows_per_block) {
  pdl_enter();
  __shared__ float red[32][65];
  const int cchunks = cols >> 3;
  const int cstrip = blockIdx.x * 8;           // first chunk of this strip
  const int cc = cstrip + (threadIdx.x & 7);   // this thread's chunk
  const int rlane = threadIdx.x >> 3;          // 32 row lanes
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (cc < cchunks) {
    for (int r = r0 + rlane; r < r1; r += 32) {
      const int64_t i = static_cast<int64_t>(r) * ld_chunks + cc;
      float v[8];
      unpack8(dy[i], v);
      if (d.threshold != 0u) {
        bool k[8];
        keep8(d, static_cast<uint64_t>(d.row_offset + r) * d.drop_ld + d.col_offset + cc * 8, k);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = k[j] ? v[j] * d.scale : 0.f;
        const uint4 o = pack8(v);
        dz[i] = o;
        unpack8(o, v);  // column sums of the bf16 values actually used downstream
      } else if (dz != dy) {
        dz[i] = dy[i];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += v[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[rlane][(threadIdx.x & 7) * 8 + j] = acc[j];
  __syncthreads();
  if (threadIdx.x < 64) {
    float s = 0.f;
    for (int r = 0; r < 32; ++r) s += red[r][threadIdx.x];
    const int col = cstrip * 8 + threadIdx.x;
    if (dbias != nullptr && col < cols) atomicAdd(dbias + col, s);
  }
}

int dropout_bwd_colsum(const void* dy, void* dz, void* dbias, int rows, int cols,
                       const gx_dropout& d, cudaStream_t st) {
  if (cols % 8) return set_error(kErrConfig, "dropout_bwd: cols % 8 != 0");
  if (rows <= 0) return kOk;
  const int strips = (cols / 8 + 7) / 8;
  int ysplit = (num_sms() * 4 + strips - 1) / strips;
  const int max_y = (rows + 31) / 32;
  if (ysplit > max_y) ysplit = max_y;
  if (ysplit < 1) ysplit = 1;
  const int rpb = (rows + ysplit - 1) / ysplit;
  dim3 grid(strips, ysplit);
  launch_k(dropout_bwd_colsum_kernel, grid, dim3(256), 0, st, static_cast<const uint4*>(dy),
           static_cast<uint4*>(dz), static_cast<float*>(dbias), rows, cols,
           static_cast<int64_t>(cols / 8), d, rpb);
  return check_launch("dropout_bwd_colsum_kernel");
}

int colsum(const void* x, int64_t ld, void* acc, int rows, int cols, cudaStream_t st) {
  if (cols % 8 || ld % 8) return set_error(kErrConfig, "colsum: cols/ld % 8 != 0");
  if (rows <= 0) return kOk;
  gx_dropout off{};
  const int strips = (cols / 8 + 7) / 8;
  int ysplit = (num_sms() * 4 + strips - 1) / strips;
  const int max_y = (rows + 31) / 32;
  if (ysplit > max_y) ysplit = max_y;
  if (ysplit < 1) ysplit = 1;
  const int rpb = (rows + ysplit - 1) / ysplit;
  dim3 grid(strips, ysplit);
  launch_k(dropout_bwd_colsum_kernel, grid, dim3(256), 0, st, static_cast<const uint4*>(x),
           const_cast<uint4*>(static_cast<const uint4*>(x)), static_cast<float*>(acc), rows,
           cols, static_cast<int64_t>(ld / 8), off, rpb);
  return check_launch("colsum_kernel");
}

// ------------------------------------------------------------------------------ loss
__global__ void mse_loss_kernel(const uint4* __restrict__ y, const uint4* __restrict__ t,
                                uint4* __restrict__ dy, float* __restrict__ loss, int64_t n8,
                                float inv) {
  pdl_enter();
  float acc = 0.f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float a[8], b[8], g[8];
    unpack8(y[i], a);
    unpack8(t[i], b);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float d = a[j] - b[j];
      acc += d * d;
      g[j] = 2.f * d * inv;
    }
    dy[i] = pack8(g);
  }
  acc = warp_sum(acc);
  __shared__ float s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? s[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) atomicAdd(loss, v * inv);
  }
}

int mse_loss(const void* y, const void* target, void* dy, void* loss, int64_t n, float inv_count,
             cudaStream_t st) {
  if (n % 8) return set_error(kErrConfig, "mse_loss: n % 8 != 0");
  launch_k(mse_loss_kernel, dim3(grid_for(n / 8, 256)), dim3(256), 0, st,
           static_cast<const uint4*>(y), static_cast<const uint4*>(target),
           static_cast<uint4*>(dy), static_cast<float*>(loss), n / 8, inv_count);
  return check_launch("mse_loss_kernel");
}

// ------------------------------------------------------------------------------ AdamW
__global__ void adamw_kernel(float4* __restrict__ p, const float4* __restrict__ g,
                             float4* __restrict__ m, float4* __restrict__ v,
                             uint2* __restrict__ out, int64_t n4, float lr, float b1, float b2,
                             float eps, float wd, float bc1, float bc2) {
  pdl_enter();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 pp = p[i];
    const float4 gg = g[i];
    float4 mm = m[i], vv = v[i];
    float* pf = &pp.x;
    const float* gf = &gg.x;
    float* mf = &mm.x;
    float* vf = &vv.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mf[j] = b1 * mf[j] + (1.f - b1) * gf[j];
      vf[j] = b2 * vf[j] + (1.f - b2) * gf[j] * gf[j];
      const float mh = mf[j] / bc1, vh = vf[j] / bc2;
      pf[j] = pf[j] - lr * (mh / (sqrtf(vh) + eps) + wd * pf[j]);
    }
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
    out[i] = make_uint2(pk(pp.x, pp.y), pk(pp.z, pp.w));
  }
}

int adamw(void* master, const void* grad, void* m, void* v, void* bf16_out, int64_t n, float lr,
          float beta1, float beta2, float eps, float wd, float bc1, float bc2, cudaStream_t st) {
  if (n % 4) return set_error(kErrConfig, "adamw: n % 4 != 0");
  if (n == 0) return kOk;
  adamw_kernel<<<grid_for(n / 4, 256), 256, 0, st>>>(
      static_cast<float4*>(master), static_cast<const float4*>(grad), static_cast<float4*>(m),
      static_cast<float4*>(v), static_cast<uint2*>(bf16_out), n / 4, lr, beta1, beta2, eps, wd,
      bc1, bc2);
  return check_launch("adamw_kernel");
}

// Same update with the step count read from device memory (CUDA-graph friendly).
__global__ void adamw_dev_kernel(float4* __restrict__ p, const float4* __restrict__ g,
                                 float4* __restrict__ m, float4* __restrict__ v,
                                 uint2* __restrict__ out, int64_t n4, float lr, float b1, float b2,
                                 float eps, float wd, const int64_t* __restrict__ step) {
  pdl_enter();
  const float t = static_cast<float>(*step);
  const float bc1 = 1.f - powf(b1, t), bc2 = 1.f - powf(b2, t);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 pp = p[i];
    const float4 gg = g[i];
    float4 mm = m[i], vv = v[i];
    float* pf = &pp.x;
    const float* gf = &gg.x;
    float* mf = &mm.x;
    float* vf = &vv.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mf[j] = b1 * mf[j] + (1.f - b1) * gf[j];
      vf[j] = b2 * vf[j] + (1.f - b2) * gf[j] * gf[j];
      const float mh = mf[j] / bc1, vh = vf[j] / bc2;
      pf[j] = pf[j] - lr * (mh / (sqrtf(vh) + eps) + wd * pf[j]);
    }
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
    out[i] = make_uint2(pk(pp.x, pp.y), pk(pp.z, pp.w));
  }
}

int adamw_dev(void* master, const void* grad, void* m, void* v, void* bf16_out, int64_t n,
              float lr, float beta1, float beta2, float eps, float wd, const int64_t* step,
              cudaStream_t st, int max_blocks) {
  if (n % 4) return set_error(kErrConfig, "adamw: n % 4 != 0");
  if (n == 0) return kOk;
  int blocks = grid_for(n / 4, 256);
  if (max_blocks > 0 && blocks > max_blocks) blocks = max_blocks;
  launch_k(adamw_dev_kernel, dim3(blocks), dim3(256), 0, st,
           static_cast<float4*>(master), static_cast<const float4*>(grad),
           static_cast<float4*>(m), static_cast<float4*>(v), static_cast<uint2*>(bf16_out), n / 4,
           lr, beta1, beta2, eps, wd, step);
  return check_launch("adamw_dev_kernel");
}

__global__ void step_counters_kernel(int64_t* step, uint64_t* seed_offset) {
  pdl_enter();
  if (step != nullptr) *step += 1;
  if (seed_offset != nullptr) *seed_offset += 0x9E3779B97F4A7C15ull;
}

int bump_step(int64_t* step, uint64_t* seed_offset, cudaStream_t st) {
  step_counters_kernel<<<1, 1, 0, st>>>(step, seed_offset);
  return check_launch("step_counters_kernel");
}

// out[i] = sum_j src_j[i] for up to 16 sources (fp32 accumulate) — the simulated-world
// reduction used when several ranks share one device (collectives in "sim" comm mode).
template <typename T>
__global__ void sum_ptrs_kernel(PtrPack pk_, T* __restrict__ out, int64_t n) {
  pdl_enter();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < pk_.n; ++j) {
      if constexpr (sizeof(T) == 2) {
        acc += __bfloat162float(static_cast<const __nv_bfloat16*>(pk_.p[j])[i]);
      } else {
        acc += static_cast<const float*>(pk_.p[j])[i];
      }
    }
    if constexpr (sizeof(T) == 2) {
      out[i] = __float2bfloat16_rn(acc);
    } else {
      out[i] = acc;
    }
  }
}

int sum_ptrs(const PtrPack& srcs, void* out, int64_t n, bool bf16, cudaStream_t st) {
  if (n == 0) return kOk;
  if (bf16) {
    sum_ptrs_kernel<__nv_bfloat16><<<grid_for(n, 256), 256, 0, st>>>(
        srcs, static_cast<__nv_bfloat16*>(out), n);
  } else {
    sum_ptrs_kernel<float><<<grid_for(n, 256), 256, 0, st>>>(srcs, static_cast<float*>(out), n);
  }
  return check_launch("sum_ptrs_kernel");
}

__global__ void cast_bf16_kernel(const float4* __restrict__ s, uint2* __restrict__ d, int64_t n4) {
  pdl_enter();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 v = s[i];
    d[i] = make_uint2(pk(v.x, v.y), pk(v.z, v.w));
  }
}

int cast_bf16(const void* src, void* dst, int64_t n, cudaStream_t st) {
  if (n % 4) return set_error(kErrConfig, "cast_bf16: n % 4 != 0");
  if (n == 0) return kOk;
  cast_bf16_kernel<<<grid_for(n / 4, 256), 256, 0, st>>>(static_cast<const float4*>(src),
                                                         static_cast<uint2*>(dst), n / 4);
  return check_launch("cast_bf16_kernel");
}

}  // namespace gx
