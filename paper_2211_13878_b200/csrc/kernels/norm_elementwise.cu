// norm_elementwise.cu — the HBM-bound kernels of the layer: LayerNorm fwd/bwd, bias +
// dropout + residual, dropout backward with fused bias-gradient column sums, MSE loss,
// AdamW, casts.  All are one pass over their operands with 16-byte vector accesses; grids
// are sized in multiples of the SM count.  LayerNorm is one warp per row with the row held
// in registers (h <= 8192), statistics reduced with warp shuffles.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gx_internal.h"
#include "launch.cuh"
#include "sm100.cuh"
#include "adam.cuh"
#include "philox.cuh"

namespace gx {

namespace {

constexpr float kLnEps = 1e-5f;
// RMSNorm (T5): selected by a null `mean` pointer -- y = x * rsqrt(mean(x^2) + 1e-6) * gamma,
// no centring and no beta (its gradient is left untouched)
constexpr float kRmsEps = 1e-6f;

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

// fp32: the fixed-order sum of `slices` split-K slices `stride` elements apart
template <bool kF32>
__device__ __forceinline__ void load8s(const void* base, int64_t i, float (&f)[8], int slices,
                                       int64_t stride) {
  load8<kF32>(base, i, f);
  if constexpr (kF32) {
    for (int s = 1; s < slices; ++s) {
      float g[8];
      load8<true>(static_cast<const float*>(base) + s * stride, i, g);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += g[j];
    }
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
    const bool rms = mean == nullptr;
    const float mu = rms ? 0.f : warp_sum(s) / static_cast<float>(h);
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
    const float rs = rsqrtf(warp_sum(ss) / static_cast<float>(h) + (rms ? kRmsEps : kLnEps));
    uint4* yr = y + static_cast<int64_t>(r) * chunks;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ci = c * 32 + lane;
      if (ci < chunks) {
        float gm[8], bt[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, o[8];
        unpack8(__ldg(gamma + ci), gm);
        if (!rms) unpack8(__ldg(beta + ci), bt);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = (v[c][j] - mu) * rs * gm[j] + bt[j];
        yr[ci] = pack8(o);
      }
    }
    if (lane == 0) {
      if (!rms) mean[r] = mu;
      rstd[r] = rs;
    }
  }
}

int layernorm_fwd(const void* x, const void* gamma, const void* beta, void* y, void* mean,
                  void* rstd, int rows, int h, cudaStream_t st) {
  if (h % 8 != 0 || h > 8192) return set_error(kErrConfig, "layernorm: h must be a multiple of 8, <= 8192");
  if (rows <= 0) return kOk;
  int nc = (h / 8 + 31) / 32;
  nc = nc <= 6 ? nc : (nc <= 8 ? 8 : (nc <= 10 ? 10 : (nc <= 12 ? 12 : (nc <= 16 ? 16 : (nc <= 20 ? 20 : 32)))));
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
    GX_LN_FWD(8) GX_LN_FWD(10) GX_LN_FWD(12) GX_LN_FWD(16) GX_LN_FWD(20) GX_LN_FWD(32)
    default: break;
  }
#undef GX_LN_FWD
  return check_launch("layernorm_fwd_kernel");
}

// ---------------------------------------------------------------------- LayerNorm bwd
// Two passes, both deterministic (no floating-point atomics):
//  rows:    one warp per row computes dx = rstd * (g - mean(g) - xhat * mean(g * xhat)) + dres
//           with g = dy * gamma; with `drop` set it also emits dz = dropout_mask(dx), the
//           gradient entering the preceding bias + dropout (the dropout_bwd_colsum of dx,
//           fused in).
//  columns: dgamma += sum_r dy * xhat, dbeta += sum_r dy (and dbias += sum_r dz), computed by
//           (64-column strip x row slice) blocks; each writes its partial sums and the last
//           block of a strip (ticket counter) adds the slices in slice order.
// One block per row, one thread per 8-element chunk (h / 8 threads, rounded up to whole
// warps): every load of the row -- all split-K slices of dy included -- is issued at once,
// which is what a latency-bound 512-row problem needs; the two row sums go through a
// warp-shuffle + shared-memory reduction.
template <bool kF32Dy, bool kDrop, int kMaxThreads = 512>
__global__ void __launch_bounds__(kMaxThreads) layernorm_bwd_rows_kernel(
    const void* dy, const uint4* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ rstd, const uint4* __restrict__ gamma, const uint4* __restrict__ dres,
    uint4* __restrict__ dx, uint4* __restrict__ dz, gx_dropout d, int rows, int h, int dy_slices,
    int64_t dy_stride, float* __restrict__ dy_fold) {
  pdl_enter();
  __shared__ float red[2][kMaxThreads / 32];
  const int chunks = h >> 3;
  const int ci = threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int r = blockIdx.x;
  const bool active = ci < chunks;
  const int64_t i = static_cast<int64_t>(r) * chunks + ci;
  const bool rms = mean == nullptr;
  const float mu = rms ? 0.f : mean[r], rs = rstd[r];
  float xh[8], dv[8], gm[8], rv[8];
  float s1 = 0.f, s2 = 0.f;
  if (active) {
    load8<kF32Dy>(dy, i, dv);
    if constexpr (kF32Dy) {
      float acc[kMaxSplits - 1][8];
#pragma unroll
      for (int sl = 1; sl < kMaxSplits; ++sl)
        if (sl < dy_slices) load8<true>(static_cast<const float*>(dy) + sl * dy_stride, i, acc[sl - 1]);
#pragma unroll
      for (int sl = 1; sl < kMaxSplits; ++sl)
        if (sl < dy_slices) {
#pragma unroll
          for (int j = 0; j < 8; ++j) dv[j] += acc[sl - 1][j];
        }
      if (dy_slices > 1 && dy_fold == nullptr) {  // fold the slices into slice 0 for the column pass
        float4* o = reinterpret_cast<float4*>(const_cast<void*>(dy)) + 2 * i;
        o[0] = make_float4(dv[0], dv[1], dv[2], dv[3]);
        o[1] = make_float4(dv[4], dv[5], dv[6], dv[7]);
      }
    }
    if (dy_fold != nullptr) {  // fp32 dy for a deferred column pass
      float4* o = reinterpret_cast<float4*>(dy_fold) + 2 * i;
      o[0] = make_float4(dv[0], dv[1], dv[2], dv[3]);
      o[1] = make_float4(dv[4], dv[5], dv[6], dv[7]);
    }
    unpack8(x[i], xh);
    unpack8(__ldg(gamma + ci), gm);
    if (dres != nullptr) {
      unpack8(dres[i], rv);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) rv[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      xh[j] = (xh[j] - mu) * rs;
      const float g = dv[j] * gm[j];
      s1 += g;
      s2 += g * xh[j];
    }
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    red[0][warp] = s1;
    red[1][warp] = s2;
  }
  __syncthreads();
  float t1 = 0.f, t2 = 0.f;
  for (int w = 0; w < nwarps; ++w) {
    t1 += red[0][w];
    t2 += red[1][w];
  }
  if (!active) return;
  const float m1 = rms ? 0.f : t1 / static_cast<float>(h), m2 = t2 / static_cast<float>(h);
  float o[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j] = rs * (dv[j] * gm[j] - m1 - xh[j] * m2) + rv[j];
  const uint4 ob = pack8(o);
  dx[i] = ob;
  if constexpr (kDrop) {
    // identical arithmetic to dropout_bwd_colsum on the stored bf16 dx
    float v[8];
    unpack8(ob, v);
    if (d.threshold != 0u) {
      bool k[8];
      keep8(d, static_cast<uint64_t>(d.row_offset + r) * d.drop_ld + d.col_offset + ci * 8, k);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = k[j] ? v[j] * d.scale : 0.f;
    }
    dz[i] = pack8(v);
  }
}

template <bool kF32Dy, bool kDrop>
__global__ void __launch_bounds__(256) layernorm_bwd_cols_kernel(
    const void* __restrict__ dy, const uint4* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ rstd, const uint4* __restrict__ dz, float* __restrict__ dgamma,
    float* __restrict__ dbeta, float* __restrict__ dbias, float* __restrict__ ws,
    unsigned int* __restrict__ tickets, int rows, int h, int rows_per_slice, int dy_slices,
    int64_t dy_stride) {
  pdl_enter();
  constexpr int kParts = kDrop ? 3 : 2;
  __shared__ float red[32][kParts * 64 + 1];
  const int chunks = h >> 3;
  const int strip = blockIdx.x;
  const int cl = threadIdx.x & 7;       // chunk within the 64-column strip
  const int ci = strip * 8 + cl;        // global chunk index
  const int rlane = threadIdx.x >> 3;   // 32 row lanes
  const int r0 = blockIdx.y * rows_per_slice;
  const int r1 = min(rows, r0 + rows_per_slice);
  float ag[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ab[8] = {0, 0, 0, 0, 0, 0, 0, 0},
        az[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (ci < chunks) {
    for (int r = r0 + rlane; r < r1; r += 32) {
      const int64_t i = static_cast<int64_t>(r) * chunks + ci;
      float xv[8], dv[8];
      unpack8(x[i], xv);
      load8s<kF32Dy>(dy, i, dv, dy_slices, dy_stride);
      const float mu = mean != nullptr ? mean[r] : 0.f, rs = rstd[r];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ag[j] += dv[j] * ((xv[j] - mu) * rs);
        ab[j] += dv[j];
      }
      if constexpr (kDrop) {
        float zv[8];
        unpack8(dz[i], zv);
#pragma unroll
        for (int j = 0; j < 8; ++j) az[j] += zv[j];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    red[rlane][cl * 8 + j] = ag[j];
    red[rlane][64 + cl * 8 + j] = ab[j];
    if constexpr (kDrop) red[rlane][128 + cl * 8 + j] = az[j];
  }
  __syncthreads();
  const int width = kParts * h;
  const int slices = gridDim.y;
  // column t of this strip's partial: part t / 64, column strip*64 + t % 64
  const int t = threadIdx.x;
  const int col = strip * 64 + (t & 63);
  const bool owner = t < kParts * 64 && col < h;
  float s = 0.f;
  if (owner) {
    for (int rl = 0; rl < 32; ++rl) s += red[rl][t];
  }
  // RMSNorm (null mean): no beta, so its gradient is not touched
  float* outs[3] = {dgamma, mean != nullptr ? dbeta : nullptr, dbias};
  if (slices == 1) {
    if (owner && outs[t >> 6] != nullptr) outs[t >> 6][col] += s;
    return;
  }
  // the row slices of a strip form one cluster along y: slice 0 adds the slices' partials
  // in slice order over DSMEM (no global partials, fences or tickets)
  __shared__ float part_s[kParts * 64];
  if (t < kParts * 64) part_s[t] = s;
  cluster_sync();
  if (blockIdx.y == 0 && owner) {
    float acc = 0.f;
    for (int y = 0; y < slices; ++y)
      acc += ld_shared_cluster_f32(mapa_shared(smem_u32(&part_s[t]), y));
    if (outs[t >> 6] != nullptr) outs[t >> 6][col] += acc;
  }
  cluster_sync();  // the peers' shared memory stays alive until slice 0 has read it
  (void)ws;
  (void)tickets;
  (void)width;
}

constexpr int kLnColsClusterMax = 8;  // row slices of a strip: one portable cluster along y
static void ln_cols_grid(int rows, int h, int* strips, int* slices, int* rows_per_slice) {
  *strips = (h / 8 + 7) / 8;
  int ys = (2 * num_sms() + *strips - 1) / *strips;
  const int max_y = (rows + 31) / 32;
  if (ys > max_y) ys = max_y;
  if (ys > kLnColsClusterMax) ys = kLnColsClusterMax;
  if (ys < 1) ys = 1;
  *rows_per_slice = (rows + ys - 1) / ys;
  *slices = (rows + *rows_per_slice - 1) / *rows_per_slice;
}

// Workspace: kLnBwdTickets ticket words first (a fixed offset, so one workspace serves
// LayerNorms of different widths -- Swin stages), then [slices][3][h] fp32 partials.
constexpr int kLnBwdTickets = 256;  // one per 64-column strip: h <= 16384
int64_t layernorm_bwd_ws_floats(int h) {
  return kLnBwdTickets + static_cast<int64_t>(kLnBwdMaxSlices) * 3 * h;
}

int layernorm_bwd_rows(const void* dy, const void* x, const void* mean, const void* rstd,
                       const void* gamma, const void* dres, void* dx, int rows, int h,
                       cudaStream_t st, bool dy_f32, const gx_dropout* drop, void* dz,
                       int dy_slices, int64_t dy_slice_stride, float* dy_fold) {
  if (h % 8 != 0 || h > 8192) return set_error(kErrConfig, "layernorm: h must be a multiple of 8, <= 8192");
  if (rows <= 0) return kOk;
  if (dy_slices < 1 || dy_slices > kMaxSplits || (dy_slices > 1 && !dy_f32))
    return set_error(kErrConfig, "layernorm_bwd: dy slices need fp32 dy");
  const bool fuse = drop != nullptr;
  if (fuse && dz == nullptr) return set_error(kErrConfig, "layernorm_bwd: fused dropout needs dz");
  const gx_dropout dd = fuse ? *drop : gx_dropout{};
  const int threads = ((h / 8) + 31) / 32 * 32;  // <= 512 for h <= 4096, <= 1024 for 8192
  auto* krows = dy_f32 ? (fuse ? layernorm_bwd_rows_kernel<true, true> : layernorm_bwd_rows_kernel<true, false>)
                       : (fuse ? layernorm_bwd_rows_kernel<false, true> : layernorm_bwd_rows_kernel<false, false>);
  if (threads > 512) {  // wide rows (patch-merging LayerNorm over 4 x hidden/2 channels)
    if (fuse || dy_f32) return set_error(kErrConfig, "layernorm_bwd: h > 4096 needs plain bf16 dy");
    krows = layernorm_bwd_rows_kernel<false, false, 1024>;
  }
  launch_k(krows, dim3(rows), dim3(threads), 0, st, dy, static_cast<const uint4*>(x),
           static_cast<const float*>(mean), static_cast<const float*>(rstd),
           static_cast<const uint4*>(gamma), static_cast<const uint4*>(dres),
           static_cast<uint4*>(dx), static_cast<uint4*>(dz), dd, rows, h, dy_slices,
           dy_slice_stride, dy_fold);
  return check_launch("layernorm_bwd_rows_kernel");
}

int layernorm_bwd_cols(const void* dy, bool dy_f32, const void* x, const void* mean,
                       const void* rstd, const void* dz, void* dgamma, void* dbeta, void* dbias,
                       int rows, int h, float* workspace, cudaStream_t st) {
  if (rows <= 0) return kOk;
  const bool fuse = dz != nullptr;
  if (fuse && dbias == nullptr) return set_error(kErrConfig, "layernorm_bwd: dz needs dbias");
  int strips, slices, rps;
  ln_cols_grid(rows, h, &strips, &slices, &rps);
  unsigned int* tickets = reinterpret_cast<unsigned int*>(workspace);
  auto* kcols = dy_f32 ? (fuse ? layernorm_bwd_cols_kernel<true, true> : layernorm_bwd_cols_kernel<true, false>)
                       : (fuse ? layernorm_bwd_cols_kernel<false, true> : layernorm_bwd_cols_kernel<false, false>);
  launch_k_cluster_y(kcols, dim3(strips, slices), dim3(256), 0, st, static_cast<unsigned>(slices),
                     dy, static_cast<const uint4*>(x),
                     static_cast<const float*>(mean), static_cast<const float*>(rstd),
                     static_cast<const uint4*>(dz), static_cast<float*>(dgamma), static_cast<float*>(dbeta),
                     static_cast<float*>(dbias), workspace + kLnBwdTickets, tickets, rows, h, rps, 1,
                     int64_t{0});
  return check_launch("layernorm_bwd_cols_kernel");
}

int layernorm_bwd(const void* dy, const void* x, const void* mean, const void* rstd,
                  const void* gamma, const void* dres, void* dx, void* dgamma, void* dbeta,
                  int rows, int h, float* workspace, cudaStream_t st, bool dy_f32,
                  const gx_dropout* drop, void* dz, void* dbias, int dy_slices,
                  int64_t dy_slice_stride) {
  if (drop != nullptr && (dz == nullptr || dbias == nullptr))
    return set_error(kErrConfig, "layernorm_bwd: fused dropout needs dz and dbias");
  GX_RC(layernorm_bwd_rows(dy, x, mean, rstd, gamma, dres, dx, rows, h, st, dy_f32, drop, dz,
                           dy_slices, dy_slice_stride, nullptr));
  // the column pass reads slice 0, into which the row pass folded the slices
  return layernorm_bwd_cols(dy, dy_f32, x, mean, rstd, drop != nullptr ? dz : nullptr, dgamma,
                            dbeta, dbias, rows, h, workspace, st);
}

// -------------------------------------------------------- bias + dropout + residual
template <bool kF32In>
__global__ void bias_dropout_add_kernel(const void* __restrict__ x, const uint4* __restrict__ bias,
                                        const uint4* __restrict__ res, uint4* __restrict__ out,
                                        int rows, int cols, gx_dropout d, int x_slices,
                                        int64_t x_stride) {
  pdl_enter();
  const int cchunks = cols >> 3;
  const int64_t n = static_cast<int64_t>(rows) * cchunks;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / cchunks), c = static_cast<int>(i % cchunks);
    float v[8], b[8], rr[8];
    load8s<kF32In>(x, i, v, x_slices, x_stride);
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
                     int cols, const gx_dropout& d, cudaStream_t st, bool x_f32, int x_slices,
                     int64_t slice_stride) {
  if (cols % 8) return set_error(kErrConfig, "bias_dropout_add: cols % 8 != 0");
  if (x_slices < 1 || (x_slices > 1 && !x_f32))
    return set_error(kErrConfig, "bias_dropout_add: slices need fp32 x");
  const int64_t n = static_cast<int64_t>(rows) * (cols / 8);
  launch_k(x_f32 ? bias_dropout_add_kernel<true> : bias_dropout_add_kernel<false>,
           dim3(grid_for(n, 256)), dim3(256), 0, st, x, static_cast<const uint4*>(bias),
           static_cast<const uint4*>(residual), static_cast<uint4*>(out), rows, cols, d, x_slices,
           slice_stride);
  return check_launch("bias_dropout_add_kernel");
}

// ------------------------------------------- split-K sum + bias + dropout + residual + LN
// y = residual + bf16(dropout(sum_s x_s + bias)) for one row per block (thread per 8-column
// chunk), then -- when gamma is given -- the LayerNorm of the stored (bf16) y: ln, mean,
// rstd.  Replaces bias_dropout_add + layernorm_fwd after a split-K GEMM (out-projection ->
// LN2, MLP down-projection -> the next layer's LN1) with one pass over the row.
__global__ void __launch_bounds__(512) residual_layernorm_kernel(
    const float* __restrict__ x, int slices, int64_t stride, const uint4* __restrict__ bias,
    const uint4* __restrict__ res, uint4* __restrict__ y, gx_dropout d,
    const uint4* __restrict__ gamma, const uint4* __restrict__ beta, uint4* __restrict__ ln,
    float* __restrict__ mean, float* __restrict__ rstd, int rows, int h) {
  pdl_enter();
  __shared__ float red[16];
  const int chunks = h >> 3;
  const int ci = threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int r = blockIdx.x;
  const bool active = ci < chunks;
  const int64_t i = static_cast<int64_t>(r) * chunks + ci;
  float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (active) {
    load8<true>(x, i, v);
    float acc[kMaxSplits - 1][8];
#pragma unroll
    for (int sl = 1; sl < kMaxSplits; ++sl)
      if (sl < slices) load8<true>(x + sl * stride, i, acc[sl - 1]);
#pragma unroll
    for (int sl = 1; sl < kMaxSplits; ++sl)
      if (sl < slices) {
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] += acc[sl - 1][j];
      }
    float b[8], rr[8];
    if (bias != nullptr) {
      unpack8(__ldg(bias + ci), b);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += b[j];
    }
    if (d.threshold != 0u) {
      bool k[8];
      keep8(d, static_cast<uint64_t>(d.row_offset + r) * d.drop_ld + d.col_offset + ci * 8, k);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = k[j] ? v[j] * d.scale : 0.f;
    }
    unpack8(res[i], rr);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(__float2bfloat16_rn(v[j])) + rr[j];
    const uint4 yb = pack8(v);
    y[i] = yb;
    unpack8(yb, v);  // the LayerNorm sees the stored bf16 values
  }
  if (gamma == nullptr) return;
  // mean, then variance about it (two-pass, as layernorm_fwd); RMSNorm: no centring
  const bool rms = mean == nullptr;
  float s1 = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s1 += v[j];
  s1 = warp_sum(s1);
  if (lane == 0) red[warp] = s1;
  __syncthreads();
  float t = 0.f;
  for (int w = 0; w < nwarps; ++w) t += red[w];
  const float mu = rms ? 0.f : t / static_cast<float>(h);
  float s2 = 0.f;
  if (active) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float dd = v[j] - mu;
      s2 += dd * dd;
    }
  }
  s2 = warp_sum(s2);
  __syncthreads();
  if (lane == 0) red[warp] = s2;
  __syncthreads();
  float t2 = 0.f;
  for (int w = 0; w < nwarps; ++w) t2 += red[w];
  const float rs = rsqrtf(t2 / static_cast<float>(h) + (rms ? kRmsEps : kLnEps));
  if (active) {
    float gm[8], bt[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, o[8];
    unpack8(__ldg(gamma + ci), gm);
    if (!rms) unpack8(__ldg(beta + ci), bt);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (v[j] - mu) * rs * gm[j] + bt[j];
    ln[i] = pack8(o);
  }
  if (threadIdx.x == 0) {
    if (!rms) mean[r] = mu;
    rstd[r] = rs;
  }
}

int residual_layernorm(const float* x, int slices, int64_t slice_stride, const void* bias,
                       const void* residual, void* y, const gx_dropout& d, const void* gamma,
                       const void* beta, void* ln, void* mean, void* rstd, int rows, int h,
                       cudaStream_t st) {
  if (h % 8 != 0 || h > 4096) return set_error(kErrConfig, "residual_layernorm: h % 8 != 0 or h > 4096");
  if (slices < 1 || slices > kMaxSplits) return set_error(kErrConfig, "residual_layernorm: slices");
  if (rows <= 0) return kOk;
  const int threads = ((h / 8) + 31) / 32 * 32;
  launch_k(residual_layernorm_kernel, dim3(rows), dim3(threads), 0, st, x, slices, slice_stride,
           static_cast<const uint4*>(bias), static_cast<const uint4*>(residual),
           static_cast<uint4*>(y), d, static_cast<const uint4*>(gamma),
           static_cast<const uint4*>(beta), static_cast<uint4*>(ln), static_cast<float*>(mean),
           static_cast<float*>(rstd), rows, h);
  return check_launch("residual_layernorm_kernel");
}

// --------------------------------------------- dropout backward + bias-grad column sums
// Block = (64-column strip, row slice): 8 chunks x 32 row lanes accumulate, the 32 lanes are
// combined in shared memory in a fixed order, and the slices of a strip (one cluster) are
// added in slice order over DSMEM -- deterministic, no floating-point atomics.  (ws: unused,
// kept in the signature of the C ABI entry points.)
__global__ void __launch_bounds__(256) dropout_bwd_colsum_kernel(
    const uint4* __restrict__ dy, uint4* __restrict__ dz, float* __restrict__ dbias, int rows,
    int cols, int64_t ld_chunks, gx_dropout d, int rows_per_block, float* __restrict__ ws) {
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
    // four rows' loads in flight before any is used (a lane strides 32 rows)
    int r = r0 + rlane;
    for (; r + 96 < r1; r += 128) {
      uint4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = dy[static_cast<int64_t>(r + 32 * u) * ld_chunks + cc];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = static_cast<int64_t>(r + 32 * u) * ld_chunks + cc;
        float v[8];
        unpack8(x[u], v);
        if (d.threshold != 0u) {
          bool k[8];
          keep8(d, static_cast<uint64_t>(d.row_offset + r + 32 * u) * d.drop_ld + d.col_offset + cc * 8, k);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = k[j] ? v[j] * d.scale : 0.f;
          const uint4 o = pack8(v);
          dz[i] = o;
          unpack8(o, v);
        } else if (dz != dy) {
          dz[i] = x[u];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += v[j];
      }
    }
    for (; r < r1; r += 32) {
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
  const int col = cstrip * 8 + threadIdx.x;  // threads 0..63 own the strip's columns
  float sum = 0.f;
  if (threadIdx.x < 64) {
    for (int rl = 0; rl < 32; ++rl) sum += red[rl][threadIdx.x];
  }
  if (dbias == nullptr) return;
  if (gridDim.y == 1) {
    if (threadIdx.x < 64 && col < cols) dbias[col] += sum;
    return;
  }
  // The row slices of a strip form one thread-block cluster along y: each slice leaves its 64
  // column sums in shared memory, and slice 0 adds them in slice order over DSMEM after a
  // cluster barrier -- no global partials, fences or tickets on the path.
  __shared__ float part_s[64];
  if (threadIdx.x < 64) part_s[threadIdx.x] = sum;
  cluster_sync();
  if (blockIdx.y == 0 && threadIdx.x < 64 && col < cols) {
    float t = 0.f;
    for (int y = 0; y < static_cast<int>(gridDim.y); ++y)
      t += ld_shared_cluster_f32(mapa_shared(smem_u32(&part_s[threadIdx.x]), y));
    dbias[col] += t;
  }
  cluster_sync();  // the peers' shared memory stays alive until slice 0 has read it
  (void)ws;
}

constexpr int kColsumSlicesUsed = 8;  // (<= 8: a portable cluster along y)

// the column-sum kernel, its row slices clustered along y when there is more than one
static void launch_colsum(dim3 grid, cudaStream_t st, const uint4* dy, uint4* dz, float* dbias,
                          int rows, int cols, int64_t ld_chunks, const gx_dropout& d, int rpb,
                          float* ws) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (grid.y > 1 && dbias != nullptr) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = 1;
    attr[n].val.clusterDim.y = grid.y;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  cudaLaunchKernelEx(&cfg, dropout_bwd_colsum_kernel, dy, dz, dbias, rows, cols, ld_chunks, d,
                     rpb, ws);
}
static void colsum_grid(int rows, int cols, dim3* grid, int* rpb) {
  const int strips = (cols / 8 + 7) / 8;
  int ysplit = num_sms() / strips;  // about one wave of blocks
  const int max_y = (rows + 31) / 32;
  if (ysplit > max_y) ysplit = max_y;
  if (ysplit > kColsumSlicesUsed) ysplit = kColsumSlicesUsed;  // fewer, longer slices measured best
  if (ysplit < 1) ysplit = 1;
  *rpb = (rows + ysplit - 1) / ysplit;
  *grid = dim3(strips, (rows + *rpb - 1) / *rpb);
}

int64_t colsum_ws_floats(int max_cols) {
  return kColsumTickets + static_cast<int64_t>(kColsumMaxSlices) * max_cols;
}

int dropout_bwd_colsum(const void* dy, void* dz, void* dbias, int rows, int cols,
                       const gx_dropout& d, cudaStream_t st, float* ws) {
  if (cols % 8) return set_error(kErrConfig, "dropout_bwd: cols % 8 != 0");
  if (cols / 64 + 1 > kColsumTickets) return set_error(kErrConfig, "dropout_bwd: too many columns");
  if (rows <= 0) return kOk;
  dim3 grid;
  int rpb;
  colsum_grid(rows, cols, &grid, &rpb);
  launch_colsum(grid, st, static_cast<const uint4*>(dy), static_cast<uint4*>(dz),
                static_cast<float*>(dbias), rows, cols, static_cast<int64_t>(cols / 8), d, rpb, ws);
  return check_launch("dropout_bwd_colsum_kernel");
}

int colsum(const void* x, int64_t ld, void* acc, int rows, int cols, cudaStream_t st, float* ws) {
  if (cols % 8 || ld % 8) return set_error(kErrConfig, "colsum: cols/ld % 8 != 0");
  if (cols / 64 + 1 > kColsumTickets) return set_error(kErrConfig, "colsum: too many columns");
  if (rows <= 0) return kOk;
  gx_dropout off{};
  dim3 grid;
  int rpb;
  colsum_grid(rows, cols, &grid, &rpb);
  launch_colsum(grid, st, static_cast<const uint4*>(x), const_cast<uint4*>(static_cast<const uint4*>(x)),
                static_cast<float*>(acc), rows, cols, static_cast<int64_t>(ld / 8), off, rpb, ws);
  return check_launch("colsum_kernel");
}

// ------------------------------------------------------------------------------ loss
// Deterministic: a fixed grid writes one partial per block; the last block to finish (ticket)
// adds them in block order, so the loss is bit-reproducible run to run.
__global__ void __launch_bounds__(256) mse_loss_kernel(const uint4* __restrict__ y,
                                                       const uint4* __restrict__ t,
                                                       uint4* __restrict__ dy,
                                                       float* __restrict__ loss, int64_t n8,
                                                       float inv, float* __restrict__ partials,
                                                       unsigned int* __restrict__ ticket) {
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
  __shared__ float s[8];
  __shared__ bool last;
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += s[w];
    partials[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    float v = 0.f;
    for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += 32)
      v += *reinterpret_cast<volatile float*>(partials + b);
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      *loss += v * inv;
      *ticket = 0u;  // ready for the next call (graph replays)
    }
  }
}

int mse_loss(const void* y, const void* target, void* dy, void* loss, int64_t n, float inv_count,
             cudaStream_t st, float* workspace) {
  if (n % 8) return set_error(kErrConfig, "mse_loss: n % 8 != 0");
  int grid = grid_for(n / 8, 256);
  if (grid > kLossBlocks) grid = kLossBlocks;
  launch_k(mse_loss_kernel, dim3(grid), dim3(256), 0, st, static_cast<const uint4*>(y),
           static_cast<const uint4*>(target), static_cast<uint4*>(dy), static_cast<float*>(loss),
           n / 8, inv_count, workspace, reinterpret_cast<unsigned int*>(workspace + kLossBlocks));
  return check_launch("mse_loss_kernel");
}

// ------------------------------------------------------------------------------ AdamW
// p <- p - lr * (m_hat / (sqrt(v_hat) + eps) + wd * p), restated with the bias corrections
// folded into two per-launch scalars (step_size = lr / bc1, 1/sqrt(bc2)) so the per-element
// work is FMAs, one sqrt and one fast divide: the kernel shares the SMs with the backward
// GEMMs, so its issue cost matters as much as its 30 B/param of HBM traffic.
// kU float4 per thread per iteration: 4*kU independent 16-byte loads in flight per thread, so
// a small (SM-slot-frugal) grid still keeps HBM busy while the backward runs beside it
template <int kU>
__device__ __forceinline__ void adam_range(const AdamScalars& c, float4* __restrict__ p,
                                           const float4* __restrict__ g, float4* __restrict__ m,
                                           float4* __restrict__ v, uint2* __restrict__ out,
                                           int64_t n4) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (; i + (kU - 1) * stride < n4; i += kU * stride) {
    float4 pp[kU], gg[kU], mm[kU], vv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      pp[u] = p[i + u * stride];
      gg[u] = g[i + u * stride];
      mm[u] = m[i + u * stride];
      vv[u] = v[i + u * stride];
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      adam4(c, pp[u], gg[u], mm[u], vv[u]);
      p[i + u * stride] = pp[u];
      m[i + u * stride] = mm[u];
      v[i + u * stride] = vv[u];
      out[i + u * stride] = make_uint2(pk(pp[u].x, pp[u].y), pk(pp[u].z, pp[u].w));
    }
  }
  for (; i < n4; i += stride) {
    float4 p0 = p[i];
    const float4 g0 = g[i];
    float4 m0 = m[i], v0 = v[i];
    adam4(c, p0, g0, m0, v0);
    p[i] = p0;
    m[i] = m0;
    v[i] = v0;
    out[i] = make_uint2(pk(p0.x, p0.y), pk(p0.z, p0.w));
  }
}

__global__ void adamw_kernel(float4* __restrict__ p, const float4* __restrict__ g,
                             float4* __restrict__ m, float4* __restrict__ v,
                             uint2* __restrict__ out, int64_t n4, float lr, float b1, float b2,
                             float eps, float wd, float bc1, float bc2) {
  pdl_enter();
  adam_range<2>(adam_scalars(lr, b1, b2, eps, wd, bc1, bc2), p, g, m, v, out, n4);
}

int adamw(void* master, const void* grad, void* m, void* v, void* bf16_out, int64_t n, float lr,
          float beta1, float beta2, float eps, float wd, float bc1, float bc2, cudaStream_t st) {
  if (n % 4) return set_error(kErrConfig, "adamw: n % 4 != 0");
  if (n == 0) return kOk;
  launch_k(adamw_kernel, dim3(grid_for(n / 8, 256)), dim3(256), 0, st,
           static_cast<float4*>(master), static_cast<const float4*>(grad), static_cast<float4*>(m),
           static_cast<float4*>(v), static_cast<uint2*>(bf16_out), n / 4, lr, beta1, beta2, eps,
           wd, bc1, bc2);
  return check_launch("adamw_kernel");
}

// Same update with the step count read from device memory (CUDA-graph friendly).
// <= 64 registers (256 x 64 = 16K): a block fits beside a 128-register GEMM CTA (48K), so
// the optimizer can share SMs with the backward instead of waiting for whole free SMs.
__global__ void __launch_bounds__(256, 4) adamw_dev_kernel(float4* __restrict__ p, const float4* __restrict__ g,
                                 float4* __restrict__ m, float4* __restrict__ v,
                                 uint2* __restrict__ out, int64_t n4, float lr, float b1, float b2,
                                 float eps, float wd, const int64_t* __restrict__ step) {
  pdl_enter();
  adam_range<2>(adam_scalars_step(lr, b1, b2, eps, wd, step), p, g, m, v,
             out, n4);
}

int adamw_dev(void* master, const void* grad, void* m, void* v, void* bf16_out, int64_t n,
              float lr, float beta1, float beta2, float eps, float wd, const int64_t* step,
              cudaStream_t st, int max_blocks) {
  if (n % 4) return set_error(kErrConfig, "adamw: n % 4 != 0");
  if (n == 0) return kOk;
  // Short-lived blocks (one 4-float4 strip per thread, no grid-stride loop): the block
  // scheduler can hand every SM freed by this kernel back to the higher-priority backward
  // stream, instead of long-resident optimizer blocks pinning SMs for the whole update.
  const int64_t per_block = 256 * 4;
  int64_t nb = (n / 4 + per_block - 1) / per_block;
  if (nb > (1ll << 30)) nb = 1ll << 30;
  int blocks = static_cast<int>(nb);
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
