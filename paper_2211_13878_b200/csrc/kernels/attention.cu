// attention.cu — fused multi-head self-attention forward / backward (flash-style, exact).
//
//   ctx = dropout(softmax(Q K^T / sqrt(d))) V      per (sample, head), no materialised S
//
// Layout: qkv rows are tokens ([M = b*s][3][H][d], row stride ld_qkv), ctx rows [M][H*d].
// Forward keeps a running (max, sum) per query row and stores lse (log2 domain) for the
// backward, which recomputes P = exp2(S*c - lse) per key block (FA2 scheme: each CTA owns a
// block of keys, accumulates dK/dV in registers and adds dQ into an fp32 buffer).
// Dropout (philox.cuh byte scheme): the forward thread that owns query row q and lane t of a
// 64-key block kb draws ONE Philox call, counter ((bh*s + q)*ceil(s/64) + kb)*4 + t with
// bh = global_sample*H_tot + global_head, whose 16 bytes decide its 16 elements: key
// kb*64 + 8*(j/2) + 2*t + (j%2) for byte j.  The forward stores those 16 keep bits (uint16,
// [b*H][s][ceil(s/64)][4]) and the backward reads them back instead of re-drawing.  Masks
// depend only on global (sample, head, q, k), so any TP/DP split reproduces them exactly.
//
// Tensor-core path: mma.sync m16n8k16 bf16 with ldmatrix fragments.  (A tcgen05/TMEM
// variant is the planned next step; attention is ~7% of the layer FLOPs at s=512.)
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gx_internal.h"
#include "launch.cuh"
#include "philox.cuh"

namespace gx {

namespace {

constexpr int kBlk = 64;      // queries (fwd) / keys (bwd) per CTA, 16 per warp
constexpr int kThreads = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 t = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&t);
}

// Loads a [64][HD] tile of rows [r0, r0+64) (rows >= nrows zero-filled) into padded smem.
template <int HD>
__device__ __forceinline__ void load_tile(__nv_bfloat16* dst, const __nv_bfloat16* src,
                                          int64_t ld, int r0, int nrows) {
  constexpr int kChunks = HD / 8;  // 16 B per chunk
  for (int i = threadIdx.x; i < kBlk * kChunks; i += kThreads) {
    const int r = i / kChunks, c = i % kChunks;
    const bool ok = r0 + r < nrows;
    const __nv_bfloat16* g = src + static_cast<int64_t>(ok ? r0 + r : 0) * ld + c * 8;
    cp_async16(dst + r * (HD + 8) + c * 8, g, ok);
  }
}

// Swin shifted-window region (0..8) of token `tok` of attention sequence (window) `b`: the
// window's position in the rolled grid gives the token's (y, x); rows / columns within
// `side` of the far edge came from the other side of the grid (SW-MSA attention mask).
__device__ __forceinline__ int swin_region(const gx_attention_args& p, int b, int tok) {
  const int nw = p.win_grid / p.win_side;
  const int w = b % (nw * nw);
  const int y = (w / nw) * p.win_side + tok / p.win_side;
  const int x = (w % nw) * p.win_side + tok % p.win_side;
  const int l0 = p.win_grid - p.win_side, l1 = p.win_grid - p.win_shift;
  return (y < l0 ? 0 : (y < l1 ? 1 : 2)) * 3 + (x < l0 ? 0 : (x < l1 ? 1 : 2));
}

// Relative-position bias staged in shared memory per CTA (one head): the head's table in log2
// units and each window token's (y, x), so a score's bias is two byte loads and one table load.
constexpr int kRpbMaxTab = 15 * 15;  // (2 * 8 - 1)^2: windows of up to 8 x 8 tokens
struct RpbSmem {
  float tab[kRpbMaxTab];
  int8_t y[64], x[64];  // token -> (row, column) inside its window (rel-pos bias)
  int8_t reg[64];       // token -> shifted-window region of this CTA's window (SW-MSA mask)
};
// Per-CTA staging of the window masks / bias: attention sequence b (one window), head h.
__device__ __forceinline__ void win_stage(const gx_attention_args& p, int b, int h, RpbSmem* r) {
  if (p.rpb != nullptr) {
    const int w = p.rpb_side, n = 2 * w - 1;
    const auto* t = static_cast<const __nv_bfloat16*>(p.rpb) + h * n * n;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x)
      r->tab[e] = __bfloat162float(t[e]) * 1.4426950408889634f;
    for (int i = threadIdx.x; i < 64; i += blockDim.x) {
      r->y[i] = static_cast<int8_t>(i / w);
      r->x[i] = static_cast<int8_t>(i % w);
    }
  }
  if (p.win_shift > 0)
    for (int i = threadIdx.x; i < 64; i += blockDim.x)
      r->reg[i] = static_cast<int8_t>(i < p.seq ? swin_region(p, b, i) : 0);
}
__device__ __forceinline__ float rpb_bias(const gx_attention_args& p, const RpbSmem* r, int q,
                                          int k) {
  const int w = p.rpb_side;
  return r->tab[(r->y[q] - r->y[k] + w - 1) * (2 * w - 1) + (r->x[q] - r->x[k] + w - 1)];
}

}  // namespace

// --------------------------------------------------------------------------- forward
// kMask: causal / shifted-window masking compiled in only when used (register pressure)
template <int HD, bool kMask>
__global__ void __launch_bounds__(kThreads) attn_fwd_kernel(const gx_attention_args p) {
  pdl_enter();
  constexpr int LDS = HD + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sK = sQ + kBlk * LDS;        // [2][64][LDS]
  __nv_bfloat16* sV = sK + 2 * kBlk * LDS;    // [2][64][LDS]
  RpbSmem* sRp = reinterpret_cast<RpbSmem*>(sV + 2 * kBlk * LDS);  // (kMask: shift / rpb)

  const int s = p.seq;
  const int H = p.heads;
  const int bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int q0 = blockIdx.x * kBlk;
  if (kMask) win_stage(p, b, h, sRp);  // visible after the first tile barrier
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;

  const auto* qkv = static_cast<const __nv_bfloat16*>(p.qkv);
  const int64_t ld = p.ld_qkv;
  const __nv_bfloat16* Qg = qkv + static_cast<int64_t>(b) * s * ld + h * HD;
  const __nv_bfloat16* Kg = Qg + static_cast<int64_t>(H) * HD;
  const __nv_bfloat16* Vg = Kg + static_cast<int64_t>(H) * HD;

  load_tile<HD>(sQ, Qg, ld, q0, s);
  load_tile<HD>(sK, Kg, ld, 0, s);
  load_tile<HD>(sV, Vg, ld, 0, s);
  cp_async_commit();

  const float c2 = p.scale * 1.4426950408889634f;  // softmax scale in log2 units
  const uint32_t thr = p.drop_threshold;
  const float inv_keep = p.drop_scale;
  const uint64_t seed = p.seed + (p.seed_offset != nullptr ? *p.seed_offset : 0ull);
  const uint64_t stream =
      (static_cast<uint64_t>(p.sample_offset + b) * p.heads_total + (p.head_offset + h)) * s;
  const int nkb = (s + kBlk - 1) / kBlk;
  uint16_t* mask = static_cast<uint16_t*>(p.mask);

  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];

  for (int kb = 0; kb < nkb; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nkb) {
      load_tile<HD>(sK + (buf ^ 1) * kBlk * LDS, Kg, ld, (kb + 1) * kBlk, s);
      load_tile<HD>(sV + (buf ^ 1) * kBlk * LDS, Vg, ld, (kb + 1) * kBlk, s);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        ldsm_x4(qf[kk], sQ + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
    }
    const __nv_bfloat16* cK = sK + buf * kBlk * LDS;
    const __nv_bfloat16* cV = sV + buf * kBlk * LDS;

    float sacc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) sacc[i][0] = sacc[i][1] = sacc[i][2] = sacc[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t kf[4];
        ldsm_x4(kf, cK + (np * 16 + (lane & 7) + ((lane >> 4) << 3)) * LDS + kk * 16 +
                        ((lane >> 3) & 1) * 8);
        mma_bf16(sacc[2 * np], qf[kk], kf[0], kf[1]);
        mma_bf16(sacc[2 * np + 1], qf[kk], kf[2], kf[3]);
      }
    }
    // scale, mask key tail, online softmax
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int key = kb * kBlk + nb * 8 + 2 * t + (j & 1);
        float v = sacc[nb][j] * c2;
        const int qrow = q0 + warp * 16 + g + 8 * (j >> 1);
        if (kMask && p.rpb != nullptr && key < s && qrow < s) v += rpb_bias(p, sRp, qrow, key);
        if (key >= s || (kMask && ((p.causal && key > qrow) ||
                                   (p.win_shift > 0 && key < s && qrow < s &&
                                    sRp->reg[qrow] != sRp->reg[key]))))
          v = -INFINITY;
        sacc[nb][j] = v;
        mx[j >> 1] = fmaxf(mx[j >> 1], v);
      }
    }
    float corr[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 2));
      const float m_new = fmaxf(m_r[r], mx[r]);
      corr[r] = exp2f(m_r[r] - m_new);
      m_r[r] = m_new;
    }
    float rs[2] = {0.f, 0.f};
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float e = exp2f(sacc[nb][j] - m_r[j >> 1]);
        sacc[nb][j] = e;
        rs[j >> 1] += e;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) l_r[r] = l_r[r] * corr[r] + rs[r];  // quad-partial sums
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= corr[0];
      o[i][1] *= corr[0];
      o[i][2] *= corr[1];
      o[i][3] *= corr[1];
    }
    if (thr != 0u) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int q = q0 + warp * 16 + g + 8 * r;
        const uint64_t call = ((stream + static_cast<uint64_t>(q)) * nkb + kb) * 4 + t;
        const uint32_t bits = keep16(seed, p.site, call, thr);
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
          sacc[nb][2 * r] = (bits >> (2 * nb)) & 1u ? sacc[nb][2 * r] * inv_keep : 0.f;
          sacc[nb][2 * r + 1] = (bits >> (2 * nb + 1)) & 1u ? sacc[nb][2 * r + 1] * inv_keep : 0.f;
        }
        if (q < s) mask[((static_cast<int64_t>(bh) * s + q) * nkb + kb) * 4 + t] =
            static_cast<uint16_t>(bits);
      }
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // 16 keys per step
      uint32_t pa[4];
      pa[0] = pack2(sacc[2 * kk][0], sacc[2 * kk][1]);
      pa[1] = pack2(sacc[2 * kk][2], sacc[2 * kk][3]);
      pa[2] = pack2(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
      pa[3] = pack2(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < HD / 16; ++np) {
        uint32_t vf[4];
        ldsm_x4_t(vf, cV + (kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + np * 16 +
                          (lane >> 4) * 8);
        mma_bf16(o[2 * np], pa, vf[0], vf[1]);
        mma_bf16(o[2 * np + 1], pa, vf[2], vf[3]);
      }
    }
    __syncthreads();
  }
  // finalize
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l_r[r] += __shfl_xor_sync(0xffffffff, l_r[r], 1);
    l_r[r] += __shfl_xor_sync(0xffffffff, l_r[r], 2);
  }
  auto* ctx = static_cast<__nv_bfloat16*>(p.ctx);
  auto* lse = static_cast<float*>(p.lse);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int q = q0 + warp * 16 + g + 8 * r;
    if (q >= s) continue;
    const float inv = 1.f / l_r[r];
    __nv_bfloat16* out = ctx + (static_cast<int64_t>(b) * s + q) * p.ld_ctx + h * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      *reinterpret_cast<uint32_t*>(out + i * 8 + 2 * t) =
          pack2(o[i][2 * r] * inv, o[i][2 * r + 1] * inv);
    }
    if (t == 0) lse[static_cast<int64_t>(bh) * s + q] = m_r[r] + log2f(l_r[r]);
  }
}

// -------------------------------------------------------------- backward pre-process
// D[bh][q] = sum_d dctx*ctx ; zero the fp32 dQ accumulator.
template <int HD>
__global__ void attn_bwd_prep_kernel(const gx_attention_args p) {
  pdl_enter();
  const int s = p.seq, H = p.heads;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int total = p.batch * H * s;
  if (warp_global >= total) return;
  const int bh = warp_global / s, q = warp_global % s;
  const int b = bh / H, h = bh % H;
  const int64_t row = static_cast<int64_t>(b) * s + q;
  const auto* o = static_cast<const __nv_bfloat16*>(p.ctx) + row * p.ld_ctx + h * HD;
  const auto* d = static_cast<const __nv_bfloat16*>(p.dctx) + row * p.ld_ctx + h * HD;
  float acc = 0.f;
  for (int i = lane; i < HD; i += 32) acc += __bfloat162float(o[i]) * __bfloat162float(d[i]);
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, m);
  if (lane == 0) static_cast<float*>(p.dsum)[static_cast<int64_t>(bh) * s + q] = acc;
  float* dq = static_cast<float*>(p.dq_accum) + (static_cast<int64_t>(bh) * s + q) * HD;
  for (int i = lane; i < HD; i += 32) dq[i] = 0.f;
}

// --------------------------------------------------------------------------- backward
template <int HD, bool kMask>
__global__ void __launch_bounds__(kThreads) attn_bwd_kernel(const gx_attention_args p) {
  pdl_enter();
  constexpr int LDS = HD + 8;
  constexpr int LDP = kBlk + 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sV = sK + kBlk * LDS;
  __nv_bfloat16* sQ = sV + kBlk * LDS;
  __nv_bfloat16* sdO = sQ + kBlk * LDS;
  __nv_bfloat16* sdS = sdO + kBlk * LDS;                              // [64 keys][LDP]
  float* sL = reinterpret_cast<float*>(sdS + kBlk * LDP);             // lse [64]
  float* sD = sL + kBlk;                                              // D   [64]
  uint16_t* sM = reinterpret_cast<uint16_t*>(sD + kBlk);              // keep bits [64][4]
  float* sRB = reinterpret_cast<float*>(sM + kBlk * 4);  // rel-pos bias: dS tile [64][64] (kMask)
  RpbSmem* sRp = reinterpret_cast<RpbSmem*>(sRB + kBlk * kBlk);

  const int s = p.seq, H = p.heads;
  const int bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int k0 = blockIdx.x * kBlk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  if (kMask) win_stage(p, b, h, sRp);  // visible after the first tile barrier

  const auto* qkv = static_cast<const __nv_bfloat16*>(p.qkv);
  const int64_t ld = p.ld_qkv;
  const __nv_bfloat16* Qg = qkv + static_cast<int64_t>(b) * s * ld + h * HD;
  const __nv_bfloat16* Kg = Qg + static_cast<int64_t>(H) * HD;
  const __nv_bfloat16* Vg = Kg + static_cast<int64_t>(H) * HD;
  const __nv_bfloat16* dOg =
      static_cast<const __nv_bfloat16*>(p.dctx) + static_cast<int64_t>(b) * s * p.ld_ctx + h * HD;
  const float* lse = static_cast<const float*>(p.lse) + static_cast<int64_t>(bh) * s;
  const float* dsum = static_cast<const float*>(p.dsum) + static_cast<int64_t>(bh) * s;
  float* dqacc = static_cast<float*>(p.dq_accum) + static_cast<int64_t>(bh) * s * HD;

  load_tile<HD>(sK, Kg, ld, k0, s);
  load_tile<HD>(sV, Vg, ld, k0, s);
  cp_async_commit();

  const float c2 = p.scale * 1.4426950408889634f;
  const uint32_t thr = p.drop_threshold;
  const float inv_keep = p.drop_scale;
  const int nkb = (s + kBlk - 1) / kBlk;
  const int kbi = blockIdx.x;
  const uint16_t* mask = static_cast<const uint16_t*>(p.mask);

  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) dk[i][j] = dv[i][j] = 0.f;
  uint32_t kf[HD / 16][4], vfr[HD / 16][4];

  const int nqb = (s + kBlk - 1) / kBlk;
  for (int qb = 0; qb < nqb; ++qb) {
    const int q0 = qb * kBlk;
    load_tile<HD>(sQ, Qg, ld, q0, s);
    load_tile<HD>(sdO, dOg, p.ld_ctx, q0, s);
    for (int i = threadIdx.x; i < kBlk; i += kThreads) {
      const bool ok = q0 + i < s;
      sL[i] = ok ? lse[q0 + i] : 0.f;
      sD[i] = ok ? dsum[q0 + i] : 0.f;
    }
    if (thr != 0u) {
      for (int i = threadIdx.x; i < kBlk * 4; i += kThreads) {
        const int qi = i >> 2;
        sM[i] = q0 + qi < s ? mask[((static_cast<int64_t>(bh) * s + q0 + qi) * nkb + kbi) * 4 + (i & 3)]
                            : static_cast<uint16_t>(0);
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (qb == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        ldsm_x4(kf[kk], sK + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
        ldsm_x4(vfr[kk], sV + (warp * 16 + (lane & 15)) * LDS + kk * 16 + (lane >> 4) * 8);
      }
    }
    // S^T = K Q^T and dP^T = V dO^T : 16 keys x 64 queries per warp
    float st[8][4], dpt[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) st[i][j] = dpt[i][j] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t qf[4], of[4];
        const int row = np * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int col = kk * 16 + ((lane >> 3) & 1) * 8;
        ldsm_x4(qf, sQ + row * LDS + col);
        ldsm_x4(of, sdO + row * LDS + col);
        mma_bf16(st[2 * np], kf[kk], qf[0], qf[1]);
        mma_bf16(st[2 * np + 1], kf[kk], qf[2], qf[3]);
        mma_bf16(dpt[2 * np], vfr[kk], of[0], of[1]);
        mma_bf16(dpt[2 * np + 1], vfr[kk], of[2], of[3]);
      }
    }
    // P^T, dropout, dS^T
    float pd[8][4];
#pragma unroll
    for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ql = nb * 8 + 2 * t + (j & 1);
        const int q = q0 + ql;
        const int key = k0 + warp * 16 + g + 8 * (j >> 1);
        const bool keep_pk = q < s && key < s &&
                             !(kMask && ((p.causal && key > q) ||
                                         (p.win_shift > 0 &&
                                          sRp->reg[q] != sRp->reg[key])));
        float P = keep_pk ? exp2f(st[nb][j] * c2 +
                                  (kMask && p.rpb != nullptr ? rpb_bias(p, sRp, q, key) : 0.f) -
                                  sL[ql])
                          : 0.f;
        float keep = 1.f;
        if (thr != 0u) {
          const int kk = key - k0;  // 0..63 within this CTA's key block
          const uint32_t bits = sM[ql * 4 + ((kk & 7) >> 1)];
          keep = (bits >> (((kk >> 3) << 1) | (kk & 1))) & 1u ? inv_keep : 0.f;
        }
        pd[nb][j] = P * keep;
        st[nb][j] = P * (dpt[nb][j] * keep - sD[ql]);  // dS^T
        if (kMask && p.rpb_dpart != nullptr && q < s && key < s)  // dL/d(bias) per (q, k)
          sRB[q * kBlk + key] = st[nb][j];  // (s <= 64: one query and one key block)
      }
    }
    // dV += Pd^T dO ; dK += dS^T Q   (k-dim = queries)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4], sa[4];
      pa[0] = pack2(pd[2 * kk][0], pd[2 * kk][1]);
      pa[1] = pack2(pd[2 * kk][2], pd[2 * kk][3]);
      pa[2] = pack2(pd[2 * kk + 1][0], pd[2 * kk + 1][1]);
      pa[3] = pack2(pd[2 * kk + 1][2], pd[2 * kk + 1][3]);
      sa[0] = pack2(st[2 * kk][0], st[2 * kk][1]);
      sa[1] = pack2(st[2 * kk][2], st[2 * kk][3]);
      sa[2] = pack2(st[2 * kk + 1][0], st[2 * kk + 1][1]);
      sa[3] = pack2(st[2 * kk + 1][2], st[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < HD / 16; ++np) {
        uint32_t of[4], qf[4];
        const int row = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int col = np * 16 + (lane >> 4) * 8;
        ldsm_x4_t(of, sdO + row * LDS + col);
        ldsm_x4_t(qf, sQ + row * LDS + col);
        mma_bf16(dv[2 * np], pa, of[0], of[1]);
        mma_bf16(dv[2 * np + 1], pa, of[2], of[3]);
        mma_bf16(dk[2 * np], sa, qf[0], qf[1]);
        mma_bf16(dk[2 * np + 1], sa, qf[2], qf[3]);
      }
      // stash dS^T (bf16) for the dQ product
      const int kr = warp * 16 + g;
      *reinterpret_cast<uint32_t*>(sdS + kr * LDP + kk * 16 + 2 * t) = sa[0];
      *reinterpret_cast<uint32_t*>(sdS + (kr + 8) * LDP + kk * 16 + 2 * t) = sa[1];
      *reinterpret_cast<uint32_t*>(sdS + kr * LDP + kk * 16 + 8 + 2 * t) = sa[2];
      *reinterpret_cast<uint32_t*>(sdS + (kr + 8) * LDP + kk * 16 + 8 + 2 * t) = sa[3];
    }
    __syncthreads();
    // dQ[q][d] += sum_k dS[q][k] K[k][d] : warp w owns queries [16w, 16w+16)
    {
      float dq[HD / 8][4];
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {  // 16 keys per step
        uint32_t a[4];
        // A[q][k] = dS^T[k][q]: transpose-load from the [k][q] stash
        ldsm_x4_t(a, sdS + (kk * 16 + (lane & 7) + (lane >> 4) * 8) * LDP + warp * 16 +
                         ((lane >> 3) & 1) * 8);
#pragma unroll
        for (int np = 0; np < HD / 16; ++np) {
          uint32_t bf[4];
          ldsm_x4_t(bf, sK + (kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + np * 16 +
                            (lane >> 4) * 8);
          mma_bf16(dq[2 * np], a, bf[0], bf[1]);
          mma_bf16(dq[2 * np + 1], a, bf[2], bf[3]);
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int q = q0 + warp * 16 + g + 8 * r;
        if (q >= s) continue;
        float* dst = dqacc + static_cast<int64_t>(q) * HD;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
          atomicAdd(dst + i * 8 + 2 * t, dq[i][2 * r]);
          atomicAdd(dst + i * 8 + 2 * t + 1, dq[i][2 * r + 1]);
        }
      }
    }
    __syncthreads();
  }
  if (kMask && p.rpb_dpart != nullptr) {
    // this (window, head)'s bias-table gradient: entry e sums the dS of every (q, k) at relative
    // offset e, in a fixed order; the batch sum follows in rpb_grad
    const int w = p.rpb_side, n = 2 * w - 1;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int dy = e / n - (w - 1), dx = e % n - (w - 1);
      float acc = 0.f;
      for (int q = 0; q < s; ++q) {
        const int yk = sRp->y[q] - dy, xk = sRp->x[q] - dx;
        if (yk >= 0 && yk < w && xk >= 0 && xk < w) acc += sRB[q * kBlk + yk * w + xk];
      }
      static_cast<float*>(p.rpb_dpart)[static_cast<int64_t>(bh) * n * n + e] = acc;
    }
  }
  // write dK, dV (scaled) into dqkv
  auto* dqkv = static_cast<__nv_bfloat16*>(p.dqkv);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = k0 + warp * 16 + g + 8 * r;
    if (key >= s) continue;
    __nv_bfloat16* row = dqkv + (static_cast<int64_t>(b) * s + key) * ld + h * HD;
    __nv_bfloat16* dK = row + static_cast<int64_t>(H) * HD;
    __nv_bfloat16* dV = dK + static_cast<int64_t>(H) * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      *reinterpret_cast<uint32_t*>(dK + i * 8 + 2 * t) =
          pack2(dk[i][2 * r] * p.scale, dk[i][2 * r + 1] * p.scale);
      *reinterpret_cast<uint32_t*>(dV + i * 8 + 2 * t) = pack2(dv[i][2 * r], dv[i][2 * r + 1]);
    }
  }
}

// dq (fp32, [bh][s][HD]) * scale -> bf16 Q slot of dqkv
template <int HD>
__global__ void attn_bwd_dq_kernel(const gx_attention_args p) {
  pdl_enter();
  const int s = p.seq, H = p.heads;
  const int64_t total = static_cast<int64_t>(p.batch) * H * s * (HD / 2);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int d2 = static_cast<int>(i % (HD / 2));
    const int64_t row = i / (HD / 2);  // bh * s + q
    const int q = static_cast<int>(row % s);
    const int bh = static_cast<int>(row / s);
    const int b = bh / H, h = bh % H;
    const float2 v = reinterpret_cast<const float2*>(p.dq_accum)[i];
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.dqkv) +
                         (static_cast<int64_t>(b) * s + q) * p.ld_qkv + h * HD + 2 * d2;
    *reinterpret_cast<uint32_t*>(dst) = pack2(v.x * p.scale, v.y * p.scale);
  }
}

// ------------------------------------------------------------------------------ host

template <int HD>
static int attention_fwd_impl(const gx_attention_args& a, cudaStream_t st) {
  constexpr int LDS = HD + 8;
  const int smem = 5 * kBlk * LDS * 2;
  const int smem_m = smem + static_cast<int>(sizeof(RpbSmem));
  if (a.rpb != nullptr && (a.rpb_side < 1 || a.rpb_side > 8 || a.seq != a.rpb_side * a.rpb_side))
    return set_error(kErrConfig, "attention: relative-position bias needs square windows of <= 8x8");
  if (a.win_shift > 0 && a.seq > kBlk)
    return set_error(kErrConfig, "attention: shifted windows of <= 64 tokens");
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(attn_fwd_kernel<HD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_fwd_kernel<HD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_m);
    set = true;
  }
  dim3 grid((a.seq + kBlk - 1) / kBlk, a.batch * a.heads);
  if (a.causal || a.win_shift > 0 || a.rpb != nullptr)
    launch_k(attn_fwd_kernel<HD, true>, grid, dim3(kThreads), smem_m, st, a);
  else
    launch_k(attn_fwd_kernel<HD, false>, grid, dim3(kThreads), smem, st, a);
  return check_launch("attn_fwd_kernel");
}

template <int HD>
static int attention_bwd_impl(const gx_attention_args& a, cudaStream_t st) {
  constexpr int LDS = HD + 8;
  const int smem = 4 * kBlk * LDS * 2 + kBlk * (kBlk + 8) * 2 + 2 * kBlk * 4 + kBlk * 4 * 2;
  // + the relative-position-bias dS tile and staged table
  const int smem_m = smem + kBlk * kBlk * 4 + static_cast<int>(sizeof(RpbSmem));
  if (a.rpb_dpart != nullptr && a.seq > kBlk)
    return set_error(kErrConfig, "attention: relative-position bias needs windows of <= 64 tokens");
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(attn_bwd_kernel<HD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(attn_bwd_kernel<HD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_m);
    set = true;
  }
  const int rows = a.batch * a.heads * a.seq;
  launch_k(attn_bwd_prep_kernel<HD>, dim3((rows + 7) / 8), dim3(256), 0, st, a);
  if (int rc = check_launch("attn_bwd_prep_kernel")) return rc;
  dim3 grid((a.seq + kBlk - 1) / kBlk, a.batch * a.heads);
  if (a.causal || a.win_shift > 0 || a.rpb != nullptr)
    launch_k(attn_bwd_kernel<HD, true>, grid, dim3(kThreads), smem_m, st, a);
  else
    launch_k(attn_bwd_kernel<HD, false>, grid, dim3(kThreads), smem, st, a);
  if (int rc = check_launch("attn_bwd_kernel")) return rc;
  const int64_t work = static_cast<int64_t>(rows) * (HD / 2);
  int blocks = static_cast<int>((work + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_k(attn_bwd_dq_kernel<HD>, dim3(blocks), dim3(256), 0, st, a);
  return check_launch("attn_bwd_dq_kernel");
}

// grad[h][e] (+)= sum_b sum_{(q,k): offset e} dpart[b*heads + h][q][k]: one block per (h, e),
// threads stride over b, fixed-order tree reduction (deterministic).
// grad[h][e] (+)= sum_b dpart[b*heads + h][e]: one block per (h, e); threads stride over b
// and a shared-memory tree adds their sums in a fixed order (deterministic).
__global__ void rpb_grad_kernel(const float* __restrict__ dpart, int batch, int heads, int ne,
                                float* __restrict__ grad, bool accumulate) {
  pdl_enter();
  const int i = blockIdx.x;  // h * ne + e
  float acc = 0.f;
  for (int b = threadIdx.x; b < batch; b += blockDim.x)
    acc += dpart[static_cast<int64_t>(b) * heads * ne + i];
  __shared__ float red[128];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) grad[i] = (accumulate ? grad[i] : 0.f) + red[0];
}

int rpb_grad(const float* dpart, int batch, int heads, int side, float* grad, bool accumulate,
             cudaStream_t st) {
  if (batch <= 0) return kOk;
  const int n = 2 * side - 1;
  launch_k(rpb_grad_kernel, dim3(heads * n * n), dim3(128), 0, st, dpart, batch, heads, n * n,
           grad, accumulate);
  return check_launch("rpb_grad_kernel");
}

// T5 relative-bias gradient: grad[h][b] (+)= sum over sequence tiles t, key blocks and
// relative positions d with map[d] == b of dpart[(t*heads + h)*nkt + kt][d]; one block per
// (h, b), threads stride over the terms and a shared-memory tree adds them in fixed order.
__global__ void relb_grad_kernel(const float* __restrict__ dpart, int tiles, int heads, int nkt,
                                 int nd, const int8_t* __restrict__ map, int buckets,
                                 float* __restrict__ grad, bool accumulate) {
  pdl_enter();
  const int hh = blockIdx.x / buckets, b = blockIdx.x % buckets;
  float acc = 0.f;
  const int64_t terms = static_cast<int64_t>(tiles) * nkt * nd;
  for (int64_t i = threadIdx.x; i < terms; i += blockDim.x) {
    const int d = static_cast<int>(i % nd);
    if (map[d] != b) continue;
    const int64_t tk = i / nd;  // t * nkt + kt
    const int64_t t = tk / nkt, kt = tk % nkt;
    acc += dpart[((t * heads + hh) * nkt + kt) * nd + d];
  }
  __shared__ float red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) grad[blockIdx.x] = (accumulate ? grad[blockIdx.x] : 0.f) + red[0];
}

int relb_grad(const float* dpart, int tiles, int heads, int seq, const void* map, int buckets,
              float* grad, bool accumulate, cudaStream_t st) {
  if (tiles <= 0) return kOk;
  const int nkt = (seq + 127) / 128;
  launch_k(relb_grad_kernel, dim3(heads * buckets), dim3(256), 0, st, dpart, tiles, heads, nkt,
           2 * seq - 1, static_cast<const int8_t*>(map), buckets, grad, accumulate);
  return check_launch("relb_grad_kernel");
}

int attention_fwd(const gx_attention_args& a, cudaStream_t st) {
  if (a.seq <= 0 || a.batch <= 0 || a.heads <= 0) return set_error(kErrConfig, "attention: empty");
  if (attention_tc_supported(a)) return attention_fwd_tc(a, st);
  if (a.relb != nullptr)
    return set_error(kErrConfig, "attention: the T5 relative bias needs the tcgen05 path");
  switch (a.head_dim) {
    case 32: return attention_fwd_impl<32>(a, st);
    case 64: return attention_fwd_impl<64>(a, st);
    case 80: return attention_fwd_impl<80>(a, st);
    case 128: return attention_fwd_impl<128>(a, st);
    default: return set_error(kErrConfig, "attention: head_dim must be 32, 64, 80 or 128");
  }
}

int attention_bwd(const gx_attention_args& a, cudaStream_t st) {
  if (a.seq <= 0 || a.batch <= 0 || a.heads <= 0) return set_error(kErrConfig, "attention: empty");
  if (attention_tc_supported(a) && (a.ld_ctx % 8) == 0) return attention_bwd_tc(a, st);
  if (a.relb != nullptr)
    return set_error(kErrConfig, "attention: the T5 relative bias needs the tcgen05 path");
  switch (a.head_dim) {
    case 32: return attention_bwd_impl<32>(a, st);
    case 64: return attention_bwd_impl<64>(a, st);
    case 80: return attention_bwd_impl<80>(a, st);
    case 128: return attention_bwd_impl<128>(a, st);
    default: return set_error(kErrConfig, "attention: head_dim must be 32, 64, 80 or 128");
  }
}

}  // namespace gx
