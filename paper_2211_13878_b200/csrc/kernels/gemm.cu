// gemm.cu — persistent warp-specialised tcgen05 GEMM for the Transformer layer's linear ops.
//
//   C[M,N] = A[M,K] * B[N,K]^T   (bf16 in, fp32 accumulate in TMEM, fused epilogue)
//
// Operands may be K-major or MN-major (the UMMA descriptor transposes on the fly), so one
// kernel family covers forward (X*W^T: K/K), data-gradient (dY*W: K/MN) and weight-gradient
// (dY^T*X: MN/MN) without materialised transposes.
//
// Roles (256 threads, one CTA per SM):
//   warp 0      TMA producer: A/B tiles -> smem ring (SWIZZLE_128B), mbarrier complete_tx
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma (M=128, N=BN, K=16)
//   warp 2      TMEM allocator (2 x BN fp32 columns: accumulator double buffer)
//   warps 4..7  epilogue: tcgen05.ld -> bias / GeLU / dropout+residual -> global
// The accumulator double buffer lets tile i's epilogue overlap tile i+1's main loop.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cstdio>

#include "gx_internal.h"
#include "launch.cuh"
#include "philox.cuh"
#include "sm100.cuh"

namespace gx {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B = one swizzle span
constexpr int kEpiWarps = 8;  // warps 4..11: two per TMEM lane quarter, each half the columns
constexpr int kThreads = 128 + 32 * kEpiWarps;
// 384 threads x 128 registers = 48K of the SM's 64K: a GEMM CTA leaves room for a co-resident
// block of another stream (the optimizer / column passes beside the data-gradient chain)
#ifndef GX_GEMM_MAXREGS
#define GX_GEMM_MAXREGS 128
#endif
constexpr int kGemmMaxRegs = GX_GEMM_MAXREGS;
// epilogue staging per warp: out 4 KB + two 2 KB bf16 operand buffers + 256 B bias, plus the
// operand-prefetch mbarriers (see kStagingBytes below)
constexpr int kStagingBytesDecl = kEpiWarps * (4096 + 2048 + 2048 + 256) + kEpiWarps * 2 * 8;
constexpr int kSmemBudget = 227 * 1024 - kStagingBytesDecl - 2048;  // left for the A/B ring

template <int BN>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (kSmemBudget / kStageBytes) > 8 ? 8 : (kSmemBudget / kStageBytes);
  static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int kSmemBytes =
      kStages * kStageBytes + kStagingBytesDecl + 1024 /*align*/ + 256 /*barriers*/;
};

// Exact-erf GeLU, x * Phi(x).  erf(z) for z = |x|/sqrt(2) uses the Abramowitz-Stegun 7.1.26
// rational form (|error| < 1.5e-7, far below the bf16 rounding of the stored result): one
// reciprocal, one exp2 and six FMAs instead of erff's branchy polynomial -- the GeLU epilogue
// runs on the CUDA cores of a tensor-bound GEMM, so its instruction count is on the critical
// path.  The same exp(-x^2/2) feeds the derivative Phi(x) + x phi(x).
struct GeluTerms {
  float phi_cdf;  // Phi(x) = 0.5 (1 + erf(x / sqrt 2))
  float e;        // exp(-x^2 / 2)
};
__device__ __forceinline__ GeluTerms gelu_terms(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  float t;  // MUFU.RCP (~1 ulp): __frcp_rn's IEEE slow path cost more than the whole rest
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.f)));
  const float poly =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f),
                       -0.284496736f), 0.254829592f);
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-z * z * 1.4426950408889634f));
  const float erf_abs = 1.f - poly * e;
  return GeluTerms{0.5f * (1.f + copysignf(erf_abs, x)), e};
}
__device__ __forceinline__ float gelu_erf(float x) { return x * gelu_terms(x).phi_cdf; }
// d/dx [x * Phi(x)] = Phi(x) + x * phi(x)
__device__ __forceinline__ float gelu_erf_grad(float x) {
  const GeluTerms g = gelu_terms(x);
  return g.phi_cdf + x * 0.3989422804014327f * g.e;
}

// GeLU value and derivative of two bf16-rounded pre-activations (the gelu == 2 epilogue):
// gelu_terms() on packed pairs.  The rational erf runs on the negated reciprocal
// tn = -t = 1 / (-(1 + a z)), so -poly(t) comes out of one Horner chain with alternating
// coefficient signs (negation is exact: every intermediate is the scalar chain's, negated).
__device__ __forceinline__ void gelu2_pair(float x0, float x1, float& v0, float& v1, float& d0,
                                           float& d1) {
  const f2 x = f2_pack(x0, x1);
  const f2 z = f2_mul(f2_pack(fabsf(x0), fabsf(x1)), f2_splat(0.70710678118654752f));
  const f2 den = f2_fma(f2_splat(-0.3275911f), z, f2_splat(-1.f));
  float tn0, tn1;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(tn0) : "f"(f2_lo(den)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(tn1) : "f"(f2_hi(den)));
  const f2 tn = f2_pack(tn0, tn1);
  f2 hp = f2_fma(tn, f2_splat(1.061405429f), f2_splat(1.453152027f));
  hp = f2_fma(tn, hp, f2_splat(1.421413741f));
  hp = f2_fma(tn, hp, f2_splat(0.284496736f));
  hp = f2_fma(tn, hp, f2_splat(0.254829592f));
  const f2 npoly = f2_mul(tn, hp);  // -poly
  const f2 arg = f2_mul(f2_mul(z, z), f2_splat(-1.4426950408889634f));  // (-z z) c, exactly
  float e0, e1;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(f2_lo(arg)));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(f2_hi(arg)));
  const f2 e = f2_pack(e0, e1);
  const f2 erf_abs = f2_fma(npoly, e, f2_splat(1.f));  // 1 - poly e
  const f2 s = f2_pack(copysignf(f2_lo(erf_abs), x0), copysignf(f2_hi(erf_abs), x1));
  const f2 phi = f2_fma(s, f2_splat(0.5f), f2_splat(0.5f));  // 0.5 (1 + s): *0.5 is exact
  const f2 v = f2_mul(x, phi);
  const f2 d = f2_fma(f2_mul(x, f2_splat(0.3989422804014327f)), e, phi);
  v0 = f2_lo(v);
  v1 = f2_hi(v);
  d0 = f2_lo(d);
  d1 = f2_hi(d);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Epilogue math for 32 consecutive accumulator columns of one row (the lane's): v <- final
// values, pre <- bf16-rounded pre-activation (GeLU forward).  bias_w / in_w hold the 32 bf16
// bias values of these columns and the 32 bf16 of the row's epilogue operand (gelu_bwd's
// pre-activation or the residual), both already staged on chip; out-of-range rows / columns
// read as zero and the TMA store clips them.
__device__ __forceinline__ void epilogue_math(const GemmEpilogue& ep, int64_t row, int n0,
                                              const uint32_t (&acc)[32],
                                              const uint32_t (&bias_w)[16],
                                              const uint32_t (&in_w)[16], float (&v)[32],
                                              float (&pre)[32]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(acc[j]) * ep.alpha;
  if (ep.bias != nullptr) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      v[2 * t] += bf16_lo(bias_w[t]);
      v[2 * t + 1] += bf16_hi(bias_w[t]);
    }
  }
  if (ep.gelu_bwd == 2) {  // aux already holds gelu'(pre) (written by a gelu == 2 forward)
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      v[2 * t] *= bf16_lo(in_w[t]);
      v[2 * t + 1] *= bf16_hi(in_w[t]);
    }
  } else if (ep.gelu_bwd) {  // dgrad epilogue of the MLP up-projection: v <- v * gelu'(pre)
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      v[2 * t] *= gelu_erf_grad(bf16_lo(in_w[t]));
      v[2 * t + 1] *= gelu_erf_grad(bf16_hi(in_w[t]));
    }
  }
  if (ep.gelu == 2) {
    // forward that also hands the backward its derivative: aux <- gelu'(pre), computed from
    // the same erf / exp as the value, so the backward epilogue is a plain multiply
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const float x0 = __bfloat162float(__float2bfloat16_rn(v[2 * t]));
      const float x1 = __bfloat162float(__float2bfloat16_rn(v[2 * t + 1]));
      gelu2_pair(x0, x1, v[2 * t], v[2 * t + 1], pre[2 * t], pre[2 * t + 1]);
    }
  } else if (ep.gelu) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      // GeLU is applied to the bf16-rounded pre-activation so forward and backward agree.
      pre[j] = __bfloat162float(__float2bfloat16_rn(v[j]));
      v[j] = gelu_erf(pre[j]);
    }
  }
  if (ep.residual != nullptr) {
    // out = residual + dropout(v), dropout element index = (row_offset+row)*drop_ld + col
    const uint64_t grow = static_cast<uint64_t>(ep.row_offset + row);
    if (ep.drop_threshold != 0u) {
      const uint64_t seed = ep.seed + (ep.seed_offset != nullptr ? *ep.seed_offset : 0ull);
      // e0 is a multiple of 16 (drop_ld and column offsets are; checked on host): the 32
      // columns are exactly two Philox calls
      const uint64_t e0 = grow * static_cast<uint64_t>(ep.drop_ld) +
                          static_cast<uint64_t>(ep.col_offset + n0);
      const uint32_t k0 = keep16(seed, ep.site, e0 >> 4, ep.drop_threshold);
      const uint32_t k1 = keep16(seed, ep.site, (e0 >> 4) + 1, ep.drop_threshold);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool keep = ((j < 16 ? k0 >> j : k1 >> (j - 16)) & 1u) != 0u;
        v[j] = keep ? v[j] * ep.drop_scale : 0.f;
      }
    }
    // dropout output rounded to bf16 before the add, matching the unfused path
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      v[2 * t] = __bfloat162float(__float2bfloat16_rn(v[2 * t])) + bf16_lo(in_w[t]);
      v[2 * t + 1] = __bfloat162float(__float2bfloat16_rn(v[2 * t + 1])) + bf16_hi(in_w[t]);
    }
  }
}

// ---------------------------------------------------------------- TMA-store epilogue
// Each epilogue warp owns 32 rows; a 32 x 32 block of results is written to a swizzled
// staging buffer (64 B rows + SWIZZLE_64B for bf16, 128 B rows + SWIZZLE_128B for fp32:
// conflict-free st.shared.v4 with one row per lane) and leaves through one TMA bulk
// store (or bulk reduce-add for fp32 accumulation).
// The epilogue's bf16 operand (gelu_bwd pre-activation or residual) arrives the same way in
// reverse: TMA loads of 32 x 32 blocks into two per-warp buffers, the first issued before
// the warp waits for the accumulator (so it overlaps the main loop) and each next one while
// the current block is processed.  The bias slice of a tile is staged in shared memory
// before the accumulator wait as well, so no global load latency is left in the epilogue.
constexpr int kStageOutBytes = 4096;  // 32 x 32 fp32
constexpr int kStageAuxBytes = 2048;  // 32 x 32 bf16 (gelu pre-activation out / operand in #0)
constexpr int kStageInBytes = 2048;   // 32 x 32 bf16 (operand in #1)
constexpr int kStageWarpBytes = kStageOutBytes + kStageAuxBytes + kStageInBytes;
constexpr int kBiasWarpBytes = 256;   // up to 4 chunks x 32 bf16
constexpr int kStagingBytes = kEpiWarps * (kStageWarpBytes + kBiasWarpBytes) + kEpiWarps * 2 * 8;
static_assert(kStagingBytes == kStagingBytesDecl, "epilogue staging layout");

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                             uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ void ld_shared_v4(uint32_t addr, uint32_t& a, uint32_t& b, uint32_t& c,
                                             uint32_t& d) {
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "r"(addr)
               : "memory");
}
__device__ __forceinline__ void stage_bf16_row(uint32_t base, uint32_t r, const float (&v)[32]) {
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c) {
    const uint32_t addr = base + r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
    st_shared_v4(addr, pack_bf16(v[c * 8 + 0], v[c * 8 + 1]), pack_bf16(v[c * 8 + 2], v[c * 8 + 3]),
                 pack_bf16(v[c * 8 + 4], v[c * 8 + 5]), pack_bf16(v[c * 8 + 6], v[c * 8 + 7]));
  }
}
// the 32 bf16 of row r from a SWIZZLE_64B 32 x 32 block (inverse of stage_bf16_row)
__device__ __forceinline__ void load_bf16_row(uint32_t base, uint32_t r, uint32_t (&w)[16]) {
#pragma unroll
  for (uint32_t c = 0; c < 4; ++c)
    ld_shared_v4(base + r * 64 + ((c ^ ((r >> 1) & 3)) << 4), w[4 * c], w[4 * c + 1],
                 w[4 * c + 2], w[4 * c + 3]);
}
__device__ __forceinline__ void stage_f32_row(uint32_t base, uint32_t r, const float (&v)[32]) {
#pragma unroll
  for (uint32_t c = 0; c < 8; ++c) {
    const uint32_t addr = base + r * 128 + ((c ^ (r & 7)) << 4);
    st_shared_v4(addr, __float_as_uint(v[c * 4 + 0]), __float_as_uint(v[c * 4 + 1]),
                 __float_as_uint(v[c * 4 + 2]), __float_as_uint(v[c * 4 + 3]));
  }
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int32_t c0,
                                             int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
// Output stores go through a 3-D map {cols, M, slices}: the slice coordinate is the split-K
// index, so a 32-row block that straddles row M is clipped at its own slice's end instead of
// spilling into the next slice's first rows.
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int32_t c0,
                                             int32_t c1, int32_t c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, uint32_t src, int32_t c0,
                                                  int32_t c1, int32_t c2) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_u32(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {  // all but the most recent group read
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Per-warp epilogue state: staging buffers, operand-prefetch barriers and their use count.
struct EpiWarp {
  uint32_t out_buf, aux_buf, bias_buf;
  uint32_t bar0;  // operand-prefetch barriers bar0, bar0 + 8
  uint32_t blk;   // operand blocks consumed so far (buffer = blk & 1, phase = (blk >> 1) & 1)
  uint32_t sblk;  // output blocks stored so far (staging buffer = sblk & 1)
  // operand buffer b: buffer 0 is the aux staging (never live together with the gelu
  // pre-activation output), buffer 1 follows it
  __device__ __forceinline__ uint32_t in_buf(uint32_t b) const { return aux_buf + b * kStageAuxBytes; }
  __device__ __forceinline__ uint32_t in_bar(uint32_t b) const { return bar0 + b * 8; }
};

__device__ __forceinline__ void epi_prefetch(const EpiWarp& w, const CUtensorMap* map_in,
                                             uint32_t blk, int32_t col, int32_t row) {
  if (lane_id() == 0) {
    const uint32_t b = blk & 1;
    fence_proxy_async_smem();  // this buffer's previous (generic) reads are complete
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(w.in_bar(b)),
                 "r"(kStageInBytes)
                 : "memory");
    tma_load_2d_u32(w.in_buf(b), map_in, w.in_bar(b), col, row);
  }
}

// Stage this warp's bias columns [n0 + c_lo*32, n0 + c_hi*32) of the tile in shared memory.
__device__ __forceinline__ void epi_stage_bias(const GemmEpilogue& ep, const EpiWarp& w, int n0,
                                               int N, int c_lo, int c_hi) {
  if (ep.bias == nullptr) return;
  const __nv_bfloat16* bias = static_cast<const __nv_bfloat16*>(ep.bias);
  const int lane = static_cast<int>(lane_id());
  const int ncols = (c_hi - c_lo) * 32;
  for (int c = lane * 4; c < ncols; c += 128) {
    uint32_t w0 = 0, w1 = 0;
    const int col = n0 + c_lo * 32 + c;
    if (col + 4 <= N) {
      const uint2 v = *reinterpret_cast<const uint2*>(bias + col);
      w0 = v.x;
      w1 = v.y;
    } else {
      __nv_bfloat16 t[4];
      for (int k = 0; k < 4; ++k) t[k] = col + k < N ? bias[col + k] : __float2bfloat16(0.f);
      w0 = *reinterpret_cast<uint32_t*>(&t[0]);
      w1 = *reinterpret_cast<uint32_t*>(&t[2]);
    }
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(w.bias_buf + c * 2), "r"(w0), "r"(w1)
                 : "memory");
  }
  __syncwarp();
}

// One 32 x 32 output block: math, staging, TMA store.  Executed by a whole epilogue warp.
__device__ __forceinline__ void epilogue_block(const GemmEpilogue& ep, const CUtensorMap* map_out,
                                               const CUtensorMap* map_aux, EpiWarp& w,
                                               bool has_in, int cb, int64_t m_base,
                                               int32_t store_z, int n0, int M, int N,
                                               const uint32_t (&acc)[32]) {
  const uint32_t lane = lane_id();
  const int64_t row = m_base + lane;
  uint32_t bias_w[16], in_w[16];
  if (ep.bias != nullptr) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      ld_shared_v4(w.bias_buf + cb * 64 + c * 16, bias_w[4 * c], bias_w[4 * c + 1],
                   bias_w[4 * c + 2], bias_w[4 * c + 3]);
  }
  if (has_in) {
    const uint32_t b = w.blk & 1;
    mbar_wait_addr(w.in_bar(b), (w.blk >> 1) & 1);
    load_bf16_row(w.in_buf(b), lane, in_w);
    ++w.blk;
  }
  float v[32], pre[32];
  const bool dstamp = ep.trace != nullptr && lane == 0 && (threadIdx.x >> 5) == 4 && w.sblk == 0;
  if (dstamp) ep.trace[blockIdx.x * 16 + 12] = clock64();
  epilogue_math(ep, row, n0, acc, bias_w, in_w, v, pre);
  if (dstamp) ep.trace[blockIdx.x * 16 + 13] = clock64();
  // Double-buffered staging, so block i+1's math overlaps block i's store: bf16 outputs use
  // the two halves of the 4 KB out buffer; fp32 outputs (weight gradients: no operand, no
  // aux) use the out buffer and the 4 KB operand/aux area; the GeLU pre-activation output
  // alternates over the operand/aux area (gelu has no operand).
  // (an fp32 output next to an operand or the GeLU output falls back to one buffer)
  const uint32_t k = w.sblk & 1;
  ++w.sblk;
  const bool f32 = ep.out_kind != kOutBF16;
  const bool dbl = !f32 || (!ep.gelu && !has_in);
  const uint32_t obuf = !f32 ? w.out_buf + k * 2048 : (dbl && k ? w.aux_buf : w.out_buf);
  const uint32_t abuf = w.aux_buf + k * kStageAuxBytes;
  if (lane == 0) {  // the store that last used these buffers has read them
    if (dbl) {
      bulk_wait_read1();
    } else {
      bulk_wait_read0();
    }
  }
  __syncwarp();
  if (!f32) {
    stage_bf16_row(obuf, lane, v);
  } else {
    stage_f32_row(obuf, lane, v);
  }
  if (ep.gelu) stage_bf16_row(abuf, lane, pre);
  fence_proxy_async_smem();
  __syncwarp();
  if (dstamp) ep.trace[blockIdx.x * 16 + 14] = clock64();
  if (lane == 0) {
    if (ep.out_kind == kOutF32Accumulate) {
      tma_reduce_add_3d(map_out, obuf, n0, static_cast<int32_t>(m_base), store_z);
    } else {
      tma_store_3d(map_out, obuf, n0, static_cast<int32_t>(m_base), store_z);
    }
    if (ep.gelu) tma_store_2d(map_aux, abuf, n0, static_cast<int32_t>(m_base));
    bulk_commit();
  }
  if (dstamp) ep.trace[blockIdx.x * 16 + 15] = clock64();
}


// All BN/32 chunks of one accumulator tile for one epilogue warp.  (A ping-pong variant
// that keeps the next chunk's TMEM load in flight measured slower: the extra 32 live
// registers cost more than the hidden LDTM latency.)
// `ew` (0..kEpiWarps-1) selects the column half this warp owns.
template <int BN>
__device__ __forceinline__ void epilogue_chunks(int ew, int* c_lo, int* c_hi) {
  constexpr int NC = BN / 32;
  constexpr int kHalves = kEpiWarps / 4;
  *c_lo = (ew / 4) * NC / kHalves;
  *c_hi = (ew / 4 + 1) * NC / kHalves;
}
template <int BN>
__device__ __forceinline__ void epilogue_tile(const GemmEpilogue& ep, const CUtensorMap* map_out,
                                              const CUtensorMap* map_aux, EpiWarp& w, int ew,
                                              bool has_in, uint32_t taddr, int64_t m_base,
                                              int32_t store_z, int n0, int M, int N) {
  int c_lo, c_hi;
  epilogue_chunks<BN>(ew, &c_lo, &c_hi);
#pragma unroll 1
  for (int c = c_lo; c < c_hi; ++c) {
    // next block of the operand streams in while this one is processed
    if (has_in && c + 1 < c_hi)
      epi_prefetch(w, map_aux, w.blk + 1, n0 + (c + 1) * 32, static_cast<int32_t>(m_base));
    uint32_t r[32];
    const bool stamp = ep.trace != nullptr && ew == 0 && lane_id() == 0 && c - c_lo < 2;
    if (stamp) ep.trace[blockIdx.x * 16 + 8 + 2 * (c - c_lo)] = clock64();
    tmem_ld32(taddr + c * 32, r);
    tmem_ld_wait();
    if (stamp) ep.trace[blockIdx.x * 16 + 9 + 2 * (c - c_lo)] = clock64();
    if (m_base < M && n0 + c * 32 < N) {
      epilogue_block(ep, map_out, map_aux, w, has_in, c - c_lo, m_base, store_z, n0 + c * 32, M,
                     N, r);
    } else if (has_in) {
      // keep the operand pipeline in step: consume (wait for) the block even if unused
      mbar_wait_addr(w.in_bar(w.blk & 1), (w.blk >> 1) & 1);
      ++w.blk;
    }
  }
}

// Before the accumulator wait of a tile: stage bias, start the first operand block.
template <int BN>
__device__ __forceinline__ void epilogue_tile_prologue(const GemmEpilogue& ep,
                                                       const CUtensorMap* map_aux, EpiWarp& w,
                                                       int ew, bool has_in, int64_t m_base,
                                                       int n0, int N) {
  int c_lo, c_hi;
  epilogue_chunks<BN>(ew, &c_lo, &c_hi);
  if (has_in) epi_prefetch(w, map_aux, w.blk, n0 + c_lo * 32, static_cast<int32_t>(m_base));
  epi_stage_bias(ep, w, n0, N, c_lo, c_hi);
}

__device__ __forceinline__ EpiWarp epi_warp_init(uint8_t* staging, int ew) {
  EpiWarp w;
  const uint32_t base = smem_u32(staging);
  w.out_buf = base + ew * kStageWarpBytes;
  w.aux_buf = w.out_buf + kStageOutBytes;
  w.bias_buf = base + kEpiWarps * kStageWarpBytes + ew * kBiasWarpBytes;
  w.bar0 = base + kEpiWarps * (kStageWarpBytes + kBiasWarpBytes) + ew * 16;
  w.blk = 0;
  w.sblk = 0;
  return w;
}

template <int BN, bool kAMN, bool kBMN>
__global__ void __maxnreg__(kGemmMaxRegs)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_out,
                        const __grid_constant__ CUtensorMap map_aux, int M, int N, int K,
                        int splits, const GemmEpilogue ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* staging = smem + S * Cfg::kStageBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + kStagingBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = static_cast<int>(warp_id());
  const int num_m = (M + kBM - 1) / kBM;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_units = num_tiles * splits;  // split-K: unit = (split, tile)
  const int kb_total = (K + kBK - 1) / kBK;
  const int kb_per = (kb_total + splits - 1) / splits;

  if (warp == 0 && elect_one()) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 32 * kEpiWarps);
    }
    for (int i = 0; i < 2 * kEpiWarps; ++i)  // epilogue operand-prefetch barriers
      mbar_init(reinterpret_cast<uint64_t*>(staging + kEpiWarps * (kStageWarpBytes + kBiasWarpBytes)) + i, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();  // everything above overlapped the previous kernel's tail

  if (warp == 0) {
    if (elect_one()) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
        const int tile = unit % num_tiles;
        const int kb0 = (unit / num_tiles) * kb_per;
        const int num_kb = min(kb_per, kb_total - kb0);
        const int m0 = (tile % num_m) * kBM;
        const int n0 = (tile / num_m) * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          uint8_t* a_dst = sA + stage * Cfg::kABytes;
          uint8_t* b_dst = sB + stage * Cfg::kBBytes;
          const int k0 = (kb0 + kb) * kBK;
          if constexpr (!kAMN) {
            tma_load_2d(a_dst, &map_a, &full_bar[stage], k0, m0);
          } else {
#pragma unroll
            for (int c = 0; c < kBM / 64; ++c)
              tma_load_2d(a_dst + c * kBK * 128, &map_a, &full_bar[stage], m0 + c * 64, k0);
          }
          if constexpr (!kBMN) {
            tma_load_2d(b_dst, &map_b, &full_bar[stage], k0, n0);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_2d(b_dst + c * kBK * 128, &map_b, &full_bar[stage], n0 + c * 64, k0);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(kBM, BN, kAMN, kBMN);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x, ++local) {
      const int num_kb = min(kb_per, kb_total - (unit / num_tiles) * kb_per);
      const int buf = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tempty_bar[buf], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t a_base = smem_u32(sA + stage * Cfg::kABytes);
          const uint32_t b_base = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t adesc = kAMN ? sdesc_sw128(a_base + k * 2048, kBK * 128, 1024)
                                        : sdesc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bdesc = kBMN ? sdesc_sw128(b_base + k * 2048, kBK * 128, 1024)
                                        : sdesc_sw128(b_base + k * 32, 16, 1024);
            umma_bf16(d_tmem, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);
          if (kb == num_kb - 1) umma_commit(&tfull_bar[buf]);
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    EpiWarp ew = epi_warp_init(staging, warp - 4);
    const bool has_in = ep.gelu_bwd || ep.residual != nullptr;
    int local = 0;
    for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x, ++local) {
      const int tile = unit % num_tiles;
      const int buf = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile % num_m) * kBM;
      const int n0 = (tile / num_m) * BN;
      const int64_t m_base = m0 + q * 32;
      epilogue_tile_prologue<BN>(ep, &map_aux, ew, warp - 4, has_in, m_base, n0, N);
      mbar_wait(&tfull_bar[buf], acc_phase);
      tc_fence_after();
      // split-K slices: split s stores into slice s of the [splits][M][N] output
      const int32_t store_z = ep.out_kind == kOutF32Split ? unit / num_tiles : 0;
      epilogue_tile<BN>(ep, &map_out, &map_aux, ew, warp - 4, has_in,
                        tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * BN, m_base,
                        store_z, n0, M, N);
      tc_fence_before();
      mbar_arrive(&tempty_bar[buf]);
    }
    // only the shared-memory reads of the outstanding TMA stores must finish before the CTA
    // releases its shared memory; their global writes complete with the grid
    if (lane_id() == 0) bulk_wait_read0();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ CTA-pair variant
// cta_group::2: a cluster of 2 CTAs on one TPC computes a 256 x BN tile.  Each CTA stages
// its own 128 rows of A and HALF of the BN columns of B (so each SM receives 2x fewer B
// bytes per MAC than the 1-CTA kernel), the leader's elected thread issues
// tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' smem, and each CTA's TMEM holds the
// accumulator rows of its own half.  TMA completions of both CTAs land on the leader's
// full barrier; the leader's MMA commits multicast to both CTAs' empty / tmem-full
// barriers; epilogue warps of both CTAs release the accumulator on the leader's barrier.
template <int BN>
struct PairCfg {
  static constexpr int kABytes = 128 * kBK * 2;        // this CTA's 128 rows of A
  static constexpr int kBBytes = (BN / 2) * kBK * 2;   // this CTA's half of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = kSmemBudget / kStageBytes > 8 ? 8 : kSmemBudget / kStageBytes;
  // two accumulator buffers, rounded up to the power-of-two allocation granule
  static constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;
  static constexpr int kSmemBytes = kStages * kStageBytes + kStagingBytesDecl + 1024 + 256;
};

template <int BN, bool kAMN, bool kBMN>
__global__ void __cluster_dims__(2, 1, 1) __maxnreg__(kGemmMaxRegs)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                     const __grid_constant__ CUtensorMap map_b,
                     const __grid_constant__ CUtensorMap map_out,
                     const __grid_constant__ CUtensorMap map_aux, int M, int N, int K,
                     int splits, const GemmEpilogue ep) {
  using Cfg = PairCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* staging = smem + S * Cfg::kStageBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + kStagingBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = static_cast<int>(warp_id());
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int num_pairs = gridDim.x >> 1;
  const int num_pm = (M + 255) / 256;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_pm * num_n;
  const int num_units = num_tiles * splits;
  const int kb_total = (K + kBK - 1) / kBK;
  const int kb_per = (kb_total + splits - 1) / splits;

  if (ep.trace != nullptr && threadIdx.x == 0) ep.trace[blockIdx.x * 16 + 0] = gtimer();
  if (warp == 0 && elect_one()) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);   // leader: its arrive.expect_tx (+ both CTAs' tx bytes)
      mbar_init(&empty_bar[s], 1);  // the leader's multicast MMA commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);  // the leader's multicast MMA commit
      mbar_init(&tempty_bar[b], 2 * kEpiWarps);  // epilogue warps x 2 CTAs (leader copy)
    }
    for (int i = 0; i < 2 * kEpiWarps; ++i)  // epilogue operand-prefetch barriers
      mbar_init(reinterpret_cast<uint64_t*>(staging + kEpiWarps * (kStageWarpBytes + kBiasWarpBytes)) + i, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_enter();  // everything above overlapped the previous kernel's tail
  if (ep.trace != nullptr && threadIdx.x == 0) ep.trace[blockIdx.x * 16 + 1] = gtimer();

  if (warp == 0) {
    if (elect_one()) {
      // -------------------------------------------------------- TMA producer (both CTAs)
      const uint32_t leader_full0 = mapa_shared(smem_u32(&full_bar[0]), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = pair; unit < num_units; unit += num_pairs) {
        const int tile = unit % num_tiles;
        const int kb0 = (unit / num_tiles) * kb_per;
        const int num_kb = min(kb_per, kb_total - kb0);
        const int m0 = (tile % num_pm) * 256 + static_cast<int>(rank) * 128;
        const int nb0 = (tile / num_pm) * BN + static_cast<int>(rank) * (BN / 2);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full_bar[stage], 2 * Cfg::kStageBytes);
          const uint32_t fb = leader_full0 + stage * 8;
          uint8_t* a_dst = sA + stage * Cfg::kABytes;
          uint8_t* b_dst = sB + stage * Cfg::kBBytes;
          const int k0 = (kb0 + kb) * kBK;
          if constexpr (!kAMN) {
            tma_load_2d_pair(a_dst, &map_a, fb, k0, m0);
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c)
              tma_load_2d_pair(a_dst + c * kBK * 128, &map_a, fb, m0 + c * 64, k0);
          }
          if constexpr (!kBMN) {
            tma_load_2d_pair(b_dst, &map_b, fb, k0, nb0);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 128; ++c)
              tma_load_2d_pair(b_dst + c * kBK * 128, &map_b, fb, nb0 + c * 64, k0);
          }
          if (ep.trace != nullptr && unit == pair && kb == 0) ep.trace[blockIdx.x * 16 + 2] = gtimer();
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------------------ MMA issuer (leader)
      constexpr uint32_t idesc = idesc_bf16_f32(256, BN, kAMN, kBMN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int unit = pair; unit < num_units; unit += num_pairs, ++local) {
        const int num_kb = min(kb_per, kb_total - (unit / num_tiles) * kb_per);
        const int buf = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait_cluster(&tempty_bar[buf], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (ep.trace != nullptr && local == 0 && kb == 0 && lane_id() == 0)
            ep.trace[blockIdx.x * 16 + 3] = gtimer();
          if (elect_one()) {
            const uint32_t a_base = smem_u32(sA + stage * Cfg::kABytes);
            const uint32_t b_base = smem_u32(sB + stage * Cfg::kBBytes);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint64_t adesc = kAMN ? sdesc_sw128(a_base + k * 2048, kBK * 128, 1024)
                                          : sdesc_sw128(a_base + k * 32, 16, 1024);
              const uint64_t bdesc = kBMN ? sdesc_sw128(b_base + k * 2048, kBK * 128, 1024)
                                          : sdesc_sw128(b_base + k * 32, 16, 1024);
              umma_bf16_pair(d_tmem, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
            }
            umma_commit_pair(&empty_bar[stage], 0x3);
            if (kb == num_kb - 1) umma_commit_pair(&tfull_bar[buf], 0x3);
            if (ep.trace != nullptr && local == 0 && kb == num_kb - 1)
              ep.trace[blockIdx.x * 16 + 4] = gtimer();
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    const uint32_t leader_tempty0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    EpiWarp ew = epi_warp_init(staging, warp - 4);
    const bool has_in = ep.gelu_bwd || ep.residual != nullptr;
    int local = 0;
    for (int unit = pair; unit < num_units; unit += num_pairs, ++local) {
      const int tile = unit % num_tiles;
      const int buf = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile % num_pm) * 256 + static_cast<int>(rank) * 128;
      const int n0 = (tile / num_pm) * BN;
      const int64_t m_base = m0 + q * 32;
      epilogue_tile_prologue<BN>(ep, &map_aux, ew, warp - 4, has_in, m_base, n0, N);
      mbar_wait(&tfull_bar[buf], acc_phase);
      tc_fence_after();
      if (ep.trace != nullptr && local == 0 && warp == 4 && lane_id() == 0)
        ep.trace[blockIdx.x * 16 + 5] = gtimer();
      // split-K slices: split s stores into slice s of the [splits][M][N] output
      const int32_t store_z = ep.out_kind == kOutF32Split ? unit / num_tiles : 0;
      epilogue_tile<BN>(ep, &map_out, &map_aux, ew, warp - 4, has_in,
                        tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * BN, m_base,
                        store_z, n0, M, N);
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive_remote_relaxed(leader_tempty0 + buf * 8);
    }
    if (ep.trace != nullptr && warp == 4 && lane_id() == 0) ep.trace[blockIdx.x * 16 + 6] = gtimer();
    // only the shared-memory reads of the outstanding TMA stores must finish before the CTA
    // releases its shared memory; their global writes complete with the grid
    if (lane_id() == 0) bulk_wait_read0();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (ep.trace != nullptr && threadIdx.x == 0) ep.trace[blockIdx.x * 16 + 7] = gtimer();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<Cfg::kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------------------ host side

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      return nullptr;
    }
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Epilogue maps: 32 x 32 boxes over the [M][ld] output; bf16 uses 64 B swizzle, fp32 128 B
// (matching the staging layout in epilogue_block).  The output map is 3-D {cols, M, slices}
// (slices = the split-K count for kOutF32Split, else 1); the operand / aux map is 2-D.
static bool make_out_map(CUtensorMap* map, const void* ptr, uint64_t cols, uint64_t rows,
                         uint64_t ld, bool f32, uint64_t slices = 0) {
  auto fn = encode_fn();
  if (fn == nullptr || ptr == nullptr) return false;
  const uint64_t eb = f32 ? 4 : 2;
  cuuint64_t dims[3] = {cols, rows, slices};
  cuuint64_t strides[2] = {ld * eb, rows * ld * eb};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                  slices > 0 ? 3 : 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static bool make_epi_maps(const GemmEpilogue& ep, int M, int N, int splits, CUtensorMap* mo,
                          CUtensorMap* mx) {
  const bool f32 = ep.out_kind != kOutBF16;
  const uint64_t slices = ep.out_kind == kOutF32Split ? static_cast<uint64_t>(splits) : 1;
  if (!make_out_map(mo, ep.out, N, M, ep.ldo, f32, slices)) return false;
  // map_aux: the GeLU pre-activation (written by gelu, read by gelu_bwd) or the residual read
  // by the epilogue's operand prefetch (never both in one GEMM)
  if (ep.gelu || ep.gelu_bwd) return make_out_map(mx, ep.aux, N, M, ep.ld_aux, false);
  if (ep.residual != nullptr) return make_out_map(mx, ep.residual, N, M, ep.ld_res, false);
  *mx = *mo;
  return true;
}

// 2-D bf16 map over a row-major [outer][inner] view with row stride `ld` elements,
// box {64 inner, box_outer}, 128 B swizzle, zero fill out of bounds.
static bool make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer,
                     uint64_t ld, uint32_t box_outer) {
  auto fn = encode_fn();
  if (fn == nullptr) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool kAMN, bool kBMN>
static int launch_gemm(const GemmOperand& a, const GemmOperand& b, int M, int N, int K,
                       const GemmEpilogue& ep, cudaStream_t stream, int splits) {
  using Cfg = GemmCfg<BN>;
  CUtensorMap ma, mb;
  // A: K-major view [M][K] (inner K); MN-major view [K][M] (inner M)
  bool ok = kAMN ? make_map(&ma, a.ptr, M, K, a.ld, kBK) : make_map(&ma, a.ptr, K, M, a.ld, kBM);
  ok = ok && (kBMN ? make_map(&mb, b.ptr, N, K, b.ld, kBK) : make_map(&mb, b.ptr, K, N, b.ld, BN));
  CUtensorMap mo, mx;
  ok = ok && make_epi_maps(ep, M, N, splits, &mo, &mx);
  if (!ok) return set_error(kErrCuda, "gemm: cuTensorMapEncodeTiled failed");
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tcgen05_kernel<BN, kAMN, kBMN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    attr_set = true;
  }
  const int units = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN) * splits;
  const int grid = units < num_sms() ? units : num_sms();
  launch_k(gemm_tcgen05_kernel<BN, kAMN, kBMN>, dim3(grid), dim3(kThreads), Cfg::kSmemBytes,
           stream, ma, mb, mo, mx, M, N, K, splits, ep);
  return check_launch("gemm_tcgen05_kernel");
}

template <int BN, bool kAMN, bool kBMN>
static int launch_gemm_pair(const GemmOperand& a, const GemmOperand& b, int M, int N, int K,
                            const GemmEpilogue& ep, cudaStream_t stream, int splits) {
  using Cfg = PairCfg<BN>;
  CUtensorMap ma, mb;
  // each CTA loads 128 rows of A and BN/2 rows (K-major) / columns (MN-major) of B
  bool ok = kAMN ? make_map(&ma, a.ptr, M, K, a.ld, kBK) : make_map(&ma, a.ptr, K, M, a.ld, 128);
  ok = ok && (kBMN ? make_map(&mb, b.ptr, N, K, b.ld, kBK)
                   : make_map(&mb, b.ptr, K, N, b.ld, BN / 2));
  CUtensorMap mo, mx;
  ok = ok && make_epi_maps(ep, M, N, splits, &mo, &mx);
  if (!ok) return set_error(kErrCuda, "gemm: cuTensorMapEncodeTiled failed");
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_pair_kernel<BN, kAMN, kBMN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    attr_set = true;
  }
  const int units = ((M + 255) / 256) * ((N + BN - 1) / BN) * splits;
  const int pairs = units < num_sms() / 2 ? units : num_sms() / 2;
  launch_k(gemm_pair_kernel<BN, kAMN, kBMN>, dim3(2 * pairs), dim3(kThreads), Cfg::kSmemBytes,
           stream, ma, mb, mo, mx, M, N, K, splits, ep);
  return check_launch("gemm_pair_kernel");
}

// Picks the N tile that minimises the number of waves (ties -> larger tile).
static int pick_bn(int M, int N);
// Tile choice: CTA-pair (negative) when M >= 256, else the 1-CTA kernel.  N tile 160 (K-major
// B only: each CTA stages 80 B rows) fills one wave of pairs where 256 would leave SMs idle
// and 128 would spill into a second wave (e.g. M = 512, N = 5120: 64 pairs vs 40 / 80).
static int pick_tile(int M, int N, bool b_mn) {
  if (M < 256) return pick_bn(M, N);
  const int pairs = num_sms() / 2;
  int best = -256;
  double best_cost = 1e30;
  for (int bn : {256, 160, 128}) {
    if (bn == 256 && N <= 128) continue;
    if (bn == 160 && (b_mn || N <= 128)) continue;
    const int tiles = ((M + 255) / 256) * ((N + bn - 1) / bn);
    const int waves = (tiles + pairs - 1) / pairs;
    const double cost = waves * (bn + 48.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = -bn;
    }
  }
  // One CTA per 128 x 64 tile when that still fits one wave: at M = 512, N = 1280 (the
  // out-projection forward and data-gradient) 80 CTAs beat 20 CTA pairs of 256 x 128
  // (measured 9.6 vs 11.3 us and 8.3 vs 8.8 us, scripts/tile_sweep.py).
  static const bool tile64 = [] {
    const char* e = std::getenv("GX_TILE64");
    return e == nullptr || e[0] != '0';
  }();
  const int tiles64 = ((M + 127) / 128) * ((N + 63) / 64);
  if (tile64 && tiles64 <= num_sms() && 64 + 48.0 < best_cost - 1e-9) best = 64;
  return best;
}

static int pick_bn(int M, int N) {
  const int sms = num_sms();
  const int cands[3] = {256, 128, 64};
  int best = 128;
  double best_cost = 1e30;
  for (int bn : cands) {
    if (bn > 64 && N <= bn / 2) continue;
    const int tiles = ((M + kBM - 1) / kBM) * ((N + bn - 1) / bn);
    const int waves = (tiles + sms - 1) / sms;
    // cost ~ waves * per-tile time (proportional to bn) + fixed per-tile overhead
    const double cost = waves * (bn + 48.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

// Split-K plan for a reduce-add GEMM: the CTA-pair 256-wide tile when M allows, and as many
// K splits as fit one wave of pairs while keeping >= 4 k-blocks per split.  Returns the
// split count and sets *tile (the force_bn argument of gemm_bf16).
int splitk_plan(int M, int N, int K, int* tile, bool b_mn) {
  // At most 4 slices: every slice is an M x N fp32 partial written here and read back by the
  // consuming row pass, so beyond 4 the partials' traffic costs more inside the step than the
  // extra CTAs gain (BERT-Huge-32, M = 512: 4 -> 8.94 ms / step, 7 -> 9.12, 3 -> 9.00; a
  // kernel timed alone prefers more slices)
  constexpr int kMaxSplits = 4;
  const int kb = (K + kBK - 1) / kBK;
  if (M >= 256) {
    // N tile: the one-wave plan whose CTAs each stream the fewest operand rows (128 of A +
    // bn / 2 of B per k-block, over the split's k-blocks) -- at M = 512 the main loops are
    // bound by each SM's ~120 GB/s of L2 ingest, not by its tensor rate.  160 (K-major B
    // only) beats 256 for the MLP down-projection forward (N = 1280, K = 5120: 64 pairs of
    // 208 rows x 20 k-blocks vs 40 pairs of 256 x 20; 13.4 -> 10.9 us, step -1.2 %); ties
    // keep the wider tile.  (Charging the fp32 partial's bytes too picks 128 x 3 slices for
    // the data-gradient GEMMs: each 12-14 % faster alone, but the step 2 % slower -- 120
    // CTAs on the critical path leave fewer SMs to the weight-gradient / AdamW streams.)
    int best_sp = 1, best_bn = N > 128 ? 256 : 128;
    double best_cost = 1e30;
    for (int bn : {256, 160, 128}) {
      if ((bn == 256 && N <= 128) || (bn == 160 && (b_mn || N <= 128))) continue;
      const int tiles = ((M + 255) / 256) * ((N + bn - 1) / bn);
      int sp = std::min((num_sms() / 2) / tiles, kb / 4);
      sp = std::max(1, std::min(sp, kMaxSplits));
      const double cta_bytes = (128.0 + bn / 2) * kBK * 2 * ((kb + sp - 1) / sp);
      const double cost = cta_bytes * ((tiles * sp + num_sms() / 2 - 1) / (num_sms() / 2));
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        best_bn = bn;
        best_sp = sp;
      }
    }
    *tile = -best_bn;
    return best_sp;
  }
  *tile = 128;
  const int tiles = ((M + kBM - 1) / kBM) * ((N + 127) / 128);
  int sp = num_sms() / tiles;
  sp = std::min(sp, kb / 4);
  return std::max(1, std::min(sp, kMaxSplits));
}

int gemm_bf16(const GemmOperand& a, const GemmOperand& b, int M, int N, int K,
              const GemmEpilogue& ep, cudaStream_t stream, int force_bn, int splits) {
  if (splits < 1) splits = 1;
  {  // every split must own >= 1 k-block (an empty split would never signal its epilogue)
    const int kb_total = (K + kBK - 1) / kBK;
    const int kb_per = (kb_total + splits - 1) / splits;
    splits = (kb_total + kb_per - 1) / kb_per;
  }
  if (splits > 1 && ((ep.out_kind != kOutF32Accumulate && ep.out_kind != kOutF32Split) ||
                     ep.bias != nullptr || ep.gelu ||
                     ep.gelu_bwd || ep.residual != nullptr || ep.alpha != 1.f))
    return set_error(kErrConfig, "gemm: split-K needs a plain fp32 accumulate / split epilogue");
  if (M <= 0 || N <= 0 || K <= 0) return set_error(kErrConfig, "gemm: empty problem");
  if ((ep.gelu ? 1 : 0) + (ep.gelu_bwd ? 1 : 0) + (ep.residual != nullptr ? 1 : 0) > 1)
    return set_error(kErrConfig, "gemm: gelu, gelu_bwd and residual epilogues are exclusive");
  // TMA: row strides must be 16-byte multiples; the epilogue's vector stores need ldo too.
  if ((a.ld % 8) != 0 || (b.ld % 8) != 0 || (ep.ldo % 8) != 0 || (ep.gelu && ep.ld_aux % 8 != 0))
    return set_error(kErrConfig, "gemm: lda, ldb, ldo and ld_aux must be multiples of 8 elements");
  if (ep.drop_threshold != 0u && ((ep.drop_ld % 16) != 0 || (ep.col_offset % 16) != 0))
    return set_error(kErrConfig, "gemm: dropout row length / column offset must be multiples of 16");
  // force_bn: >0 selects the 1-CTA kernel with that N tile, <0 the CTA-pair kernel with
  // N tile -force_bn, 0 = automatic (pair kernel whenever M spans at least one 256-row tile).
  int bn = force_bn;
  if (bn == 0) bn = pick_tile(M, N, b.mn_major);
  if (bn == -160 && b.mn_major) return set_error(kErrConfig, "gemm: N tile 160 needs K-major B");
#define GX_GEMM_DISPATCH(BN_, LAUNCH)                                                        \
  if (bn == BN_) {                                                                           \
    if (!a.mn_major && !b.mn_major) return LAUNCH<BN_ < 0 ? -BN_ : BN_, false, false>(a, b, M, N, K, ep, stream, splits); \
    if (!a.mn_major && b.mn_major) return LAUNCH<BN_ < 0 ? -BN_ : BN_, false, true>(a, b, M, N, K, ep, stream, splits);   \
    if (a.mn_major && b.mn_major) return LAUNCH<BN_ < 0 ? -BN_ : BN_, true, true>(a, b, M, N, K, ep, stream, splits);     \
    return LAUNCH<BN_ < 0 ? -BN_ : BN_, true, false>(a, b, M, N, K, ep, stream, splits);                 \
  }
  GX_GEMM_DISPATCH(256, launch_gemm)
  GX_GEMM_DISPATCH(128, launch_gemm)
  GX_GEMM_DISPATCH(64, launch_gemm)
  GX_GEMM_DISPATCH(-256, launch_gemm_pair)
  GX_GEMM_DISPATCH(-128, launch_gemm_pair)
  if (bn == -160) {
    if (!a.mn_major) return launch_gemm_pair<160, false, false>(a, b, M, N, K, ep, stream, splits);
    return launch_gemm_pair<160, true, false>(a, b, M, N, K, ep, stream, splits);
  }
#undef GX_GEMM_DISPATCH
  return set_error(kErrConfig, "gemm: unsupported N tile");
}

}  // namespace gx
