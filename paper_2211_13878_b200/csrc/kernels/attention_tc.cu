// attention_tc.cu — attention forward on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   ctx = dropout(softmax(Q K^T * scale)) V        one CTA per (sample*head, 128-query tile)
//
// Same contract as attention.cu's forward (ctx, lse in log2 units, 16-bit keep masks with the
// identical Philox call -> key mapping), restated for sm_100a with the whole key range of a
// head resident on chip (seq <= 512, head_dim 64):
//   1. one thread issues TMA loads of Q [128 x 64], K and V [NK x 64] (NK = seq rounded up to
//      64; rows past the sample read as finite neighbours or zero fill and are masked) into
//      128B-swizzled smem, then tcgen05.mma S = Q K^T into TMEM columns [0, NK) (fp32);
//   2. sixteen warps (four per TMEM lane quarter, 64-key blocks round-robin) read S back with
//      tcgen05.ld: pass 1 row max, pass 2 exp2, row sum, Philox dropout, bf16 P written into
//      smem in the UMMA K-major SWIZZLE_128B layout (over the dead Q/K tiles), keep bits to
//      global for the backward;
//   3. tcgen05.mma O = P V (V as an MN-major operand, straight from its TMA tile) into TMEM
//      columns [0, 64), and the epilogue scales by 1/rowsum and stores bf16 ctx.
// No online rescaling is needed: the full row of scores is in TMEM when the max is taken.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gx_internal.h"
#include "launch.cuh"
#include "philox.cuh"
#include "sm100.cuh"

namespace gx {

namespace {

constexpr int kTcQ = 128;       // queries per CTA (UMMA M)
constexpr int kTcHD = 64;       // head dim (one 128 B swizzle row)
constexpr int kTcMaxKeys = 512; // TMEM columns

struct TcLayout {
  int nk;          // keys rounded up to 64
  int qk_bytes;    // Q + K tiles (P groups overlay them first)
  int v_off;       // V tile
  int p_hi_off;    // P groups that do not fit over Q + K
  int p_lo_groups; // P groups placed at [0, qk_bytes)
  int red_off;     // row max / row sum exchange [2][4][128] floats
  int bar_off;
  int bytes;
};

__host__ __device__ inline TcLayout tc_layout(int seq) {
  TcLayout L{};
  L.nk = (seq + 63) / 64 * 64;
  L.qk_bytes = kTcQ * 128 + L.nk * 128;
  L.v_off = L.qk_bytes;
  const int groups = L.nk / 64;
  L.p_lo_groups = L.qk_bytes / (16 * 1024);
  if (L.p_lo_groups > groups) L.p_lo_groups = groups;
  L.p_hi_off = L.v_off + L.nk * 128;
  const int hi = groups - L.p_lo_groups;
  L.red_off = L.p_hi_off + hi * 16 * 1024;
  L.bar_off = L.red_off + 8 * kTcQ * 4;  // [max | sum][4 column quarters][128 rows]
  L.bytes = L.bar_off + 64;
  return L;
}

__device__ __forceinline__ uint32_t p_group_addr(const TcLayout& L, uint32_t base, int g) {
  return g < L.p_lo_groups ? base + g * 16384 : base + L.p_hi_off + (g - L.p_lo_groups) * 16384;
}

__device__ __forceinline__ unsigned long long gtimer_tc() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// debug stamps: slot i of CTA (blockIdx.y * gridDim.x + blockIdx.x), 32 slots per CTA
#define GX_ATTN_STAMP(p, i)                                                                   \
  do {                                                                                        \
    if ((p).trace != nullptr && threadIdx.x == 0)                                             \
      (p).trace[(blockIdx.y * gridDim.x + blockIdx.x) * 32 + (i)] = gtimer_tc();              \
  } while (0)
__device__ __forceinline__ float ex2_ftz(float x) {  // MUFU.EX2, no denormal fix-up
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void fence_proxy_async_smem_tc() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void st_shared_v4_tc(uint32_t addr, uint32_t a, uint32_t b, uint32_t c,
                                                uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

// 32 lanes x 16 consecutive 32-bit TMEM columns
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
constexpr int kBwdSoftmax = 512;  // 16 softmax warps: four per TMEM lane quarter, 32 queries each
constexpr int kBwdThreads = kBwdSoftmax + 32;  // + one producer / MMA-issue warp (warp 16)
constexpr int kBwdMmaWarp = kBwdSoftmax / 32;
constexpr int kFwdThreads = 512;  // 16 warps: four per TMEM lane quarter

}  // namespace

template <uint32_t kCols>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap map_qkv, const gx_attention_args p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-align by offsetting the shared array itself, so every access below stays in the
  // shared state space (an integer-cast pointer would compile to generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int s = p.seq;
  const TcLayout L = tc_layout(s);
  const uint32_t sbase = smem_u32(smem);
  float* red = reinterpret_cast<float*>(smem + L.red_off);  // [max|sum][quarter][128]
  uint64_t* bar_qk = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* bar_v = bar_qk + 1;
  uint64_t* bar_s = bar_qk + 2;
  uint64_t* bar_o = bar_qk + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_qk + 4);

  const int warp = static_cast<int>(warp_id());
  const int lane = static_cast<int>(lane_id());
  const int H = p.heads;
  const int bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int q0 = blockIdx.x * kTcQ;
  const int nk = L.nk;

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    mbar_init(bar_qk, 1);
    mbar_init(bar_v, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_o, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<kCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  GX_ATTN_STAMP(p, 0);
  pdl_enter();
  GX_ATTN_STAMP(p, 1);

  // ---------------------------------------------------------------- loads + S = Q K^T
  if (warp == 0) {  // warp-uniform: lane 0 issues, the rest wait here
    if (lane == 0) {
      const int row0 = b * s;  // first token row of this sample
      const int slot_q = h, slot_k = H + h, slot_v = 2 * H + h;
      // 64-row boxes (128 B rows, 128B swizzle): Q 2 boxes, K and V nk/64 boxes each
      mbar_expect_tx(bar_qk, (kTcQ + nk) * 128);
      tma_load_3d(smem, &map_qkv, bar_qk, 0, slot_q, row0 + q0);
      tma_load_3d(smem + 64 * 128, &map_qkv, bar_qk, 0, slot_q, row0 + q0 + 64);
      for (int r = 0; r < nk; r += 64)
        tma_load_3d(smem + kTcQ * 128 + r * 128, &map_qkv, bar_qk, 0, slot_k, row0 + r);
      mbar_expect_tx(bar_v, nk * 128);
      for (int r = 0; r < nk; r += 64)
        tma_load_3d(smem + L.v_off + r * 128, &map_qkv, bar_v, 0, slot_v, row0 + r);
      mbar_wait(bar_qk, 0);
      tc_fence_after();
      for (int n0 = 0; n0 < nk; n0 += 256) {
        const int n = nk - n0 < 256 ? nk - n0 : 256;
        const uint32_t idesc = idesc_bf16_f32(kTcQ, n, false, false);
#pragma unroll
        for (int k = 0; k < kTcHD / 16; ++k) {
          const uint64_t ad = sdesc_sw128(sbase + k * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sbase + kTcQ * 128 + n0 * 128 + k * 32, 16, 1024);
          umma_bf16(tmem + n0, ad, bd, idesc, k != 0 ? 1u : 0u);
        }
      }
      umma_commit(bar_s);
    }
    __syncwarp();
  }

  // ---------------------------------------------------------------- softmax over TMEM rows
  // 16 warps: four per TMEM lane quarter; 64-key blocks go round-robin to the four column
  // quarters (a block's two 32-key halves stay with one thread, so its Philox draws are
  // shared), and the quarters exchange row max / row sum through shared memory.
  const int qd = warp & 3, cq = warp >> 2;
  const int r = qd * 32 + lane;  // tile row == TMEM lane
  const int q = q0 + r;
  const int nblk = nk / 64;
  const uint32_t trow = tmem + (static_cast<uint32_t>(qd * 32) << 16);
  const float c2 = p.scale * 1.4426950408889634f;
  mbar_wait(bar_s, 0);
  tc_fence_after();
  GX_ATTN_STAMP(p, 2);

  // keys [0, lim) exist for this row: the sequence, and with a causal mask only k <= q
  const int lim = p.causal ? (q + 1 < s ? q + 1 : s) : s;
  float mx = -INFINITY;
  for (int kb = cq; kb < nblk; kb += 4) {
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const int c0 = kb * 64 + hb * 32;
      uint32_t v[32];
      tmem_ld32(trow + c0, v);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float x = c0 + j < lim ? __uint_as_float(v[j]) * c2 : -INFINITY;
        mx = fmaxf(mx, x);
      }
    }
  }
  red[cq * kTcQ + r] = mx;
  named_sync(1, kFwdThreads);
  GX_ATTN_STAMP(p, 3);
  const float m = fmaxf(fmaxf(red[r], red[kTcQ + r]), fmaxf(red[2 * kTcQ + r], red[3 * kTcQ + r]));

  const uint32_t thr = p.drop_threshold;
  const float inv_keep = p.drop_scale;
  const uint64_t seed = p.seed + (p.seed_offset != nullptr ? *p.seed_offset : 0ull);
  const int nkb = (s + 63) / 64;
  const uint64_t stream =
      (static_cast<uint64_t>(p.sample_offset + b) * p.heads_total + (p.head_offset + h)) * s;
  uint16_t* mask = static_cast<uint16_t*>(p.mask);
  const bool row_ok = q < s;
  float sum = 0.f;
  for (int kb = cq; kb < nblk; kb += 4) {
    uint32_t bits[4] = {0u, 0u, 0u, 0u};
    if (thr != 0u) {
      const uint64_t call0 = ((stream + static_cast<uint64_t>(q)) * nkb + kb) * 4;
#pragma unroll
      for (int t = 0; t < 4; ++t) bits[t] = keep16(seed, p.site, call0 + t, thr);
      if (row_ok && kb < nkb) {
        const uint64_t packed = static_cast<uint64_t>(bits[0]) |
                                (static_cast<uint64_t>(bits[1]) << 16) |
                                (static_cast<uint64_t>(bits[2]) << 32) |
                                (static_cast<uint64_t>(bits[3]) << 48);
        *reinterpret_cast<uint64_t*>(mask + ((static_cast<int64_t>(bh) * s + q) * nkb + kb) * 4) =
            packed;
      }
    }
    const uint32_t g_addr = p_group_addr(L, sbase, kb) + r * 128;
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const int c0 = kb * 64 + hb * 32;
      uint32_t v[32];
      tmem_ld32(trow + c0, v);
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int j2 = 0; j2 < 16; ++j2) {
        float e2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int i = 2 * j2 + u;
          float e = c0 + i < lim ? ex2_ftz(__uint_as_float(v[i]) * c2 - m) : 0.f;
          sum += e;
          if (thr != 0u) {
            // key i of this 32-key half: word t = (i/2)%4, bit 8*hb + 2*(i/8) + i%2
            const uint32_t bit = (bits[(i >> 1) & 3] >> (8 * hb + 2 * (i >> 3) + (i & 1))) & 1u;
            e = bit ? e * inv_keep : 0.f;
          }
          e2[u] = e;
        }
        pk[j2] = pack_bf16(e2[0], e2[1]);
      }
      // bf16 P row segment -> K-major SWIZZLE_128B tile of its 64-key group
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t sw = static_cast<uint32_t>((hb * 4 + i) ^ (r & 7));
        st_shared_v4_tc(g_addr + (sw << 4), pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
  }
  red[4 * kTcQ + cq * kTcQ + r] = sum;
  fence_proxy_async_smem_tc();  // P (generic stores) -> visible to the tensor core
  tc_fence_before();
  named_sync(1, kFwdThreads);
  GX_ATTN_STAMP(p, 4);
  const float l = red[4 * kTcQ + r] + red[5 * kTcQ + r] + red[6 * kTcQ + r] + red[7 * kTcQ + r];

  // ---------------------------------------------------------------- O = P V
  if (warp == 0) {  // warp-uniform: lane 0 issues, the rest wait here
    if (lane == 0) {
      tc_fence_after();
      mbar_wait(bar_v, 0);
      const uint32_t idesc = idesc_bf16_f32(kTcQ, kTcHD, false, true);
      for (int kk = 0; kk < nk / 16; ++kk) {
        const uint64_t ad = sdesc_sw128(p_group_addr(L, sbase, kk >> 2) + (kk & 3) * 32, 16, 1024);
        const uint64_t bd = sdesc_sw128(sbase + L.v_off + kk * 2048, nk * 128, 1024);
        umma_bf16(tmem, ad, bd, idesc, kk != 0 ? 1u : 0u);
      }
      umma_commit(bar_o);
    }
    __syncwarp();
  }
  if (cq == 0 && row_ok) {
    auto* lse = static_cast<float*>(p.lse);
    lse[static_cast<int64_t>(bh) * s + q] = m + log2f(l);
  }
  mbar_wait(bar_o, 0);
  tc_fence_after();
  GX_ATTN_STAMP(p, 5);
  {  // O columns [cq*16, cq*16 + 16) of this row
    uint32_t o[16];
    tmem_ld16(trow + cq * 16, o);
    tmem_ld_wait();
    if (row_ok) {
      const float inv = 1.f / l;
      auto* ctx = static_cast<__nv_bfloat16*>(p.ctx);
      uint4* out = reinterpret_cast<uint4*>(ctx + (static_cast<int64_t>(b) * s + q) * p.ld_ctx +
                                            h * kTcHD + cq * 16);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        out[i] = make_uint4(pack_bf16(__uint_as_float(o[8 * i + 0]) * inv, __uint_as_float(o[8 * i + 1]) * inv),
                            pack_bf16(__uint_as_float(o[8 * i + 2]) * inv, __uint_as_float(o[8 * i + 3]) * inv),
                            pack_bf16(__uint_as_float(o[8 * i + 4]) * inv, __uint_as_float(o[8 * i + 5]) * inv),
                            pack_bf16(__uint_as_float(o[8 * i + 6]) * inv, __uint_as_float(o[8 * i + 7]) * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<kCols>(tmem);
  }
}

// ------------------------------------------------------------------------------ backward
// One CTA per (sample*head, 128-key tile); the queries stream through in 128-row chunks
// (double-buffered TMA).  Per chunk j, with K, V of the tile resident:
//   S^T = K Q_j^T and dPd^T = V dO_j^T                 (tcgen05, TMEM cols [0,128) / [128,256))
//   P = exp2(S*c2 - lse), Pd = drop(P), dP = drop(dPd), dS = P (dP - D)   (thread = key row)
//   dV += Pd^T dO_j, dK += dS^T Q_j                     (TMEM cols [256,320) / [320,384))
//   dQ_j = dS K  (dS^T's smem tile read as an MN-major A operand) -> fp32 partial per key tile
// lse and the keep words of every query are staged in smem once; D = rowsum(dO * O) is
// computed per chunk from the dO / O tiles in smem.  The key tiles of a head form one
// thread-block cluster: after a cluster barrier, CTA t sums the dQ partials of query chunk t
// over the key tiles in key-tile order, so the result is deterministic and the reduction is
// spread over the cluster.
namespace {
struct BwdLayout {
  // Q and dO stream through three 16 KB buffers each (chunk j in buffer j % 3)
  static constexpr int kK = 0, kV = 16384, kQ = 32768, kDO = 81920, kPd = 131072,
                       kDS = 163840, kLse = 196608 /* [512] */, kD = kLse + 2048 /* [2][128] */,
                       kMask = kD + 1024 /* [512 q][2 kb][4] u16 */, kBar = kMask + 8192,
                       kBytes = kBar + 128;
};
}  // namespace

__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap map_qkv,
                       const __grid_constant__ CUtensorMap map_do,
                       const __grid_constant__ CUtensorMap map_o, const gx_attention_args p) {
  using BL = BwdLayout;
  extern __shared__ uint8_t smem_raw[];
  // 1024-align by offsetting the shared array itself, so every access below stays in the
  // shared state space (an integer-cast pointer would compile to generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sb = smem_u32(smem);
  float* sLse = reinterpret_cast<float*>(smem + BL::kLse);
  float* sD = reinterpret_cast<float*>(smem + BL::kD);
  uint16_t* sMask = reinterpret_cast<uint16_t*>(smem + BL::kMask);  // [512 q][2 kb][4]
  uint64_t* bar_kv = reinterpret_cast<uint64_t*>(smem + BL::kBar);
  uint64_t* bar_ld = bar_kv + 1;  // [3]
  uint64_t* bar_s = bar_kv + 4;
  uint64_t* bar_mm = bar_kv + 5;
  uint64_t* bar_pds = bar_kv + 6;  // Pd / dS of a chunk stored (all softmax threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_kv + 7);

  const int warp = static_cast<int>(warp_id());
  const int lane = static_cast<int>(lane_id());
  const int s = p.seq, H = p.heads;
  const int bh = blockIdx.y;
  const int b = bh / H, h = bh % H;
  const int kt = blockIdx.x;  // key tile
  const int nkt = gridDim.x;
  const int nq = (s + kTcQ - 1) / kTcQ;
  const int nkb = (s + 63) / 64;
  const int row0 = b * s;

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    tma_prefetch(&map_do);
    tma_prefetch(&map_o);
    mbar_init(bar_kv, 1);
    mbar_init(&bar_ld[0], 1);
    mbar_init(&bar_ld[1], 1);
    mbar_init(&bar_ld[2], 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_mm, 1);
    mbar_init(bar_pds, kBwdSoftmax);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  GX_ATTN_STAMP(p, 0);
  pdl_enter();
  GX_ATTN_STAMP(p, 1);

  const bool is_mma_warp = warp == kBwdMmaWarp;
  if (!is_mma_warp) {  // lse and keep words of every query of the head (once)
    const float* lse_g = static_cast<const float*>(p.lse) + static_cast<int64_t>(bh) * s;
    const uint16_t* mask_g = static_cast<const uint16_t*>(p.mask);
    for (int q = threadIdx.x; q < s; q += kBwdSoftmax) sLse[q] = lse_g[q];
    for (int i = threadIdx.x; i < 2 * s; i += kBwdSoftmax) {
      const int q = i >> 1, kb = kt * 2 + (i & 1);
      uint64_t w = 0;
      if (p.drop_threshold != 0u && kb < nkb)
        w = *reinterpret_cast<const uint64_t*>(mask_g + ((static_cast<int64_t>(bh) * s + q) * nkb + kb) * 4);
      *reinterpret_cast<uint64_t*>(sMask + i * 4) = w;
    }
  }

  const int qd = warp & 3, cq = (warp >> 2) & 3;  // TMEM lane quarter, 32-column quarter
  const int kr = qd * 32 + lane;      // key row of the tile == TMEM lane (S^T, dV, dK)
  const int key = kt * 128 + kr;
  const uint32_t trow = tmem + (static_cast<uint32_t>(qd * 32) << 16);
  const float c2 = p.scale * 1.4426950408889634f;
  const uint32_t thr = p.drop_threshold;
  const float inv_keep = p.drop_scale;
  const int kbl = kr >> 6, kk = kr & 63;
  const int mt = (kk >> 1) & 3, mbit = 2 * (kk >> 3) + (kk & 1);
  float* part = static_cast<float*>(p.dq_accum);

  if (is_mma_warp) {
    // ------------------------------------------------ producer / MMA issue (one lane)
    // Softmax warps never wait on this warp directly: it consumes bar_pds (Pd / dS stored)
    // and publishes bar_s (next scores) and bar_mm (gradient products), so the issue
    // latency of ~30 MMAs per chunk overlaps the softmax math instead of stalling it.
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16_f32(kTcQ, 128, false, false);
      const uint32_t idesc_kv = idesc_bf16_f32(128, kTcHD, false, true);
      const uint32_t idesc_q = idesc_bf16_f32(kTcQ, kTcHD, true, true);
      auto load_chunk = [&](int j) {  // Q_j, dO_j -> buffer j % 3
        const int bf = j % 3;
        const int r = row0 + j * kTcQ;
        mbar_expect_tx(&bar_ld[bf], 2 * kTcQ * 128);
        for (int x = 0; x < 2; ++x) {
          tma_load_3d(smem + BL::kQ + bf * 16384 + x * 8192, &map_qkv, &bar_ld[bf], 0, h, r + 64 * x);
          tma_load_3d(smem + BL::kDO + bf * 16384 + x * 8192, &map_do, &bar_ld[bf], 0, h, r + 64 * x);
        }
      };
      auto issue_s = [&](int j) {  // S^T = K Q_j^T, dPd^T = V dO_j^T
        const int bf = j % 3;
        mbar_wait(&bar_ld[bf], (j / 3) & 1);
        tc_fence_after();
        const uint32_t q_b = sb + BL::kQ + bf * 16384, do_b = sb + BL::kDO + bf * 16384;
#pragma unroll
        for (int k = 0; k < kTcHD / 16; ++k) {
          umma_bf16(tmem, sdesc_sw128(sb + BL::kK + k * 32, 16, 1024),
                    sdesc_sw128(q_b + k * 32, 16, 1024), idesc_s, k != 0 ? 1u : 0u);
          umma_bf16(tmem + 128, sdesc_sw128(sb + BL::kV + k * 32, 16, 1024),
                    sdesc_sw128(do_b + k * 32, 16, 1024), idesc_s, k != 0 ? 1u : 0u);
        }
        umma_commit(bar_s);
      };
      auto issue_grads = [&](int j) {  // dV += Pd^T dO_j, dK += dS^T Q_j, dQ_j = dS K
        const int bf = j % 3;
        const uint32_t q_b = sb + BL::kQ + bf * 16384, do_b = sb + BL::kDO + bf * 16384;
#pragma unroll
        for (int k = 0; k < kTcQ / 16; ++k) {
          const uint32_t a_kmaj = (k >> 2) * 16384 + (k & 3) * 32;
          const uint32_t acc = (j > 0 || k > 0) ? 1u : 0u;
          umma_bf16(tmem + 256, sdesc_sw128(sb + BL::kPd + a_kmaj, 16, 1024),
                    sdesc_sw128(do_b + k * 2048, 16384, 1024), idesc_kv, acc);
          umma_bf16(tmem + 320, sdesc_sw128(sb + BL::kDS + a_kmaj, 16, 1024),
                    sdesc_sw128(q_b + k * 2048, 16384, 1024), idesc_kv, acc);
          umma_bf16(tmem + 384, sdesc_sw128(sb + BL::kDS + k * 2048, 16384, 1024),
                    sdesc_sw128(sb + BL::kK + k * 2048, 16384, 1024), idesc_q, k > 0 ? 1u : 0u);
        }
        umma_commit(bar_mm);
      };
      mbar_expect_tx(bar_kv, 2 * kTcQ * 128);
      for (int x = 0; x < 2; ++x) {
        tma_load_3d(smem + BL::kK + x * 8192, &map_qkv, bar_kv, 0, H + h, row0 + kt * 128 + 64 * x);
        tma_load_3d(smem + BL::kV + x * 8192, &map_qkv, bar_kv, 0, 2 * H + h, row0 + kt * 128 + 64 * x);
      }
      for (int j = 0; j < nq && j < 3; ++j) load_chunk(j);
      mbar_wait(bar_kv, 0);
      issue_s(0);
      for (int j = 0; j < nq; ++j) {
        mbar_wait(bar_pds, j & 1);  // Pd / dS(j) in smem; S / dPd(j) and dQ(j-1) out of TMEM
        tc_fence_after();
        if (j + 1 < nq) issue_s(j + 1);  // next scores first ...
        if (j >= 1) {  // chunk j-1's gradients (at most one bar_mm phase is ever pending here)
          mbar_wait(bar_mm, (j - 1) & 1);
          if (j + 2 < nq) load_chunk(j + 2);  // ... its Q / dO buffer takes chunk j + 2
        }
        issue_grads(j);                   // ... then this chunk's gradient products
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax warps (0..15)
    // D = rowsum(dO * O) of chunk j's 128 queries -> sD[j & 1] (dO from smem, O from global)
    auto compute_d = [&](int j) {
      const int bf = j % 3;
      mbar_wait(&bar_ld[bf], (j / 3) & 1);
      const int qi = threadIdx.x >> 2, part4 = threadIdx.x & 3;  // 4 threads per query row
      const int q = j * kTcQ + qi;
      const uint8_t* dob = smem + BL::kDO + bf * 16384 + qi * 128;
      float acc = 0.f;
      if (q < s) {
        const uint4* og = reinterpret_cast<const uint4*>(
            static_cast<const __nv_bfloat16*>(p.ctx) + (static_cast<int64_t>(row0) + q) * p.ld_ctx +
            h * kTcHD + part4 * 16);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int cc = part4 * 2 + c;
          const int sw = (cc ^ (qi & 7)) << 4;
          const uint4 a = *reinterpret_cast<const uint4*>(dob + sw);
          const uint4 o = og[c];
          const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
          for (int t = 0; t < 4; ++t)
            acc += bf16_lo(aw[t]) * bf16_lo(ow[t]) + bf16_hi(aw[t]) * bf16_hi(ow[t]);
        }
      }
      acc += __shfl_xor_sync(0xffffffff, acc, 1);
      acc += __shfl_xor_sync(0xffffffff, acc, 2);
      if (part4 == 0) sD[(j & 1) * kTcQ + qi] = acc;
    };
    // dQ_j partial (fp32) out of TMEM (lane = query row of the chunk, 16 columns per warp)
    auto store_dq = [&](int j) {
      uint32_t o[16];
      tmem_ld16(trow + 384 + cq * 16, o);
      tmem_ld_wait();
      const int q = j * kTcQ + kr;
      if (q < s) {
        float4* dst = reinterpret_cast<float4*>(
            part + ((static_cast<int64_t>(kt) * gridDim.y + bh) * s + q) * kTcHD + cq * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dst[i] = make_float4(__uint_as_float(o[4 * i]), __uint_as_float(o[4 * i + 1]),
                               __uint_as_float(o[4 * i + 2]), __uint_as_float(o[4 * i + 3]));
      }
    };
    compute_d(0);
    named_sync(1, kBwdSoftmax);
    GX_ATTN_STAMP(p, 2);
    for (int j = 0; j < nq; ++j) {
      mbar_wait(bar_s, j & 1);
      tc_fence_after();
      GX_ATTN_STAMP(p, 4 + 5 * j);
      const int c0 = cq * 32;
      const int qg0 = j * kTcQ + c0;
      const float* sDj = sD + (j & 1) * kTcQ;
      uint32_t ppd[16], pds[16];
      {
        // no tail / causal masking needed for this 32-query x 128-key block
        const bool full = qg0 + 32 <= s && kt * 128 + 128 <= s && (!p.causal || kt * 128 + 127 <= qg0);
        uint32_t sv[32], dv[32];
        tmem_ld32(trow + c0, sv);
        tmem_ld32(trow + 128 + c0, dv);
        tmem_ld_wait();
#pragma unroll
        for (int i4 = 0; i4 < 8; ++i4) {
          const float4 l4 = *reinterpret_cast<const float4*>(sLse + qg0 + 4 * i4);
          const float4 d4 = *reinterpret_cast<const float4*>(sDj + c0 + 4 * i4);
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dd[4] = {d4.x, d4.y, d4.z, d4.w};
          float pd4[4], ds4[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int i = 4 * i4 + t;
            const int qg = qg0 + i;
            const bool valid = full || ((qg < s) && (key < s) && !(p.causal && key > qg));
            const float pr = valid ? ex2_ftz(__uint_as_float(sv[i]) * c2 - lv[t]) : 0.f;
            float f = 1.f;  // dropout factor: inv_keep or 0
            if (thr != 0u)
              f = valid && ((sMask[(qg * 2 + kbl) * 4 + mt] >> mbit) & 1u) != 0u ? inv_keep : 0.f;
            pd4[t] = pr * f;
            ds4[t] = pr * (__uint_as_float(dv[i]) * f - dd[t]);
          }
          ppd[2 * i4] = pack_bf16(pd4[0], pd4[1]);
          ppd[2 * i4 + 1] = pack_bf16(pd4[2], pd4[3]);
          pds[2 * i4] = pack_bf16(ds4[0], ds4[1]);
          pds[2 * i4 + 1] = pack_bf16(ds4[2], ds4[3]);
        }
      }
      GX_ATTN_STAMP(p, 5 + 5 * j);
      if (j > 0) {  // chunk j-1's gradient MMAs: done reading Pd / dS; its dQ leaves TMEM
        mbar_wait(bar_mm, (j - 1) & 1);
        tc_fence_after();
        store_dq(j - 1);
      }
      GX_ATTN_STAMP(p, 6 + 5 * j);
      {
        const uint32_t rowoff = static_cast<uint32_t>((cq >> 1) * 16384 + kr * 128);
        const int chunk0 = (cq & 1) * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t sw = static_cast<uint32_t>((chunk0 + i) ^ (kr & 7)) << 4;
          st_shared_v4_tc(sb + BL::kPd + rowoff + sw, ppd[4 * i], ppd[4 * i + 1], ppd[4 * i + 2],
                          ppd[4 * i + 3]);
          st_shared_v4_tc(sb + BL::kDS + rowoff + sw, pds[4 * i], pds[4 * i + 1], pds[4 * i + 2],
                          pds[4 * i + 3]);
        }
      }
      fence_proxy_async_smem_tc();
      tc_fence_before();
      mbar_arrive(bar_pds);  // the MMA warp may issue S(j+1) and the gradients of j
      GX_ATTN_STAMP(p, 7 + 5 * j);
      // sD is double-buffered: sD[(j+1) & 1] was last read in chunk j-1, before every softmax
      // warp passed the barrier that ended chunk j-1
      if (j + 1 < nq) compute_d(j + 1);
      named_sync(1, kBwdSoftmax);  // sD(j+1) visible
      GX_ATTN_STAMP(p, 8 + 5 * j);
    }
    mbar_wait(bar_mm, (nq - 1) & 1);
    tc_fence_after();
    store_dq(nq - 1);
    // dK (x scale), dV -> bf16 rows of dqkv
    {
      uint32_t dvv[16], dkv[16];
      tmem_ld16(trow + 256 + cq * 16, dvv);
      tmem_ld16(trow + 320 + cq * 16, dkv);
      tmem_ld_wait();
      if (key < s) {
        auto* dq = static_cast<__nv_bfloat16*>(p.dqkv);
        __nv_bfloat16* rowp = dq + (static_cast<int64_t>(row0) + key) * p.ld_qkv;
        uint4* dvp = reinterpret_cast<uint4*>(rowp + (2 * H + h) * kTcHD + cq * 16);
        uint4* dkp = reinterpret_cast<uint4*>(rowp + (H + h) * kTcHD + cq * 16);
        const float sc = p.scale;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          dvp[i] = make_uint4(pack_bf16(__uint_as_float(dvv[8 * i]), __uint_as_float(dvv[8 * i + 1])),
                              pack_bf16(__uint_as_float(dvv[8 * i + 2]), __uint_as_float(dvv[8 * i + 3])),
                              pack_bf16(__uint_as_float(dvv[8 * i + 4]), __uint_as_float(dvv[8 * i + 5])),
                              pack_bf16(__uint_as_float(dvv[8 * i + 6]), __uint_as_float(dvv[8 * i + 7])));
          dkp[i] = make_uint4(pack_bf16(__uint_as_float(dkv[8 * i]) * sc, __uint_as_float(dkv[8 * i + 1]) * sc),
                              pack_bf16(__uint_as_float(dkv[8 * i + 2]) * sc, __uint_as_float(dkv[8 * i + 3]) * sc),
                              pack_bf16(__uint_as_float(dkv[8 * i + 4]) * sc, __uint_as_float(dkv[8 * i + 5]) * sc),
                              pack_bf16(__uint_as_float(dkv[8 * i + 6]) * sc, __uint_as_float(dkv[8 * i + 7]) * sc));
        }
      }
    }
  }
  tc_fence_before();
  // every key tile's dQ partials are in global memory after the cluster barrier; CTA kt then
  // owns query chunk kt and sums its partials in key-tile order
  GX_ATTN_STAMP(p, 25);
  __threadfence();
  cluster_sync();
  GX_ATTN_STAMP(p, 26);
  {
    auto* dq = static_cast<__nv_bfloat16*>(p.dqkv);
    const float sc = p.scale;
    const int q_lo = kt * kTcQ, q_hi = min(s, q_lo + kTcQ);
#pragma unroll 4
    for (int idx = threadIdx.x; idx < (q_hi - q_lo) * (kTcHD / 8); idx += kBwdThreads) {
      const int q = q_lo + idx / (kTcHD / 8), c8 = idx % (kTcHD / 8);
      float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int t = 0; t < nkt; ++t) {
        const float4* src = reinterpret_cast<const float4*>(
            part + ((static_cast<int64_t>(t) * gridDim.y + bh) * s + q) * kTcHD + c8 * 8);
        const float4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
        a[0] += x0.x; a[1] += x0.y; a[2] += x0.z; a[3] += x0.w;
        a[4] += x1.x; a[5] += x1.y; a[6] += x1.z; a[7] += x1.w;
      }
      *reinterpret_cast<uint4*>(dq + (static_cast<int64_t>(row0) + q) * p.ld_qkv + h * kTcHD + c8 * 8) =
          make_uint4(pack_bf16(a[0] * sc, a[1] * sc), pack_bf16(a[2] * sc, a[3] * sc),
                     pack_bf16(a[4] * sc, a[5] * sc), pack_bf16(a[6] * sc, a[7] * sc));
    }
  }
  GX_ATTN_STAMP(p, 27);
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ------------------------------------------------------------------------------ host

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn_tc() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult qr;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) !=
            cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

bool attention_tc_supported(const gx_attention_args& a) {
  static const bool on = [] {
    const char* e = std::getenv("GX_ATTN_TC");
    return e == nullptr || e[0] != '0';
  }();
  return on && a.head_dim == kTcHD && a.seq >= 1 && a.seq <= kTcMaxKeys && a.win_shift == 0 && a.rpb == nullptr &&
         (a.ld_qkv % 8) == 0 && (reinterpret_cast<uintptr_t>(a.qkv) % 16) == 0 &&
         (a.ld_ctx % 8) == 0;
}

int attention_fwd_tc(const gx_attention_args& a, cudaStream_t st) {
  auto fn = encode_fn_tc();
  if (fn == nullptr) return set_error(kErrCuda, "attention_tc: no cuTensorMapEncodeTiled");
  // qkv viewed as [rows][3*heads slots][64]: one 3-D map serves Q, K and V of every head
  CUtensorMap map;
  const uint64_t rows = static_cast<uint64_t>(a.batch) * a.seq;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(kTcHD), static_cast<cuuint64_t>(3 * a.heads), rows};
  cuuint64_t strides[2] = {kTcHD * 2, static_cast<cuuint64_t>(a.ld_qkv) * 2};
  cuuint32_t box[3] = {kTcHD, 1, 64};
  cuuint32_t estr[3] = {1, 1, 1};
  const int nk = (a.seq + 63) / 64 * 64;
  CUresult rc = fn(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.qkv), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return set_error(kErrCuda, "attention_tc: tensor map encode failed");
  const TcLayout L = tc_layout(a.seq);
  const int smem = L.bytes + 1024;
  dim3 grid((a.seq + kTcQ - 1) / kTcQ, a.batch * a.heads);
#define GX_ATTN_TC(C)                                                                      \
  {                                                                                        \
    static bool set = false;                                                               \
    if (!set) {                                                                            \
      cudaFuncSetAttribute(attn_fwd_tc_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           227 * 1024);                                                    \
      set = true;                                                                          \
    }                                                                                      \
    launch_k(attn_fwd_tc_kernel<C>, grid, dim3(kFwdThreads), smem, st, map, a);             \
  }
  if (nk <= 64) GX_ATTN_TC(64)
  else if (nk <= 128) GX_ATTN_TC(128)
  else if (nk <= 256) GX_ATTN_TC(256)
  else GX_ATTN_TC(512)
#undef GX_ATTN_TC
  return check_launch("attn_fwd_tc_kernel");
}


static bool make_head_map(CUtensorMap* map, const void* base, int slots, uint64_t rows, int64_t ld) {
  auto fn = encode_fn_tc();
  if (fn == nullptr) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(kTcHD), static_cast<cuuint64_t>(slots), rows};
  cuuint64_t strides[2] = {kTcHD * 2, static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[3] = {kTcHD, 1, 64};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int attention_bwd_tc(const gx_attention_args& a, cudaStream_t st) {
  const uint64_t rows = static_cast<uint64_t>(a.batch) * a.seq;
  CUtensorMap mq, md, mo;
  if (!make_head_map(&mq, a.qkv, 3 * a.heads, rows, a.ld_qkv) ||
      !make_head_map(&md, a.dctx, a.heads, rows, a.ld_ctx) ||
      !make_head_map(&mo, a.ctx, a.heads, rows, a.ld_ctx))
    return set_error(kErrCuda, "attention_tc: tensor map encode failed");
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(attn_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         BwdLayout::kBytes + 1024);
    set = true;
  }
  dim3 grid((a.seq + 127) / 128, a.batch * a.heads);
  // the key tiles of one head form a cluster (dQ reduction after a cluster barrier)
  launch_k_cluster(attn_bwd_tc_kernel, grid, dim3(kBwdThreads), BwdLayout::kBytes + 1024, st,
                   static_cast<unsigned>(grid.x), mq, md, mo, a);
  return check_launch("attn_bwd_tc_kernel");
}

}  // namespace gx
