// attention_tc.cu — attention forward and backward on the 5th-generation tensor cores
// (tcgen05 + TMEM + TMA) for every attention shape of the BASELINE configs:
//
//   ctx = dropout(softmax(Q K^T * scale + bias, masked)) V
//
//   * head_dim 32 / 64 / 80 (any multiple of 16 up to 80): each head row is staged as one or
//     two 64-column SWIZZLE_128B panels by 2-D TMA boxes at column slot*hd + panel*64; the MMAs
//     use exactly hd/16 K-steps (hd as the K dimension) or N = hd (hd as the N dimension), so
//     the neighbouring head's columns a second panel drags in are never read;
//   * sequences of up to 512 keys, tail-masked (ViT-Huge: 257 tokens);
//   * short sequences (Swin's 49-token windows) packed wpt = 128 / seq per tile, with a
//     block-diagonal mask -- one CTA attends several windows instead of idling 60% of its rows;
//   * causal masking (decoder self-attention), Swin's shifted-window region mask (SW-MSA) and
//     its learned relative-position bias (forward bias, backward table gradient).
// Contract (identical to attention.cu's mma.sync kernels, which remain only for shapes outside
// the list above): ctx bf16, lse in log2 units [batch*heads][seq], 16-bit keep masks with the
// Philox call -> key mapping of oracle/layer_oracle.py::_attn_mask.
//
// Forward CTA = (tile of wpt sequences x head, 128-query block), 16 warps (four per TMEM lane
// quarter):
//   1. one thread issues the TMA loads of Q [128 x hd] and K, V [nk x hd] (nk = the tile's
//      keys rounded up to 64) and tcgen05.mma S = Q K^T into TMEM columns [0, nk) (fp32);
//   2. the 16 warps read S back with tcgen05.ld (64-key blocks round-robin over four column
//      quarters): pass 1 row max, pass 2 exp2, row sum, Philox dropout, bf16 P written into smem
//      in the UMMA K-major SWIZZLE_128B layout over the dead Q / K tiles, keep bits to global;
//   3. tcgen05.mma O = P V (V as an MN-major operand straight from its TMA tile) into TMEM
//      columns [0, hd); the epilogue scales by 1 / rowsum and stores bf16 ctx.
// No online rescaling: the whole row of scores is in TMEM when its max is taken.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "gx_internal.h"
#include "launch.cuh"
#include "philox.cuh"
#include "sm100.cuh"

namespace gx {

namespace {

constexpr int kTcQ = 128;        // queries per CTA (UMMA M)
constexpr int kTcMaxKeys = 512;  // TMEM columns
constexpr int kTcMaxHd = 80;     // backward TMEM budget: 256 + 3 * hd <= 512
constexpr int kMaxSide = 8;      // relative-position tables of up to (2*8 - 1)^2 entries
constexpr int kTabMax = (2 * kMaxSide - 1) * (2 * kMaxSide - 1);

// Geometry of one call, computed on the host and passed by value.
struct Geom {
  int hd;     // head dim (multiple of 16, <= 80)
  int np;     // 64-column panels per head row
  int wpt;    // attention sequences (units) per tile: 1, or 128 / seq for seq <= 64
  int vseq;   // rows (= keys) of a tile's virtual sequence: wpt * seq
  int nk;     // keys staged per forward CTA: vseq rounded up to 64
  int tiles;  // ceil(batch / wpt)
  int gmask;  // the general masked path: windows packed, causal, shifted regions or bias
  int fgen;   // forward: the general path (windows / regions / Swin bias); causal and the T5
              // bias ride the plain path with per-block masking
};

Geom make_geom(const gx_attention_args& a) {
  Geom g{};
  g.hd = a.head_dim;
  g.np = (a.head_dim + 63) / 64;
  g.wpt = a.seq <= 64 ? kTcQ / a.seq : 1;
  g.vseq = g.wpt * a.seq;
  g.nk = (g.vseq + 63) / 64 * 64;
  g.tiles = (a.batch + g.wpt - 1) / g.wpt;
  g.fgen = (g.wpt > 1 || a.win_shift > 0 || a.rpb != nullptr) ? 1 : 0;
  g.gmask = (g.wpt > 1 || a.causal || a.win_shift > 0 || a.rpb != nullptr || a.relb != nullptr)
                ? 1 : 0;
  return g;
}

// Per-tile window metadata staged in smem: token (in-window) coordinates, shifted-window
// region and the head's bias table (log2 units).
struct WinSmem {
  float rel[2 * kTcMaxKeys];  // T5 relative bias of relative position k - q + seq - 1 (log2 units)
  float tab[kTabMax];
  alignas(16) int16_t kc[kTcQ];  // ty * (2 side - 1) + tx: bias index = row base - kc[key]
  int8_t ty[kTcQ], tx[kTcQ];
  alignas(16) int8_t reg[kTcQ];  // (16 B aligned: read as vectors by the packed path)
};

// Swin shifted-window region (0..8) of token `tok` of attention sequence (window) `u`: the
// window's position in the rolled grid gives the token's (y, x); rows / columns within
// `side` of the far edge came from the other side of the grid (SW-MSA mask).
__device__ __forceinline__ int swin_region_tc(const gx_attention_args& p, int u, int tok) {
  const int nw = p.win_grid / p.win_side;
  const int w = u % (nw * nw);
  const int y = (w / nw) * p.win_side + tok / p.win_side;
  const int x = (w % nw) * p.win_side + tok % p.win_side;
  const int l0 = p.win_grid - p.win_side, l1 = p.win_grid - p.win_shift;
  return (y < l0 ? 0 : (y < l1 ? 1 : 2)) * 3 + (x < l0 ? 0 : (x < l1 ? 1 : 2));
}

__device__ __forceinline__ void win_stage_tc(const gx_attention_args& p, const Geom& g, int vb,
                                             int h, WinSmem* w, int nthreads) {
  const int s = p.seq;
  if (p.rpb != nullptr) {
    const int n = 2 * p.rpb_side - 1;
    const auto* t = static_cast<const __nv_bfloat16*>(p.rpb) + h * n * n;
    for (int e = threadIdx.x; e < n * n; e += nthreads)
      w->tab[e] = __bfloat162float(t[e]) * 1.4426950408889634f;
  }
  if (p.relb != nullptr) {  // T5: the head's bias of every relative position
    const auto* t = static_cast<const __nv_bfloat16*>(p.relb) + h * p.relb_buckets;
    const auto* map = static_cast<const int8_t*>(p.relb_map);
    for (int d = threadIdx.x; d < 2 * s - 1; d += nthreads)
      w->rel[d] = __bfloat162float(t[map[d]]) * 1.4426950408889634f;
  }
  for (int v = threadIdx.x; v < kTcQ; v += nthreads) {
    const int tok = v % s, u = vb * g.wpt + v / s;
    w->ty[v] = static_cast<int8_t>(p.rpb_side > 0 ? tok / p.rpb_side : 0);
    w->tx[v] = static_cast<int8_t>(p.rpb_side > 0 ? tok % p.rpb_side : 0);
    w->kc[v] = static_cast<int16_t>(w->ty[v] * (2 * p.rpb_side - 1) + w->tx[v]);
    w->reg[v] = static_cast<int8_t>(p.win_shift > 0 && v < g.vseq && u < p.batch
                                        ? swin_region_tc(p, u, tok) : 0);
  }
}

// keep bit of real key kk (0..63) of a 64-key block: word (kk/2)%4, bit 2*(kk/8) + kk%2
__device__ __forceinline__ uint32_t keep_bit(const uint32_t (&w)[4], int kk) {
  return (w[(kk >> 1) & 3] >> (2 * (kk >> 3) + (kk & 1))) & 1u;
}

struct FwdLayout {
  int kq, kv, p_lo, p_hi, win, red, kw, bar, bytes;
};
__host__ __device__ inline FwdLayout fwd_layout(int np, int nk) {
  FwdLayout L{};
  L.kq = np * kTcQ * 128;
  L.kv = L.kq + np * nk * 128;
  const int groups = nk / 64;
  L.p_lo = L.kv / (16 * 1024);  // P groups that fit over the dead Q + K tiles
  if (L.p_lo > groups) L.p_lo = groups;
  L.p_hi = L.kv + np * nk * 128;
  L.win = L.p_hi + (groups - L.p_lo) * 16 * 1024;
  L.red = L.win + static_cast<int>((sizeof(WinSmem) + 15) / 16 * 16);
  L.kw = L.red + 8 * kTcQ * 4;   // red: [max | sum][4 column quarters][128 rows]
  L.bar = L.kw + 4 * kTcQ * 4;   // kw: packed windows' keep words [4 calls][128 rows]
  L.bytes = L.bar + 64;
  return L;
}

__device__ __forceinline__ uint32_t p_group_addr(const FwdLayout& L, uint32_t base, int g) {
  return g < L.p_lo ? base + g * 16384 : base + L.p_hi + (g - L.p_lo) * 16384;
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
// TMA load of a 64 x 64 bf16 box of a 2-D [rows][ld] map (inner coordinate c0, row c1)
__device__ __forceinline__ void tma_box(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                        int c1) {
  tma_load_2d(dst, map, bar, c0, c1);
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

// kCB (plain path only): causal masking and / or the T5 relative bias, per 64-key block
template <uint32_t kCols, bool kGen, bool kCB = false>
__global__ void __launch_bounds__(kFwdThreads, (kGen && kCols == 128) ? 2 : 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap map_qkv, const gx_attention_args p,
                       const Geom g) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-align by offsetting the shared array itself, so every access below stays in the
  // shared state space (an integer-cast pointer would compile to generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int s = p.seq;
  const FwdLayout L = fwd_layout(g.np, g.nk);
  const uint32_t sbase = smem_u32(smem);
  float* red = reinterpret_cast<float*>(smem + L.red);  // [max|sum][quarter][128]
  WinSmem* win = reinterpret_cast<WinSmem*>(smem + L.win);
  uint64_t* bar_qk = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* bar_v = bar_qk + 1;
  uint64_t* bar_s = bar_qk + 2;
  uint64_t* bar_o = bar_qk + 3;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_qk + 4);

  const int warp = static_cast<int>(warp_id());
  const int lane = static_cast<int>(lane_id());
  const int H = p.heads, hd = g.hd, nk = g.nk, np = g.np;
  const int vb = blockIdx.y / H, h = blockIdx.y % H;
  const int q0 = blockIdx.x * kTcQ;
  const int row0 = vb * g.wpt * s;  // first token row of this tile's sequences

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
      const int cq = h * hd, ck = (H + h) * hd, cv = (2 * H + h) * hd;  // column of each slot
      // 64 x 64 boxes (128 B rows, 128B swizzle): Q 2 per panel, K and V nk/64 per panel
      mbar_expect_tx(bar_qk, np * (kTcQ + nk) * 128);
      for (int pn = 0; pn < np; ++pn) {
        tma_box(smem + pn * kTcQ * 128, &map_qkv, bar_qk, cq + pn * 64, row0 + q0);
        tma_box(smem + pn * kTcQ * 128 + 64 * 128, &map_qkv, bar_qk, cq + pn * 64, row0 + q0 + 64);
        for (int r = 0; r < nk; r += 64)
          tma_box(smem + L.kq + pn * nk * 128 + r * 128, &map_qkv, bar_qk, ck + pn * 64, row0 + r);
      }
      mbar_expect_tx(bar_v, np * nk * 128);
      for (int pn = 0; pn < np; ++pn)
        for (int r = 0; r < nk; r += 64)
          tma_box(smem + L.kv + pn * nk * 128 + r * 128, &map_qkv, bar_v, cv + pn * 64, row0 + r);
    }
    __syncwarp();
  }

  // ---------------------------------------------------------------- rows of this thread
  // 16 warps: four per TMEM lane quarter; 64-key blocks go round-robin to the four column
  // quarters (a block's two 32-key halves stay with one thread, so its Philox draws are
  // shared), and the quarters exchange row max / row sum through shared memory.
  const int qd = warp & 3, cq = warp >> 2;
  const int r = qd * 32 + lane;  // tile row == TMEM lane
  const int vq = q0 + r;         // virtual query
  const int u = vb * g.wpt + vq / s;  // its attention sequence (unit)
  const int q = vq % s;               // real query index
  const bool row_ok = vq < g.vseq && u < p.batch;
  const int nblk = nk / 64;
  const uint32_t thr = p.drop_threshold;
  const uint64_t seed = p.seed + (p.seed_offset != nullptr ? *p.seed_offset : 0ull);
  const int nkb = (s + 63) / 64;  // real 64-key blocks per query
  const uint64_t stream =
      (static_cast<uint64_t>(p.sample_offset + u) * p.heads_total + (p.head_offset + h)) * s;
  uint16_t* mask = static_cast<uint16_t*>(p.mask);
  const int64_t bh_real = static_cast<int64_t>(u) * H + h;
  // Plain path: the dropout keep bits depend only on (seed, site, element), so each thread
  // draws its blocks' Philox words while Q / K / V are still in flight (warp 0 before it
  // issues S = Q K^T), and stores them for the backward; the exp pass only tests bits.
  constexpr int kItems = (static_cast<int>(kCols) / 64 + 3) / 4;  // 64-key blocks per thread
  uint32_t kbits[kItems][4];
#pragma unroll
  for (int it = 0; it < kItems; ++it) kbits[it][0] = kbits[it][1] = kbits[it][2] = kbits[it][3] = 0u;
  if (!kGen && thr != 0u) {
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int kb = cq + 4 * it;
      if (kb < nblk) {
        keep16x4(seed, p.site, ((stream + static_cast<uint64_t>(q)) * nkb + kb) * 4, thr, kbits[it]);
        if (row_ok && kb < nkb)
          *reinterpret_cast<uint64_t*>(mask + ((bh_real * s + q) * nkb + kb) * 4) =
              static_cast<uint64_t>(kbits[it][0]) | (static_cast<uint64_t>(kbits[it][1]) << 16) |
              (static_cast<uint64_t>(kbits[it][2]) << 32) | (static_cast<uint64_t>(kbits[it][3]) << 48);
      }
    }
  }

  if (warp == 0) {
    if (lane == 0) {
      mbar_wait(bar_qk, 0);
      tc_fence_after();
      for (int n0 = 0; n0 < nk; n0 += 256) {
        const int n = nk - n0 < 256 ? nk - n0 : 256;
        const uint32_t idesc = idesc_bf16_f32(kTcQ, n, false, false);
        for (int ks = 0; ks < hd / 16; ++ks) {
          const int pn = ks >> 2, k = ks & 3;
          const uint64_t ad = sdesc_sw128(sbase + pn * kTcQ * 128 + k * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sbase + L.kq + pn * nk * 128 + n0 * 128 + k * 32, 16, 1024);
          umma_bf16(tmem + n0, ad, bd, idesc, ks != 0 ? 1u : 0u);
        }
      }
      umma_commit(bar_s);
    }
    __syncwarp();
  }
  const bool relb = (kGen || kCB) && p.relb != nullptr;  // T5 relative bias
  if (kGen || relb) win_stage_tc(p, g, vb, h, win, kFwdThreads);  // visible after the barrier below

  // ---------------------------------------------------------------- softmax over TMEM rows
  const uint32_t trow = tmem + (static_cast<uint32_t>(qd * 32) << 16);
  const float c2 = p.scale * 1.4426950408889634f;
  mbar_wait(bar_s, 0);
  tc_fence_after();
  if (kGen || relb) named_sync(1, kFwdThreads);  // window metadata staged
  GX_ATTN_STAMP(p, 2);

  // fast path (!kGen): keys [0, s) exist for every row; a 64-key block is either full or
  // the tail block, so only the tail compares per element.  The max is taken over the raw
  // scores (c2 > 0) and scaled once.
  // General path (kGen): per row, the attended keys are the virtual range [klo, khi) of the
  // row's own packed sequence (causal: up to the query), intersected with its shifted-window
  // region; the bias index is rowbase - kc[key].  Work goes in 32-column chunks: one per
  // quarter for packed windows (nk <= 128), else both halves of the 64-key blocks kb = cq +
  // 4 t (one Philox draw of four calls per block).
  const int klo = (vq / s) * s;
  const int khi = min(p.causal ? vq + 1 : klo + s, g.vseq);
  const int rq = kGen && p.win_shift > 0 ? win->reg[r] : 0;
  const int side = p.rpb_side;
  const int rowbase = kGen && p.rpb != nullptr
                          ? (win->ty[r] + side - 1) * (2 * side - 1) + win->tx[r] + side - 1 : 0;
  auto gen_x = [&](int c, uint32_t raw) -> float {  // scaled score, or -inf if not attended
    bool ok = c >= klo && c < khi;
    if (p.win_shift > 0) ok = ok && win->reg[c] == rq;
    if (!ok) return -INFINITY;
    float x = __uint_as_float(raw) * c2;
    if (p.rpb != nullptr) x += win->tab[rowbase - win->kc[c]];
    if (p.relb != nullptr) x += win->rel[c - vq + s - 1];
    return x;
  };
  const int nchunk = g.wpt > 1 ? 1 : 2;  // 32-column chunks per work item
  const int nitem = g.wpt > 1 ? (cq * 32 < nk ? 1 : 0) : (nblk - cq + 3) / 4;
  auto item_c0 = [&](int it, int hb) { return g.wpt > 1 ? cq * 32 : (cq + 4 * it) * 64 + hb * 32; };
  float mx = -INFINITY;
  // Packed short sequences (Swin windows): a warp owns exactly one 32-column chunk, so its
  // masked, biased scores are computed once here and kept in registers for the exp pass; the
  // per-column metadata (region id, bias-table coordinate) comes in with vector loads.
  float xs[32];
  const bool packed = kGen && g.wpt > 1;
  if (packed && nitem > 0) {
    const int c0 = cq * 32;
    uint32_t vmask = 0u;  // columns of this row's own window (range [klo, khi))
    {
      const int lo = max(klo - c0, 0), hi = min(khi - c0, 32);
      if (row_ok && hi > lo) vmask = (hi - lo == 32 ? ~0u : (1u << (hi - lo)) - 1u) << lo;
    }
    uint32_t regw[8], kcw[16];
    if (p.win_shift > 0) {
      const uint4 a = *reinterpret_cast<const uint4*>(&win->reg[c0]);
      const uint4 b = *reinterpret_cast<const uint4*>(&win->reg[c0 + 16]);
      regw[0] = a.x; regw[1] = a.y; regw[2] = a.z; regw[3] = a.w;
      regw[4] = b.x; regw[5] = b.y; regw[6] = b.z; regw[7] = b.w;
    }
    if (p.rpb != nullptr) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint4 a = *reinterpret_cast<const uint4*>(&win->kc[c0 + 8 * k]);
        kcw[4 * k] = a.x; kcw[4 * k + 1] = a.y; kcw[4 * k + 2] = a.z; kcw[4 * k + 3] = a.w;
      }
    }
    const bool any = __any_sync(0xffffffffu, vmask != 0u);
    uint32_t v[32];
    if (any) {
      tmem_ld32(trow + c0, v);
      tmem_ld_wait();
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      bool ok = any && ((vmask >> j) & 1u) != 0u;
      if (p.win_shift > 0)
        ok = ok && static_cast<int>(static_cast<int8_t>((regw[j >> 2] >> (8 * (j & 3))) & 0xffu)) == rq;
      float x = -INFINITY;
      if (ok) {
        x = __uint_as_float(v[j]) * c2;
        if (p.rpb != nullptr)
          x += win->tab[rowbase - static_cast<int>(static_cast<int16_t>((kcw[j >> 1] >> (16 * (j & 1))) & 0xffffu))];
      }
      xs[j] = x;
      mx = fmaxf(mx, x);
    }
  }
  if (kGen && !packed) {
    for (int it = 0; it < nitem; ++it)
      for (int hb = 0; hb < nchunk; ++hb) {
        const int c0 = item_c0(it, hb);
        // tcgen05.ld is warp-collective: skip a chunk only when no lane of the warp needs it
        if (!__any_sync(0xffffffffu, c0 < khi && c0 + 32 > klo)) continue;
        uint32_t v[32];
        tmem_ld32(trow + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, gen_x(c0 + j, v[j]));
      }
  }
  // plain path: raw maxima where no key is masked or biased (scaled once below), scaled maxima
  // of the masked / biased blocks (causal: keys past the row's query; T5: + bias)
  const bool causal = kCB && p.causal != 0;
  const int vq_lo_w = q0 + qd * 32;  // this warp's first row
  // T5 bias of key c for this row: relrow[c] (padding rows read row s - 1's; index <= 1022)
  const float* relrow = win->rel + (s - 1 - min(vq, s - 1));
  float mxs = -INFINITY;
  for (int kb = cq; kb < nblk && !kGen; kb += 4) {
    uint32_t v[64];
    tmem_ld32(trow + kb * 64, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
    tmem_ld32(trow + kb * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
    tmem_ld_wait();
    const bool clean = kb * 64 + 64 <= s && !(causal && kb * 64 + 63 > vq_lo_w) && !relb;
    if (clean) {
#pragma unroll
      for (int j = 0; j < 64; j += 2)
        mx = fmaxf(mx, fmaxf(__uint_as_float(v[j]), __uint_as_float(v[j + 1])));
    } else {
      float m2[2] = {-INFINITY, -INFINITY};  // (two chains: even / odd keys)
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int c = kb * 64 + j;
        float x = __uint_as_float(v[j]) * c2;
        if (relb) x += relrow[c];
        if (c < s && !(causal && c > vq)) m2[j & 1] = fmaxf(m2[j & 1], x);
      }
      mxs = fmaxf(mxs, fmaxf(m2[0], m2[1]));
    }
  }
  if (!kGen && mx != -INFINITY) mx *= c2;
  if (!kGen) mx = fmaxf(mx, mxs);
  // packed windows: the four column warps of a row split its four Philox calls (warp cq makes
  // call cq) and share the keep words through shared memory, instead of each drawing all four
  uint32_t* kwsm = reinterpret_cast<uint32_t*>(smem + L.kw);
  if (kGen && g.wpt > 1 && p.drop_threshold != 0u) {
    const uint64_t sd = p.seed + (p.seed_offset != nullptr ? *p.seed_offset : 0ull);
    const uint64_t st =
        (static_cast<uint64_t>(p.sample_offset + u) * p.heads_total + (p.head_offset + h)) * s;
    kwsm[cq * kTcQ + r] = keep16(sd, p.site, (st + static_cast<uint64_t>(q)) * ((s + 63) / 64) * 4 + cq,
                                 p.drop_threshold);
  }
  red[cq * kTcQ + r] = mx;
  named_sync(1, kFwdThreads);
  GX_ATTN_STAMP(p, 3);
  float m = fmaxf(fmaxf(red[r], red[kTcQ + r]), fmaxf(red[2 * kTcQ + r], red[3 * kTcQ + r]));
  if (m == -INFINITY) m = 0.f;  // an empty row (padding) keeps finite arithmetic

  const float inv_keep = p.drop_scale;
  // packed short sequences: one 64-key real block per query, drawn once per row
  uint32_t wrow[4] = {0u, 0u, 0u, 0u};
  if (kGen && g.wpt > 1 && thr != 0u) {
#pragma unroll
    for (int i = 0; i < 4; ++i) wrow[i] = kwsm[i * kTcQ + r];  // (staged before the max barrier)
    if (row_ok && cq == 0)
      *reinterpret_cast<uint64_t*>(mask + (bh_real * s + q) * nkb * 4) =
          static_cast<uint64_t>(wrow[0]) | (static_cast<uint64_t>(wrow[1]) << 16) |
          (static_cast<uint64_t>(wrow[2]) << 32) | (static_cast<uint64_t>(wrow[3]) << 48);
  }
  // P = exp2(S c2 + bias - m) with dropped keys zeroed; the keep scale 1 / (1 - p) is applied
  // once to O in the epilogue (row sums l are taken before dropout)
  float sum = 0.f;
  // one 32-column chunk of P -> the K-major SWIZZLE_128B tile of its 64-key group
  auto store_p = [&](int c0, const uint32_t (&pk)[16]) {
    const uint32_t g_addr = p_group_addr(L, sbase, c0 >> 6) + r * 128;
    const int hb = (c0 >> 5) & 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t sw = static_cast<uint32_t>((hb * 4 + i) ^ (r & 7));
      st_shared_v4_tc(g_addr + (sw << 4), pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
    }
  };
  if (packed && nitem > 0) {
    const int c0 = cq * 32;
    uint32_t pk[16];
#pragma unroll
    for (int j2 = 0; j2 < 16; ++j2) {
      float e2[2];
#pragma unroll
      for (int uu = 0; uu < 2; ++uu) {
        const int j = 2 * j2 + uu;
        float e = ex2_ftz(xs[j] - m);  // (-inf: not attended -> 0)
        sum += e;
        if (thr != 0u) e = keep_bit(wrow, (c0 + j - klo) & 63) ? e : 0.f;
        e2[uu] = e;
      }
      pk[j2] = pack_bf16(e2[0], e2[1]);
    }
    store_p(c0, pk);
  }
  if (kGen && !packed) {
    for (int it = 0; it < nitem; ++it) {
      uint32_t bits[4] = {wrow[0], wrow[1], wrow[2], wrow[3]};
      const int kb = g.wpt > 1 ? 0 : cq + 4 * it;
      if (thr != 0u && g.wpt == 1) {
        const uint64_t call0 = ((stream + static_cast<uint64_t>(q)) * nkb + kb) * 4;
        keep16x4(seed, p.site, call0, thr, bits);
        if (row_ok && kb < nkb)
          *reinterpret_cast<uint64_t*>(mask + ((bh_real * s + q) * nkb + kb) * 4) =
              static_cast<uint64_t>(bits[0]) | (static_cast<uint64_t>(bits[1]) << 16) |
              (static_cast<uint64_t>(bits[2]) << 32) | (static_cast<uint64_t>(bits[3]) << 48);
      }
      for (int hb = 0; hb < nchunk; ++hb) {
        const int c0 = item_c0(it, hb);
        uint32_t pk[16];
        if (!__any_sync(0xffffffffu, row_ok && c0 < khi && c0 + 32 > klo)) {
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = 0u;
        } else {
          uint32_t v[32];
          tmem_ld32(trow + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int j2 = 0; j2 < 16; ++j2) {
            float e2[2];
#pragma unroll
            for (int uu = 0; uu < 2; ++uu) {
              const int i = 2 * j2 + uu;
              const int c = c0 + i;
              const float x = row_ok ? gen_x(c, v[i]) : -INFINITY;
              float e = x == -INFINITY ? 0.f : ex2_ftz(x - m);
              sum += e;
              const int kk = g.wpt > 1 ? c - klo : (c & 63);
              if (thr != 0u) e = keep_bit(bits, kk) ? e : 0.f;
              e2[uu] = e;
            }
            pk[j2] = pack_bf16(e2[0], e2[1]);
          }
        }
        store_p(c0, pk);
      }
    }
  }
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int kb = cq + 4 * it;
    if (kGen || kb >= nblk) break;
    const uint32_t (&bits)[4] = kbits[it];  // drawn before S (above)
    // (warp-uniform: full blocks, i.e. all but a sequence's tail block, skip the per-key
    // bounds check; with dropout off the keep test is compiled out)
    uint32_t vv[2][32];  // both 32-column halves of the block in flight at once
    tmem_ld32(trow + kb * 64, vv[0]);
    tmem_ld32(trow + kb * 64 + 32, vv[1]);
    tmem_ld_wait();
    auto half = [&](auto tail_tag, auto drop_tag, auto bias_tag, int hb) {
      constexpr bool kTail = decltype(tail_tag)::value, kDrop = decltype(drop_tag)::value;
      constexpr bool kBias = decltype(bias_tag)::value;  // (full block, T5 bias only)
      const int c0 = kb * 64 + hb * 32;
      const uint32_t (&v)[32] = vv[hb];
      uint32_t pk[16];
#pragma unroll
      for (int j2 = 0; j2 < 16; ++j2) {
        float e2[2];
        // full, unbiased block: both exp arguments from one packed FFMA2 (not in the causal /
        // T5-bias instantiation: there it measured slower, 17.3 -> 20.0 us for T5 causal B = 2)
        float a2[2] = {0.f, 0.f};
        if constexpr (!kCB) {
          const f2 arg = f2_fma(f2_pack(__uint_as_float(v[2 * j2]), __uint_as_float(v[2 * j2 + 1])),
                                f2_splat(c2), f2_splat(-m));
          a2[0] = f2_lo(arg);
          a2[1] = f2_hi(arg);
        }
#pragma unroll
        for (int uu = 0; uu < 2; ++uu) {
          const int i = 2 * j2 + uu;
          float e;
          if (kTail && kCB) {  // masked / biased block: causal, tail keys, T5 bias
            const int c = c0 + i;
            const bool ok = c < s && !(causal && c > vq);
            const float b = relb ? relrow[c] : 0.f;
            e = ok ? ex2_ftz(fmaf(__uint_as_float(v[i]), c2, b - m)) : 0.f;
          } else if (kBias) {
            e = ex2_ftz(fmaf(__uint_as_float(v[i]), c2, relrow[c0 + i] - m));
          } else if (kTail) {  // tail keys only
            e = c0 + i < s ? ex2_ftz(fmaf(__uint_as_float(v[i]), c2, -m)) : 0.f;
          } else {
            e = ex2_ftz(kCB ? fmaf(__uint_as_float(v[i]), c2, -m) : a2[uu]);
          }
          sum += e;
          // compile-time key position: the keep bit's word and shift fold to constants
          if (kDrop) e = keep_bit(bits, hb * 32 + i) ? e : 0.f;
          e2[uu] = e;
        }
        pk[j2] = pack_bf16(e2[0], e2[1]);
      }
      store_p(c0, pk);
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    const bool full = kb * 64 + 64 <= s && !(causal && kb * 64 + 63 > vq_lo_w);
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      if (full && !relb) {
        if (thr != 0u) half(F_{}, T_{}, F_{}, hb); else half(F_{}, F_{}, F_{}, hb);
      } else if (kCB && full) {  // every key attended, T5 bias
        if (thr != 0u) half(F_{}, T_{}, T_{}, hb); else half(F_{}, F_{}, T_{}, hb);
      } else {
        if (thr != 0u) half(T_{}, T_{}, F_{}, hb); else half(T_{}, F_{}, F_{}, hb);
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
      const uint32_t idesc = idesc_bf16_f32(kTcQ, hd, false, true);
      for (int kk = 0; kk < nk / 16; ++kk) {
        const uint64_t ad = sdesc_sw128(p_group_addr(L, sbase, kk >> 2) + (kk & 3) * 32, 16, 1024);
        // V as MN-major B (N = hd): 64-column chunks are the panels, nk * 128 B apart
        const uint64_t bd = sdesc_sw128(sbase + L.kv + kk * 2048, nk * 128, 1024);
        umma_bf16(tmem, ad, bd, idesc, kk != 0 ? 1u : 0u);
      }
      umma_commit(bar_o);
    }
    __syncwarp();
  }
  if (cq == 0 && row_ok) {
    auto* lse = static_cast<float*>(p.lse);
    lse[bh_real * s + q] = m + log2f(l);
  }
  mbar_wait(bar_o, 0);
  tc_fence_after();
  GX_ATTN_STAMP(p, 5);
  const float inv = l > 0.f ? (thr != 0u ? inv_keep : 1.f) / l : 0.f;
  auto* ctx = static_cast<__nv_bfloat16*>(p.ctx);
  for (int c16 = cq; c16 < hd / 16; c16 += 4) {  // O columns [16 c16, 16 c16 + 16) of this row
    uint32_t o[16];
    tmem_ld16(trow + c16 * 16, o);
    tmem_ld_wait();
    if (row_ok) {
      uint4* out = reinterpret_cast<uint4*>(ctx + (static_cast<int64_t>(row0) + vq) * p.ld_ctx +
                                            h * hd + c16 * 16);
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
// One CTA per (tile x head, 128-key block); the queries stream through in 128-row chunks.
// Per chunk j, with K, V of the key block resident:
//   S^T = K Q_j^T and dPd^T = V dO_j^T                (tcgen05, TMEM cols [0,128) / [128,256))
//   P = exp2(S*c2 + bias - lse), Pd = drop(P), dP = drop(dPd), dS = P (dP - D)  (thread = key)
//   dV += Pd^T dO_j, dK += dS^T Q_j                    (TMEM cols 256 + [0, hd) / [hd, 2hd))
//   dQ_j = dS K  (dS^T's smem tile read as an MN-major A operand) -> fp32 partial per key block
// lse and the keep words of every query are staged in smem once; D = rowsum(dO * O) is
// computed per chunk from the dO tile in smem and O in global memory.  The key blocks of a
// head form one thread-block cluster: after a cluster barrier, CTA t sums the dQ partials of
// query chunk t over the key blocks in order, so the result is deterministic.
// Relative-position bias: the tile's fp32 dS is kept in smem and each (window, table entry)
// sums its (q, k) pairs in a fixed order into rpb_dpart (the batch sum follows in rpb_grad).
namespace {
struct BwdLayout {
  int nb;  // Q / dO chunk buffers (3: prefetch two chunks ahead; 1 when smem is short)
  int k, v, q, d_o, pd, ds, lse, dd, mask, win, ds32, diag, bar, bytes;
};
// rpb / relb: the fp32 dS tile of a chunk is kept for the bias gradients (relb: plus the
// per-relative-position sums of the CTA)
__host__ __device__ inline BwdLayout bwd_layout(int np, bool rpb, bool relb = false) {
  BwdLayout L{};
  L.nb = (np == 1 && !rpb && !relb) ? 3 : 1;
  const int tile = np * kTcQ * 128;  // one 128-row head tile
  L.k = 0;
  L.v = L.k + tile;
  L.q = L.v + tile;
  L.d_o = L.q + L.nb * tile;
  L.pd = L.d_o + L.nb * tile;
  L.ds = L.pd + 32768;
  L.lse = L.ds + 32768;                  // [512] floats
  L.dd = L.lse + 2048;                   // [512] floats: D of every query
  L.mask = L.dd + 2048;                  // [512 q][2 blocks][4] u16
  L.win = L.mask + 8192;
  L.ds32 = L.win + static_cast<int>((sizeof(WinSmem) + 15) / 16 * 16);
  L.diag = L.ds32 + (rpb || relb ? kTcQ * kTcQ * 4 : 0);  // fp32 dS [128 q][128 k]
  L.bar = L.diag + (relb ? 2 * kTcMaxKeys * 4 : 0);       // fp32 [2 seq - 1] dS sums
  L.bytes = L.bar + 128;
  return L;
}
}  // namespace

template <int HD, bool kGen>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap map_qkv,
                       const __grid_constant__ CUtensorMap map_do, const gx_attention_args p,
                       const Geom g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sb = smem_u32(smem);
  const bool has_rpb = kGen && p.rpb_dpart != nullptr;
  const bool has_relb = kGen && p.relb_dpart != nullptr;
  const BwdLayout BL = bwd_layout((HD + 63) / 64, has_rpb, has_relb);
  float* sDiag = reinterpret_cast<float*>(smem + BL.diag);
  float* sLse = reinterpret_cast<float*>(smem + BL.lse);
  float* sD = reinterpret_cast<float*>(smem + BL.dd);
  uint16_t* sMask = reinterpret_cast<uint16_t*>(smem + BL.mask);  // [512 q][2 kb][4]
  WinSmem* win = reinterpret_cast<WinSmem*>(smem + BL.win);
  float* sDs = reinterpret_cast<float*>(smem + BL.ds32);
  uint64_t* bar_kv = reinterpret_cast<uint64_t*>(smem + BL.bar);
  uint64_t* bar_ld = bar_kv + 1;  // [3]
  uint64_t* bar_s = bar_kv + 4;
  uint64_t* bar_mm = bar_kv + 5;
  uint64_t* bar_pds = bar_kv + 6;  // Pd / dS of a chunk stored (all softmax threads)
  uint64_t* bar_sfree = bar_kv + 7;  // S / dPd of a chunk read out of TMEM (all softmax threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_kv + 8);

  const int warp = static_cast<int>(warp_id());
  const int lane = static_cast<int>(lane_id());
  constexpr int hd = HD, np = (HD + 63) / 64;
  const int s = p.seq, H = p.heads, NB = BL.nb;
  const int vb = blockIdx.y / H, h = blockIdx.y % H;
  const int kt = blockIdx.x;  // key block
  const int nkt = gridDim.x;
  const int nq = (g.vseq + kTcQ - 1) / kTcQ;
  const int nkb = (s + 63) / 64;
  const int row0 = vb * g.wpt * s;
  const int tile = np * kTcQ * 128;
  // TMEM columns (hd is a multiple of 16): S^T, dPd^T, then dV, dK, dQ -- 256 + 3 hd <= 512;
  // when 256 + 4 hd fits, dQ is double-buffered so chunk j's products run while dQ(j-1)
  // drains to global memory
  constexpr bool kDqDbl = 256 + 4 * HD <= 512;
  const uint32_t t_dv = 256, t_dk = 256 + hd, t_dq = 256 + 2 * hd;

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    tma_prefetch(&map_do);
    mbar_init(bar_kv, 1);
    mbar_init(&bar_ld[0], 1);
    mbar_init(&bar_ld[1], 1);
    mbar_init(&bar_ld[2], 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_mm, 1);
    mbar_init(bar_pds, kBwdSoftmax);
    mbar_init(bar_sfree, kBwdSoftmax);
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
  if (!is_mma_warp) {  // lse and keep words of every query of the tile (once)
    const float* lse_g = static_cast<const float*>(p.lse);
    const uint16_t* mask_g = static_cast<const uint16_t*>(p.mask);
    for (int v = threadIdx.x; v < g.vseq; v += kBwdSoftmax) {
      const int u = vb * g.wpt + v / s;
      // staged negated (as is D): the exp argument and dP - D are then plain (packed) FMAs
      sLse[v] = u < p.batch ? -lse_g[(static_cast<int64_t>(u) * H + h) * s + v % s] : 0.f;
    }
    // (2 vseq <= 1024 words: both of a thread's loads issued before either store)
    uint64_t w[2];
  #pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int i = threadIdx.x + it * kBwdSoftmax;
      const int v = i >> 1, u = vb * g.wpt + v / s;
      // packed sequences: every query's keys lie in real block 0 (slot 0); else the key
      // block's two 64-key halves
      const int kb = g.wpt > 1 ? 0 : kt * 2 + (i & 1);
      w[it] = 0;
      if (i < 2 * g.vseq && p.drop_threshold != 0u && kb < nkb && u < p.batch &&
          (g.wpt == 1 || (i & 1) == 0))
        w[it] = *reinterpret_cast<const uint64_t*>(
            mask_g + (((static_cast<int64_t>(u) * H + h) * s + v % s) * nkb + kb) * 4);
    }
  #pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int i = threadIdx.x + it * kBwdSoftmax;
      if (i < 2 * g.vseq) *reinterpret_cast<uint64_t*>(sMask + i * 4) = w[it];
    }
    if (kGen) win_stage_tc(p, g, vb, h, win, kBwdSoftmax);
    if (has_relb)
      for (int d = threadIdx.x; d < 2 * s - 1; d += kBwdSoftmax) sDiag[d] = 0.f;
  }

  const int qd = warp & 3, cq = (warp >> 2) & 3;  // TMEM lane quarter, 32-column quarter
  const int kr = qd * 32 + lane;      // key row of the block == TMEM lane (S^T, dV, dK)
  const int key = kt * 128 + kr;      // virtual key
  const int ku = vb * g.wpt + key / s;  // its unit
  const bool key_ok = key < g.vseq && ku < p.batch;
  const uint32_t trow = tmem + (static_cast<uint32_t>(qd * 32) << 16);
  const float c2 = p.scale * 1.4426950408889634f;
  const uint32_t thr = p.drop_threshold;
  const float inv_keep = p.drop_scale;
  // keep-word slot and bit of this key: real key kk in its 64-key block
  const int kslot = g.wpt > 1 ? 0 : (kr >> 6);
  const int kk = g.wpt > 1 ? key % s : (kr & 63);
  const int mt = (kk >> 1) & 3, mbit = 2 * (kk >> 3) + (kk & 1);
  float* part = static_cast<float*>(p.dq_accum);
  // general path: queries attending this key (virtual indices), and its bias-index base
  const int qlo = p.causal ? key : (key / s) * s;
  const int qhi = min((key / s) * s + s, g.vseq);
  int kreg = 0, kbase = 0;  // (read from the staged window metadata after the first barrier)

  if (is_mma_warp) {
    // ------------------------------------------------ producer / MMA issue (one lane)
    // Softmax warps never wait on this warp directly: it consumes bar_pds (Pd / dS stored)
    // and publishes bar_s (next scores) and bar_mm (gradient products), so the issue
    // latency of the MMAs per chunk overlaps the softmax math instead of stalling it.
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16_f32(kTcQ, 128, false, false);
      const uint32_t idesc_kv = idesc_bf16_f32(128, hd, false, true);
      const uint32_t idesc_q = idesc_bf16_f32(kTcQ, hd, true, true);
      const int cqs = h * hd, cks = (H + h) * hd, cvs = (2 * H + h) * hd, cdo = h * hd;
      auto load_chunk = [&](int j) {  // Q_j, dO_j -> buffer j % NB
        const int bf = j % NB;
        const int r = row0 + j * kTcQ;
        mbar_expect_tx(&bar_ld[bf], 2 * tile);
        for (int pn = 0; pn < np; ++pn)
          for (int x = 0; x < 2; ++x) {
            tma_box(smem + BL.q + bf * tile + pn * 16384 + x * 8192, &map_qkv, &bar_ld[bf],
                    cqs + pn * 64, r + 64 * x);
            tma_box(smem + BL.d_o + bf * tile + pn * 16384 + x * 8192, &map_do, &bar_ld[bf],
                    cdo + pn * 64, r + 64 * x);
          }
      };
      auto issue_s = [&](int j) {  // S^T = K Q_j^T, dPd^T = V dO_j^T
        const int bf = j % NB;
        mbar_wait(&bar_ld[bf], (j / NB) & 1);
        tc_fence_after();
        const uint32_t q_b = sb + BL.q + bf * tile, do_b = sb + BL.d_o + bf * tile;
        for (int ks = 0; ks < hd / 16; ++ks) {
          const uint32_t o = (ks >> 2) * 16384 + (ks & 3) * 32;
          umma_bf16(tmem, sdesc_sw128(sb + BL.k + o, 16, 1024), sdesc_sw128(q_b + o, 16, 1024),
                    idesc_s, ks != 0 ? 1u : 0u);
          umma_bf16(tmem + 128, sdesc_sw128(sb + BL.v + o, 16, 1024),
                    sdesc_sw128(do_b + o, 16, 1024), idesc_s, ks != 0 ? 1u : 0u);
        }
        umma_commit(bar_s);
      };
      auto issue_grads = [&](int j) {  // dV += Pd^T dO_j, dK += dS^T Q_j, dQ_j = dS K
        const int bf = j % NB;
        const uint32_t q_b = sb + BL.q + bf * tile, do_b = sb + BL.d_o + bf * tile;
#pragma unroll
        for (int k = 0; k < kTcQ / 16; ++k) {
          const uint32_t a_kmaj = (k >> 2) * 16384 + (k & 3) * 32;
          const uint32_t acc = (j > 0 || k > 0) ? 1u : 0u;
          // MN-major B operands (N = hd): the 64-column chunks are the panels, 16 KB apart
          umma_bf16(tmem + t_dv, sdesc_sw128(sb + BL.pd + a_kmaj, 16, 1024),
                    sdesc_sw128(do_b + k * 2048, 16384, 1024), idesc_kv, acc);
          umma_bf16(tmem + t_dk, sdesc_sw128(sb + BL.ds + a_kmaj, 16, 1024),
                    sdesc_sw128(q_b + k * 2048, 16384, 1024), idesc_kv, acc);
          umma_bf16(tmem + t_dq + (kDqDbl ? (j & 1) * hd : 0), sdesc_sw128(sb + BL.ds + k * 2048, 16384, 1024),
                    sdesc_sw128(sb + BL.k + k * 2048, 16384, 1024), idesc_q, k > 0 ? 1u : 0u);
        }
        umma_commit(bar_mm);
      };
      mbar_expect_tx(bar_kv, 2 * tile);
      for (int pn = 0; pn < np; ++pn)
        for (int x = 0; x < 2; ++x) {
          tma_box(smem + BL.k + pn * 16384 + x * 8192, &map_qkv, bar_kv, cks + pn * 64,
                  row0 + kt * 128 + 64 * x);
          tma_box(smem + BL.v + pn * 16384 + x * 8192, &map_qkv, bar_kv, cvs + pn * 64,
                  row0 + kt * 128 + 64 * x);
        }
      for (int j = 0; j < nq && j < NB; ++j) load_chunk(j);
      mbar_wait(bar_kv, 0);
      issue_s(0);
      for (int j = 0; j < nq; ++j) {
        if (NB == 3) {
          // S / dPd(j) are in registers once bar_sfree(j) completes: the next chunk's scores
          // go into the same TMEM columns while the softmax warps still work on chunk j
          mbar_wait(bar_sfree, j & 1);
          tc_fence_after();
          if (j + 1 < nq) issue_s(j + 1);  // (chunk j + 1 was loaded one iteration ahead)
          if (j >= 1) {  // chunk j-1's products are done: its Q / dO buffer takes chunk j + 2
            mbar_wait(bar_mm, (j - 1) & 1);
            if (j + 2 < nq) load_chunk(j + 2);
          }
          mbar_wait(bar_pds, j & 1);  // Pd / dS(j) in smem; dQ buffer j & 1 drained
          tc_fence_after();
          issue_grads(j);
        } else {  // one buffer: chunk j's products finish before chunk j + 1 loads into it
          mbar_wait(bar_pds, j & 1);
          tc_fence_after();
          issue_grads(j);
          if (j + 1 < nq) {
            mbar_wait(bar_mm, j & 1);
            load_chunk(j + 1);
            issue_s(j + 1);
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax warps (0..15)
    // D = rowsum(dO * O) of every query of the tile -> sD (dO and O from global memory, four
    // threads per query; once, in the prologue, so no chunk waits on it).  Two 128-query passes
    // at a time with every load issued before the first use (the latency is paid once per
    // pair of passes, not per load); every lane runs every pass (warp-wide shuffles).
    {
      constexpr int kCc = (HD / 8 + 3) / 4;  // 8-column chunks per thread
      const int qi = threadIdx.x >> 2, part4 = threadIdx.x & 3;
      for (int v0 = 0; v0 < g.vseq; v0 += kBwdSoftmax / 2) {
        uint4 da[2][kCc], oa[2][kCc];
#pragma unroll
        for (int ps = 0; ps < 2; ++ps) {
          const int v = v0 + ps * (kBwdSoftmax / 4) + qi;
          const bool ok = v < g.vseq && vb * g.wpt + v / s < p.batch;
          const int64_t ro = (static_cast<int64_t>(row0) + v) * p.ld_ctx + h * hd;
#pragma unroll
          for (int c = 0; c < kCc; ++c) {
            const int cc = part4 + 4 * c;
            if (ok && cc < hd / 8) {
              da[ps][c] = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.dctx) + ro + cc * 8);
              oa[ps][c] = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.ctx) + ro + cc * 8);
            } else {
              da[ps][c] = make_uint4(0u, 0u, 0u, 0u);
              oa[ps][c] = make_uint4(0u, 0u, 0u, 0u);
            }
          }
        }
#pragma unroll
        for (int ps = 0; ps < 2; ++ps) {
          float acc = 0.f;
#pragma unroll
          for (int c = 0; c < kCc; ++c) {  // (zero words add exact zeros)
            const uint32_t aw[4] = {da[ps][c].x, da[ps][c].y, da[ps][c].z, da[ps][c].w};
            const uint32_t ow[4] = {oa[ps][c].x, oa[ps][c].y, oa[ps][c].z, oa[ps][c].w};
#pragma unroll
            for (int t = 0; t < 4; ++t)
              acc += bf16_lo(aw[t]) * bf16_lo(ow[t]) + bf16_hi(aw[t]) * bf16_hi(ow[t]);
          }
          acc += __shfl_xor_sync(0xffffffff, acc, 1);
          acc += __shfl_xor_sync(0xffffffff, acc, 2);
          // (queries past the tile's end get D = 0: the last chunk reads them, and a stale
          // smem value could be NaN, which the zero P of a masked pair would not cancel)
          const int v = v0 + ps * (kBwdSoftmax / 4) + qi;
          if (part4 == 0) sD[v] = -acc;
        }
      }
    }
    // dQ_j partial (fp32) out of TMEM (lane = query row of the chunk, 16 columns per load)
    // dQ_j partial (fp32) out of TMEM (lane = query row of the chunk, 16 columns per load),
    // stored column-major per (key block, sequence x head): [hd][vld] (vld = vseq rounded up
    // to 4), so a warp's 32 lanes (consecutive queries) write 128 contiguous bytes per column
    const int vld = (g.vseq + 3) & ~3;
    auto store_dq = [&](int j) {
      const int v = j * kTcQ + kr;
      const uint32_t tq = t_dq + (kDqDbl ? (j & 1) * hd : 0);
      for (int c16 = cq; c16 < hd / 16; c16 += 4) {
        uint32_t o[16];
        tmem_ld16(trow + tq + c16 * 16, o);
        tmem_ld_wait();
        if (nkt == 1) {  // the only key block: dQ is final -- bf16 straight into dqkv
          if (v < g.vseq && vb * g.wpt + v / s < p.batch) {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.dqkv) +
                                                  (static_cast<int64_t>(row0) + v) * p.ld_qkv +
                                                  h * hd + c16 * 16);
            const float sc = p.scale;
#pragma unroll
            for (int i = 0; i < 2; ++i)
              dst[i] = make_uint4(pack_bf16(__uint_as_float(o[8 * i]) * sc, __uint_as_float(o[8 * i + 1]) * sc),
                                  pack_bf16(__uint_as_float(o[8 * i + 2]) * sc, __uint_as_float(o[8 * i + 3]) * sc),
                                  pack_bf16(__uint_as_float(o[8 * i + 4]) * sc, __uint_as_float(o[8 * i + 5]) * sc),
                                  pack_bf16(__uint_as_float(o[8 * i + 6]) * sc, __uint_as_float(o[8 * i + 7]) * sc));
          }
        } else if (v < g.vseq) {
          float* dst = part + ((static_cast<int64_t>(kt) * gridDim.y + blockIdx.y) * hd + c16 * 16) *
                                  vld + v;
#pragma unroll
          for (int i = 0; i < 16; ++i) dst[static_cast<int64_t>(i) * vld] = __uint_as_float(o[i]);
        }
      }
    };
    named_sync(1, kBwdSoftmax);  // sD, sLse, sMask and the window metadata staged
    if (kGen && key < kTcQ) {
      if (p.win_shift > 0) kreg = win->reg[key];
      if (p.rpb != nullptr)
        kbase = (p.rpb_side - 1) * (2 * p.rpb_side - 1) + p.rpb_side - 1 - win->kc[key];
    }
    GX_ATTN_STAMP(p, 2);
    for (int j = 0; j < nq; ++j) {
      mbar_wait(bar_s, j & 1);
      tc_fence_after();
      GX_ATTN_STAMP(p, 4 + 5 * j);
      const int c0 = cq * 32;
      const int qg0 = j * kTcQ + c0;  // first virtual query of this warp's 32
      uint32_t ppd[16], pds[16];
      if (!kGen) {
        // Plain (unmasked) path: the validity of a partial chunk is one bit mask, the keep bit
        // one shared load at a compile-time offset, and every element is FFMA, EX2, two
        // selects and three multiply-adds.
        uint32_t sv[32], dv[32];
        tmem_ld32(trow + c0, sv);
        tmem_ld32(trow + 128 + c0, dv);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(bar_sfree);  // the MMA warp may overwrite S / dPd with the next chunk's
        // this key's keep word for query qg0 + i sits i * 16 B further (compile-time offsets)
        const uint16_t* mk = sMask + (qg0 * 2 + kslot) * 4 + mt;
        const uint32_t mbitm = 1u << mbit;
        // valid (query, key) pairs of this 32-query slice: query < s and key < s
        const uint32_t vmask = key >= s || qg0 >= s ? 0u
                               : (qg0 + 32 <= s ? ~0u : (1u << (s - qg0)) - 1u);
        const float fk = thr != 0u ? inv_keep : 1.f;
#pragma unroll
        for (int i4 = 0; i4 < 8; ++i4) {
          const float4 l4 = *reinterpret_cast<const float4*>(sLse + qg0 + 4 * i4);
          const float4 d4 = *reinterpret_cast<const float4*>(sD + qg0 + 4 * i4);
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dd[4] = {d4.x, d4.y, d4.z, d4.w};
          float pd4[4], ds4[4];
          // (lv, dd hold -lse, -D) pairs of queries on packed fp32 math: FFMA2 / FMUL2
#pragma unroll
          for (int t = 0; t < 4; t += 2) {
            const int i = 4 * i4 + t;
            const f2 arg = f2_fma(f2_pack(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])),
                                  f2_splat(c2), f2_pack(lv[t], lv[t + 1]));
            float pr0 = ex2_ftz(f2_lo(arg)), pr1 = ex2_ftz(f2_hi(arg));
            pr0 = (vmask >> i) & 1u ? pr0 : 0.f;  // (padding: lse / D may be stale there)
            pr1 = (vmask >> (i + 1)) & 1u ? pr1 : 0.f;
            const float f0 = thr == 0u || (mk[i * 8] & mbitm) != 0u ? fk : 0.f;
            const float f1 = thr == 0u || (mk[(i + 1) * 8] & mbitm) != 0u ? fk : 0.f;
            const f2 pr = f2_pack(pr0, pr1), f = f2_pack(f0, f1);
            const f2 pd = f2_mul(pr, f);
            const f2 ds = f2_mul(pr, f2_fma(f2_pack(__uint_as_float(dv[i]), __uint_as_float(dv[i + 1])),
                                            f, f2_pack(dd[t], dd[t + 1])));
            pd4[t] = f2_lo(pd);
            pd4[t + 1] = f2_hi(pd);
            ds4[t] = f2_lo(ds);
            ds4[t + 1] = f2_hi(ds);
          }
          ppd[2 * i4] = pack_bf16(pd4[0], pd4[1]);
          ppd[2 * i4 + 1] = pack_bf16(pd4[2], pd4[3]);
          pds[2 * i4] = pack_bf16(ds4[0], ds4[1]);
          pds[2 * i4 + 1] = pack_bf16(ds4[2], ds4[3]);
        }
      } else {
        uint32_t sv[32], dv[32];
        tmem_ld32(trow + c0, sv);
        tmem_ld32(trow + 128 + c0, dv);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(bar_sfree);  // the MMA warp may overwrite S / dPd with the next chunk's
        // the key's own packed sequence / causal range [qlo, qhi) as one 32-bit mask over the
        // warp's queries; its shifted-window region and the biases per pair (see the forward)
        uint32_t vmask = 0u;
        if (key_ok) {
          const int lo = max(qlo - qg0, 0), hi = min(qhi - qg0, 32);
          if (hi > lo) vmask = (hi - lo == 32 ? ~0u : (1u << (hi - lo)) - 1u) << lo;
        }
        const uint16_t* mk = sMask + (qg0 * 2 + kslot) * 4 + mt;  // keep word of query qg0 + i: + 8 i
        const uint32_t mbitm = 1u << mbit;
        const float fk = thr != 0u ? inv_keep : 1.f;
#pragma unroll
        for (int i4 = 0; i4 < 8; ++i4) {
          const float4 l4 = *reinterpret_cast<const float4*>(sLse + qg0 + 4 * i4);
          const float4 d4 = *reinterpret_cast<const float4*>(sD + qg0 + 4 * i4);
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dd[4] = {d4.x, d4.y, d4.z, d4.w};
          float pd4[4], ds4[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int i = 4 * i4 + t;
            const int qg = qg0 + i;
            bool valid = ((vmask >> i) & 1u) != 0u;
            if (p.win_shift > 0) valid = valid && win->reg[qg] == kreg;
            float bias = 0.f;
            if (valid && p.rpb != nullptr) bias = win->tab[win->kc[qg] + kbase];
            if (valid && p.relb != nullptr) bias += win->rel[key - qg + s - 1];
            float pr = ex2_ftz(fmaf(__uint_as_float(sv[i]), c2, bias + lv[t]));  // (lv = -lse)
            pr = valid ? pr : 0.f;
            const float f = thr == 0u || (mk[i * 8] & mbitm) != 0u ? fk : 0.f;
            pd4[t] = pr * f;
            ds4[t] = pr * fmaf(__uint_as_float(dv[i]), f, dd[t]);  // (dd = -D)
            if (has_rpb || has_relb) sDs[(c0 + i) * kTcQ + kr] = ds4[t];
          }
          ppd[2 * i4] = pack_bf16(pd4[0], pd4[1]);
          ppd[2 * i4 + 1] = pack_bf16(pd4[2], pd4[3]);
          pds[2 * i4] = pack_bf16(ds4[0], ds4[1]);
          pds[2 * i4 + 1] = pack_bf16(ds4[2], ds4[3]);
        }
      }
      GX_ATTN_STAMP(p, 5 + 5 * j);
      if (j > 0) {  // chunk j-1's gradient MMAs are done reading Pd / dS
        mbar_wait(bar_mm, (j - 1) & 1);
        tc_fence_after();
        if (!kDqDbl) store_dq(j - 1);  // (single dQ buffer: drained before chunk j's products)
      }
      GX_ATTN_STAMP(p, 6 + 5 * j);
      {
        const uint32_t rowoff = static_cast<uint32_t>((cq >> 1) * 16384 + kr * 128);
        const int chunk0 = (cq & 1) * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t sw = static_cast<uint32_t>((chunk0 + i) ^ (kr & 7)) << 4;
          st_shared_v4_tc(sb + BL.pd + rowoff + sw, ppd[4 * i], ppd[4 * i + 1], ppd[4 * i + 2],
                          ppd[4 * i + 3]);
          st_shared_v4_tc(sb + BL.ds + rowoff + sw, pds[4 * i], pds[4 * i + 1], pds[4 * i + 2],
                          pds[4 * i + 3]);
        }
      }
      fence_proxy_async_smem_tc();
      if (kDqDbl && j > 0) {
        tc_fence_before();
        mbar_arrive(bar_pds);  // the MMA warp may issue the gradients of chunk j ...
        store_dq(j - 1);       // ... into the other dQ buffer while this one drains
      } else {
        tc_fence_before();
        mbar_arrive(bar_pds);
      }
      GX_ATTN_STAMP(p, 7 + 5 * j);
      if (has_relb) {
        // T5 bias gradient: thread t sums the chunk tile's diagonal delta = key - query
        // (local) = t - 127 in query order and adds it to the CTA's sum of relative position
        // (kt - j) 128 + delta; chunks go in order (deterministic)
        // All 512 threads: thread t sums one half (t / 256) of diagonal t % 256 - 127 with
        // four interleaved accumulators; the halves are added in order after a barrier.
        named_sync(1, kBwdSoftmax);  // the fp32 dS tile of chunk j is complete
        const int dl = static_cast<int>(threadIdx.x & 255);
        const int delta = dl - (kTcQ - 1);
        float acc = 0.f;
        if (dl < 2 * kTcQ - 1) {
          const int lo = max(0, -delta), hi = min(kTcQ, kTcQ - delta);
          const int mid = (lo + hi) >> 1;
          const int a0 = threadIdx.x < 256 ? lo : mid, a1 = threadIdx.x < 256 ? mid : hi;
          float e[4] = {0.f, 0.f, 0.f, 0.f};
          int qi = a0;
          for (; qi + 3 < a1; qi += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] += sDs[(qi + u) * (kTcQ + 1) + delta];
          }
          for (; qi < a1; ++qi) e[0] += sDs[qi * (kTcQ + 1) + delta];
          acc = (e[0] + e[1]) + (e[2] + e[3]);
        }
        float* dhalf = sDs + kTcQ * kTcQ - 256;  // (row 127's last 256 words: read above)
        named_sync(1, kBwdSoftmax);
        if (threadIdx.x >= 256) dhalf[dl] = acc;
        named_sync(1, kBwdSoftmax);
        if (threadIdx.x < 2 * kTcQ - 1) {
          const int idx = (kt - j) * kTcQ + delta + s - 1;
          if (idx >= 0 && idx < 2 * s - 1) sDiag[idx] += acc + dhalf[dl];
        }
      }
      // the fp32 dS tile (bias gradients) is rewritten by the next chunk: all readers first
      if (has_rpb || has_relb) named_sync(1, kBwdSoftmax);
      GX_ATTN_STAMP(p, 8 + 5 * j);
    }
    if (has_rpb) {
      // each (window of the tile, bias-table entry e) sums dS over its (q, k) pairs at
      // relative offset e in a fixed order (vseq <= 128: one key block, one query chunk)
      const int side = p.rpb_side, n = 2 * side - 1;
      for (int task = threadIdx.x; task < g.wpt * n * n; task += kBwdSoftmax) {
        const int wl = task / (n * n), e = task % (n * n);
        const int u = vb * g.wpt + wl;
        if (u >= p.batch) continue;
        const int dy = e / n - (side - 1), dx = e % n - (side - 1);
        // the query tokens (yq, xq) whose key (yq - dy, xq - dx) lies in the window, in
        // increasing token order (the same pairs and order as a scan over all queries)
        float acc = 0.f;
        const int y0 = max(0, dy), y1 = min(side, side + dy);
        const int x0 = max(0, dx), x1 = min(side, side + dx);
        const float* base = sDs + wl * s * kTcQ + wl * s;
        for (int yq = y0; yq < y1; ++yq)
          for (int xq = x0; xq < x1; ++xq)
            acc += base[(yq * side + xq) * kTcQ + (yq - dy) * side + (xq - dx)];
        static_cast<float*>(p.rpb_dpart)[(static_cast<int64_t>(u) * H + h) * n * n + e] = acc;
      }
    }
    if (has_relb) {  // (the last chunk's sums are visible after the chunk-end barrier)
      float* out = static_cast<float*>(p.relb_dpart) +
                   (static_cast<int64_t>(blockIdx.y) * nkt + kt) * (2 * s - 1);
      for (int d = threadIdx.x; d < 2 * s - 1; d += kBwdSoftmax) out[d] = sDiag[d];
    }
    mbar_wait(bar_mm, (nq - 1) & 1);
    tc_fence_after();
    store_dq(nq - 1);
    // dK (x scale), dV -> bf16 rows of dqkv
    auto* dqkv = static_cast<__nv_bfloat16*>(p.dqkv);
    __nv_bfloat16* rowp = dqkv + (static_cast<int64_t>(row0) + key) * p.ld_qkv;
    const float sc = p.scale;
    for (int c16 = cq; c16 < hd / 16; c16 += 4) {
      uint32_t dvv[16], dkv[16];
      tmem_ld16(trow + t_dv + c16 * 16, dvv);
      tmem_ld16(trow + t_dk + c16 * 16, dkv);
      tmem_ld_wait();
      if (key_ok) {
        uint4* dvp = reinterpret_cast<uint4*>(rowp + (2 * H + h) * hd + c16 * 16);
        uint4* dkp = reinterpret_cast<uint4*>(rowp + (H + h) * hd + c16 * 16);
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
  // every key block's dQ partials are in global memory after the cluster barrier; CTA kt then
  // owns query chunk kt and sums its partials in key-block order
  GX_ATTN_STAMP(p, 25);
  if (nkt > 1) {  // (one key block: dQ was written final above)
  __threadfence();
  cluster_sync();
  GX_ATTN_STAMP(p, 26);
  {
    // per (4 queries, 4 columns): the key blocks' partials (column-major [hd][vseq] each;
    // consecutive threads = consecutive query quads: 16 B coalesced loads), summed in
    // key-block order; two key blocks' loads in flight at a time
    auto* dq = static_cast<__nv_bfloat16*>(p.dqkv);
    const float* __restrict__ src0 = part;
    const float sc = p.scale;
    const int q_lo = kt * kTcQ, q_hi = min(g.vseq, q_lo + kTcQ);
    const int nq4 = (q_hi - q_lo + 3) / 4, c4n = hd / 4;
    const int vld = (g.vseq + 3) & ~3;  // column stride of the partials (16 B aligned quads)
    for (int idx = threadIdx.x; idx < nq4 * c4n; idx += kBwdThreads) {
      const int v0 = q_lo + 4 * (idx % nq4), c0 = 4 * (idx / nq4);
      float a[4][4] = {};  // [query][column]
      for (int t0 = 0; t0 < nkt; t0 += 2) {
        float4 x[2][4];
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          const int t = t0 + tt;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float* src = src0 + ((static_cast<int64_t>(t) * gridDim.y + blockIdx.y) * hd +
                                       c0 + cc) * vld + v0;
            if (t >= nkt) {
              x[tt][cc] = make_float4(0.f, 0.f, 0.f, 0.f);
            } else if (v0 + 4 <= q_hi) {
              x[tt][cc] = __ldcg(reinterpret_cast<const float4*>(src));
            } else {
              x[tt][cc] = make_float4(v0 < q_hi ? __ldcg(src) : 0.f,
                                      v0 + 1 < q_hi ? __ldcg(src + 1) : 0.f,
                                      v0 + 2 < q_hi ? __ldcg(src + 2) : 0.f,
                                      v0 + 3 < q_hi ? __ldcg(src + 3) : 0.f);
            }
          }
        }
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
          if (t0 + tt >= nkt) break;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            a[0][cc] += x[tt][cc].x;
            a[1][cc] += x[tt][cc].y;
            a[2][cc] += x[tt][cc].z;
            a[3][cc] += x[tt][cc].w;
          }
        }
      }
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const int v = v0 + qq;
        if (v >= q_hi || vb * g.wpt + v / s >= p.batch) continue;
        *reinterpret_cast<uint2*>(dq + (static_cast<int64_t>(row0) + v) * p.ld_qkv + h * hd + c0) =
            make_uint2(pack_bf16(a[qq][0] * sc, a[qq][1] * sc),
                       pack_bf16(a[qq][2] * sc, a[qq][3] * sc));
      }
    }
  }
  }  // nkt > 1
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

// 2-D [rows][ld] bf16 map, 64 x 64 boxes, 128 B swizzle (columns past ld / rows past the end
// read as zero)
static bool make_map_2d(CUtensorMap* map, const void* base, uint64_t ld, uint64_t rows) {
  auto fn = encode_fn_tc();
  if (fn == nullptr) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool attention_tc_supported(const gx_attention_args& a) {
  if (a.head_dim % 16 != 0 || a.head_dim < 32 || a.head_dim > kTcMaxHd || a.seq < 1 ||
      a.batch < 1)
    return false;
  const Geom g = make_geom(a);
  if (g.nk > kTcMaxKeys) return false;
  if (fwd_layout(g.np, g.nk).bytes + 1024 > 227 * 1024) return false;
  if (a.rpb != nullptr && (a.seq > 64 || a.rpb_side < 1 || a.rpb_side > kMaxSide ||
                           a.rpb_side * a.rpb_side != a.seq))
    return false;
  if (a.win_shift > 0 && a.seq > 64) return false;
  if (a.relb != nullptr && (a.relb_map == nullptr || a.relb_buckets < 1 || a.relb_buckets > 127))
    return false;
  if (g.gmask && g.vseq > kTcQ && g.wpt > 1) return false;
  return (a.ld_qkv % 8) == 0 && (a.ld_ctx % 8) == 0 &&
         (reinterpret_cast<uintptr_t>(a.qkv) % 16) == 0 &&
         (reinterpret_cast<uintptr_t>(a.ctx) % 16) == 0;
}

int attention_fwd_tc(const gx_attention_args& a, cudaStream_t st) {
  const Geom g = make_geom(a);
  CUtensorMap map;
  const uint64_t rows = static_cast<uint64_t>(a.batch) * a.seq;
  if (!make_map_2d(&map, a.qkv, a.ld_qkv, rows))
    return set_error(kErrCuda, "attention_tc: tensor map encode failed");
  const int smem = fwd_layout(g.np, g.nk).bytes + 1024;
  dim3 grid((g.vseq + kTcQ - 1) / kTcQ, g.tiles * a.heads);
#define GX_ATTN_TC(C, G, CB)                                                                     \
  {                                                                                          \
    static bool set = false;                                                                 \
    if (!set) {                                                                              \
      cudaFuncSetAttribute(attn_fwd_tc_kernel<C, G, CB>,                                         \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);         \
      set = true;                                                                            \
    }                                                                                        \
    launch_k(attn_fwd_tc_kernel<C, G, CB>, grid, dim3(kFwdThreads), smem, st, map, a, g);        \
  }
  if (g.fgen) {
    if (g.nk <= 128) GX_ATTN_TC(128, true, false)
    else if (g.nk <= 256) GX_ATTN_TC(256, true, false)
    else GX_ATTN_TC(512, true, false)
  } else if (a.causal || a.relb != nullptr) {
    if (g.nk <= 128) GX_ATTN_TC(128, false, true)
    else if (g.nk <= 256) GX_ATTN_TC(256, false, true)
    else GX_ATTN_TC(512, false, true)
  } else {
    if (g.nk <= 128) GX_ATTN_TC(128, false, false)
    else if (g.nk <= 256) GX_ATTN_TC(256, false, false)
    else GX_ATTN_TC(512, false, false)
  }
#undef GX_ATTN_TC
  return check_launch("attn_fwd_tc_kernel");
}

int attention_bwd_tc(const gx_attention_args& a, cudaStream_t st) {
  const Geom g = make_geom(a);
  if (a.rpb_dpart != nullptr && g.vseq > kTcQ)
    return set_error(kErrConfig, "attention_tc: bias gradient needs sequences of <= 128 rows");
  const uint64_t rows = static_cast<uint64_t>(a.batch) * a.seq;
  CUtensorMap mq, md;
  if (!make_map_2d(&mq, a.qkv, a.ld_qkv, rows) || !make_map_2d(&md, a.dctx, a.ld_ctx, rows))
    return set_error(kErrCuda, "attention_tc: tensor map encode failed");
  if (a.relb_dpart != nullptr && g.np > 1)
    return set_error(kErrConfig, "attention_tc: the T5 bias gradient needs head_dim <= 64");
  const int smem = bwd_layout(g.np, a.rpb_dpart != nullptr, a.relb_dpart != nullptr).bytes + 1024;
  dim3 grid((g.vseq + 127) / 128, g.tiles * a.heads);
  // the key blocks of one tile x head form a cluster (dQ reduction after a cluster barrier)
#define GX_ATTN_BWD(D, G)                                                                    \
  {                                                                                          \
    static bool set = false;                                                                 \
    if (!set) {                                                                              \
      cudaFuncSetAttribute(attn_bwd_tc_kernel<D, G>,                                         \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);         \
      set = true;                                                                            \
    }                                                                                        \
    launch_k_cluster(attn_bwd_tc_kernel<D, G>, grid, dim3(kBwdThreads), smem, st,            \
                     static_cast<unsigned>(grid.x), mq, md, a, g);                           \
  }
  const bool gen = g.gmask || a.rpb_dpart != nullptr || a.relb_dpart != nullptr;
  switch (a.head_dim) {
    case 32: if (gen) GX_ATTN_BWD(32, true) else GX_ATTN_BWD(32, false) break;
    case 48: if (gen) GX_ATTN_BWD(48, true) else GX_ATTN_BWD(48, false) break;
    case 64: if (gen) GX_ATTN_BWD(64, true) else GX_ATTN_BWD(64, false) break;
    case 80: if (gen) GX_ATTN_BWD(80, true) else GX_ATTN_BWD(80, false) break;
    default: return set_error(kErrConfig, "attention_tc: backward head_dim must be 32, 48, 64 or 80");
  }
#undef GX_ATTN_BWD
  return check_launch("attn_bwd_tc_kernel");
}

}  // namespace gx
