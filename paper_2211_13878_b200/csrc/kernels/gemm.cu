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
#include <cstdio>

#include "gx_internal.h"
#include "philox.cuh"
#include "sm100.cuh"

namespace gx {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 B = one swizzle span
constexpr int kThreads = 256;

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}
// d/dx [x * Phi(x)] = Phi(x) + x * phi(x)
__device__ __forceinline__ float gelu_erf_grad(float x) {
  return 0.5f * (1.0f + erff(x * 0.70710678118654752f)) +
         x * 0.3989422804014327f * __expf(-0.5f * x * x);
}

// Applies the epilogue to 32 consecutive accumulator columns [n0, n0+32) of row `row`.
__device__ __forceinline__ void epilogue_row32(const GemmEpilogue& ep, int64_t row, int n0,
                                               int N, const uint32_t (&acc)[32]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(acc[j]) * ep.alpha;
  const bool full = n0 + 32 <= N;
  const __nv_bfloat16* bias = static_cast<const __nv_bfloat16*>(ep.bias);
  const __nv_bfloat16* residual = static_cast<const __nv_bfloat16*>(ep.residual);
  if (bias != nullptr) {
    if (full) {
      const uint4* bp = reinterpret_cast<const uint4*>(bias + n0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 b = __ldg(bp + q);
        const uint32_t w[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          v[q * 8 + 2 * t] += bf16_lo(w[t]);
          v[q * 8 + 2 * t + 1] += bf16_hi(w[t]);
        }
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) v[j] += __bfloat162float(bias[n0 + j]);
    }
  }
  if (ep.gelu_bwd) {
    // dgrad epilogue of the MLP up-projection: v <- v * gelu'(pre)
    const __nv_bfloat16* auxp = static_cast<const __nv_bfloat16*>(ep.aux) + row * ep.ld_aux + n0;
    if (full) {
      const uint4* ap = reinterpret_cast<const uint4*>(auxp);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 b = ap[q];
        const uint32_t w[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          v[q * 8 + 2 * t] *= gelu_erf_grad(bf16_lo(w[t]));
          v[q * 8 + 2 * t + 1] *= gelu_erf_grad(bf16_hi(w[t]));
        }
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) v[j] *= gelu_erf_grad(__bfloat162float(auxp[j]));
    }
  }
  if (ep.gelu) {
    // aux <- pre-activation (needed by the GeLU backward), v <- gelu(v)
    __nv_bfloat16* auxp = static_cast<__nv_bfloat16*>(ep.aux) + row * ep.ld_aux + n0;
    if (full) {
      uint4* ap = reinterpret_cast<uint4*>(auxp);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 o;
        o.x = pack_bf16(v[q * 8 + 0], v[q * 8 + 1]);
        o.y = pack_bf16(v[q * 8 + 2], v[q * 8 + 3]);
        o.z = pack_bf16(v[q * 8 + 4], v[q * 8 + 5]);
        o.w = pack_bf16(v[q * 8 + 6], v[q * 8 + 7]);
        ap[q] = o;
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) auxp[j] = __float2bfloat16_rn(v[j]);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      // GeLU is applied to the bf16-rounded pre-activation so forward and backward agree.
      const float pre = __bfloat162float(__float2bfloat16_rn(v[j]));
      v[j] = gelu_erf(pre);
    }
  }
  if (residual != nullptr) {
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
    for (int j = 0; j < 32; ++j) v[j] = __bfloat162float(__float2bfloat16_rn(v[j]));
    const __nv_bfloat16* rp = residual + row * ep.ld_res + n0;
    if (full) {
      const uint4* rq = reinterpret_cast<const uint4*>(rp);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 b = rq[q];
        const uint32_t w[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          v[q * 8 + 2 * t] += bf16_lo(w[t]);
          v[q * 8 + 2 * t + 1] += bf16_hi(w[t]);
        }
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) v[j] += __bfloat162float(rp[j]);
    }
  }
  if (ep.out_kind == kOutBF16) {
    __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(ep.out) + row * ep.ldo + n0;
    if (full) {
      uint4* oq = reinterpret_cast<uint4*>(op);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 o;
        o.x = pack_bf16(v[q * 8 + 0], v[q * 8 + 1]);
        o.y = pack_bf16(v[q * 8 + 2], v[q * 8 + 3]);
        o.z = pack_bf16(v[q * 8 + 4], v[q * 8 + 5]);
        o.w = pack_bf16(v[q * 8 + 6], v[q * 8 + 7]);
        oq[q] = o;
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) op[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* op = reinterpret_cast<float*>(ep.out) + row * ep.ldo + n0;
    const bool acc_mode = ep.out_kind == kOutF32Accumulate;
    if (full) {
      float4* oq = reinterpret_cast<float4*>(op);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 o = make_float4(v[q * 4], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]);
        if (acc_mode) {
          const float4 p = oq[q];
          o.x += p.x;
          o.y += p.y;
          o.z += p.z;
          o.w += p.w;
        }
        oq[q] = o;
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (n0 + j < N) op[j] = acc_mode ? op[j] + v[j] : v[j];
    }
  }
}

template <int BN, bool kAMN, bool kBMN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b, int M, int N, int K,
                        const GemmEpilogue ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = static_cast<int>(warp_id());
  const int num_m = (M + kBM - 1) / kBM;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + kBK - 1) / kBK;

  if (warp == 0 && elect_one()) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // ------------------------------------------------------------ TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile % num_m) * kBM;
        const int n0 = (tile / num_m) * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          uint8_t* a_dst = sA + stage * Cfg::kABytes;
          uint8_t* b_dst = sB + stage * Cfg::kBBytes;
          const int k0 = kb * kBK;
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
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
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
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int buf = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile % num_m) * kBM;
      const int n0 = (tile / num_m) * BN;
      mbar_wait(&tfull_bar[buf], acc_phase);
      tc_fence_after();
      const int64_t row = m0 + q * 32 + static_cast<int>(lane_id());
      const bool row_ok = row < M;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * BN + c * 32, r);
        tmem_ld_wait();
        const int col = n0 + c * 32;
        if (row_ok && col < N) epilogue_row32(ep, row, col, N, r);
      }
      tc_fence_before();
      mbar_arrive(&tempty_bar[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
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
                       const GemmEpilogue& ep, cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  CUtensorMap ma, mb;
  // A: K-major view [M][K] (inner K); MN-major view [K][M] (inner M)
  bool ok = kAMN ? make_map(&ma, a.ptr, M, K, a.ld, kBK) : make_map(&ma, a.ptr, K, M, a.ld, kBM);
  ok = ok && (kBMN ? make_map(&mb, b.ptr, N, K, b.ld, kBK) : make_map(&mb, b.ptr, K, N, b.ld, BN));
  if (!ok) return set_error(kErrCuda, "gemm: cuTensorMapEncodeTiled failed");
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tcgen05_kernel<BN, kAMN, kBMN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    attr_set = true;
  }
  const int tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  gemm_tcgen05_kernel<BN, kAMN, kBMN>
      <<<grid, kThreads, Cfg::kSmemBytes, stream>>>(ma, mb, M, N, K, ep);
  return check_launch("gemm_tcgen05_kernel");
}

// Picks the N tile that minimises the number of waves (ties -> larger tile).
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

int gemm_bf16(const GemmOperand& a, const GemmOperand& b, int M, int N, int K,
              const GemmEpilogue& ep, cudaStream_t stream, int force_bn) {
  if (M <= 0 || N <= 0 || K <= 0) return set_error(kErrConfig, "gemm: empty problem");
  // TMA: row strides must be 16-byte multiples; the epilogue's vector stores need ldo too.
  if ((a.ld % 8) != 0 || (b.ld % 8) != 0 || (ep.ldo % 8) != 0)
    return set_error(kErrConfig, "gemm: lda, ldb and ldo must be multiples of 8 elements");
  if (ep.drop_threshold != 0u && ((ep.drop_ld % 16) != 0 || (ep.col_offset % 16) != 0))
    return set_error(kErrConfig, "gemm: dropout row length / column offset must be multiples of 16");
  const int bn = force_bn > 0 ? force_bn : pick_bn(M, N);
#define GX_GEMM_DISPATCH(BN_)                                                           \
  if (bn == BN_) {                                                                      \
    if (!a.mn_major && !b.mn_major) return launch_gemm<BN_, false, false>(a, b, M, N, K, ep, stream); \
    if (!a.mn_major && b.mn_major) return launch_gemm<BN_, false, true>(a, b, M, N, K, ep, stream);   \
    if (a.mn_major && b.mn_major) return launch_gemm<BN_, true, true>(a, b, M, N, K, ep, stream);     \
    return launch_gemm<BN_, true, false>(a, b, M, N, K, ep, stream);                     \
  }
  GX_GEMM_DISPATCH(256)
  GX_GEMM_DISPATCH(128)
  GX_GEMM_DISPATCH(64)
#undef GX_GEMM_DISPATCH
  return set_error(kErrConfig, "gemm: unsupported N tile");
}

}  // namespace gx
