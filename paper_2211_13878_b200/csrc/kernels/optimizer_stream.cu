// optimizer_stream.cu — AdamW as one persistent kernel on a slice of the SMs, fed by per-layer
// "gradients ready" flags.
//
// At B = 1 the optimizer moves ~19 GB per step (30 B / parameter: fp32 master, m, v read and
// written, fp32 gradient read, bf16 copy written) while the backward is a chain of
// latency-bound kernels.  Launching one AdamW per layer beside that chain makes the two fight
// over every SM; instead this kernel is launched once per step with a fixed, small grid (one
// CTA per SM, ~108 KB of shared memory each, so it owns its SMs once resident) and walks the
// layers in backward order.  Before layer l it waits (acquire) until ready[l] carries the
// current step number -- written (release) by the stream that completes layer l's gradients --
// and then streams its slice of the layer through shared memory with 1-D TMA bulk copies:
// p, g, m, v in, p, m, v and the bf16 parameter out, three stages in flight.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "adam.cuh"
#include "gx_internal.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace gx {

namespace {

constexpr int kOptThreads = 256;
constexpr int kOptTile = 2048;                 // floats per array per tile (8 KB)
constexpr int kOptStages = 3;
constexpr int kOptStageBytes = 4 * kOptTile * 4 + kOptTile * 2;  // p g m v + bf16 out = 36 KB

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_opt() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read_opt() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all_opt() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ int64_t ld_acquire(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int64_t* p, int64_t v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

}  // namespace

__global__ void __launch_bounds__(kOptThreads, 1)
    adamw_persistent_kernel(const AdamSeg* __restrict__ tab, int count,
                            const int64_t* __restrict__ step, const int64_t* ready, float lr,
                            float b1, float b2, float eps, float wd) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bars[kOptStages];
  const uint32_t sb = smem_u32(smem);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kOptStages; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_enter();
  const int64_t t = *step;
  const AdamScalars c = adam_scalars_step(lr, b1, b2, eps, wd, step);
  uint32_t issued = 0, consumed = 0;  // tiles loaded / processed by this CTA (stage = n % S)
  for (int li = 0; li < count; ++li) {
    const AdamSeg L = tab[li];
    if (threadIdx.x == 0) {
      while (ld_acquire(ready + li) < t) __nanosleep(256);
    }
    __syncthreads();
    // this CTA's contiguous slice, in whole tiles except the layer's tail
    const int64_t ntiles = (L.n + kOptTile - 1) / kOptTile;
    const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t t0 = blockIdx.x * per;
    const int64_t t1 = ntiles < t0 + per ? ntiles : t0 + per;
    auto issue = [&](int64_t tile) {  // thread 0
      const uint32_t st = issued % kOptStages;
      const uint32_t base = sb + st * kOptStageBytes;
      const int64_t e0 = tile * kOptTile;
      const int64_t rem = L.n - e0;
      const uint32_t cnt = static_cast<uint32_t>(rem < kOptTile ? rem : kOptTile);
      // the stage's previous stores (the most recent group) must have read it before refill
      bulk_wait_read_opt<0>();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[st])),
                   "r"(cnt * 16u)
                   : "memory");
      bulk_g2s(base, static_cast<const float*>(L.p) + e0, cnt * 4, smem_u32(&bars[st]));
      bulk_g2s(base + kOptTile * 4, static_cast<const float*>(L.g) + e0, cnt * 4, smem_u32(&bars[st]));
      bulk_g2s(base + 2 * kOptTile * 4, static_cast<const float*>(L.m) + e0, cnt * 4, smem_u32(&bars[st]));
      bulk_g2s(base + 3 * kOptTile * 4, static_cast<const float*>(L.v) + e0, cnt * 4, smem_u32(&bars[st]));
      ++issued;
    };
    if (threadIdx.x == 0)
      for (int64_t k = t0; k < t1 && k < t0 + kOptStages - 1; ++k) issue(k);
    for (int64_t k = t0; k < t1; ++k) {
      if (threadIdx.x == 0 && k + kOptStages - 1 < t1) issue(k + kOptStages - 1);
      const uint32_t st = consumed % kOptStages;
      const uint32_t ph = (consumed / kOptStages) & 1;
      ++consumed;
      mbar_wait(&bars[st], ph);
      uint8_t* base = smem + st * kOptStageBytes;
      float* sp = reinterpret_cast<float*>(base);
      const float* sg = sp + kOptTile;
      float* sm = sp + 2 * kOptTile;
      float* sv = sp + 3 * kOptTile;
      uint2* so = reinterpret_cast<uint2*>(sp + 4 * kOptTile);
      const int64_t e0 = k * kOptTile;
      const int64_t rem = L.n - e0;
      const int cnt = static_cast<int>(rem < kOptTile ? rem : kOptTile);
      for (int i = threadIdx.x; i < cnt / 4; i += kOptThreads) {
        float4 p = reinterpret_cast<float4*>(sp)[i];
        const float4 g = reinterpret_cast<const float4*>(sg)[i];
        float4 m = reinterpret_cast<float4*>(sm)[i];
        float4 v = reinterpret_cast<float4*>(sv)[i];
        adam4(c, p, g, m, v);
        reinterpret_cast<float4*>(sp)[i] = p;
        reinterpret_cast<float4*>(sm)[i] = m;
        reinterpret_cast<float4*>(sv)[i] = v;
        so[i] = make_uint2(pack_bf16(p.x, p.y), pack_bf16(p.z, p.w));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t b = sb + st * kOptStageBytes;
        bulk_s2g(static_cast<float*>(L.p) + e0, b, cnt * 4);
        bulk_s2g(static_cast<float*>(L.m) + e0, b + 2 * kOptTile * 4, cnt * 4);
        bulk_s2g(static_cast<float*>(L.v) + e0, b + 3 * kOptTile * 4, cnt * 4);
        bulk_s2g(static_cast<__nv_bfloat16*>(L.out) + e0, b + 4 * kOptTile * 4, cnt * 2);
        bulk_commit_opt();
      }
    }
  }
  if (threadIdx.x == 0) bulk_wait_all_opt();
}

__global__ void mark_ready_kernel(int64_t* ready, const int64_t* step) {
  pdl_enter();
  __threadfence();
  st_release(ready, *step);
}

int adamw_persistent(const AdamSeg* table_dev, int count, const int64_t* step,
                     const int64_t* ready, float lr, float beta1, float beta2, float eps, float wd,
                     int ctas, cudaStream_t st) {
  if (count <= 0) return kOk;
  const int smem = kOptStages * kOptStageBytes + 1024;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(adamw_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    set = true;
  }
  launch_k(adamw_persistent_kernel, dim3(ctas), dim3(kOptThreads), smem, st, table_dev, count,
           step, ready, lr, beta1, beta2, eps, wd);
  return check_launch("adamw_persistent_kernel");
}

int mark_ready(int64_t* ready, const int64_t* step, cudaStream_t st) {
  launch_k(mark_ready_kernel, dim3(1), dim3(1), 0, st, ready, step);
  return check_launch("mark_ready_kernel");
}

}  // namespace gx
