// init_params.cu — deterministic synthetic initialisation of a rank's parameter shard on
// the device (no host traffic for multi-GB models).  Every value is a function of
// (seed, layer, canonical index) only, so any TP/SDP sharding of the same model holds
// bit-identical parameters: LayerNorm gains 1, biases and LayerNorm shifts 0, weights
// N(0, std^2) by Box-Muller over the Philox stream (patch-merging parameters included).
#include <cuda_runtime.h>

#include <cstdint>

#include "gx_internal.h"
#include "philox.cuh"

namespace gx {

__device__ int64_t canon_of(const InitLayout& L, int64_t j) {
  const int64_t h = L.h, f = L.f, ht = h / L.t, ft = f / L.t, tr = L.tr;
  const int64_t c_ln1g = 0, c_ln1b = h, c_ln2g = 2 * h, c_ln2b = 3 * h, c_bqkv = 4 * h,
                c_bo = 7 * h, c_b1 = 8 * h, c_b2 = 8 * h + f, c_wqkv = 9 * h + f,
                c_wo = c_wqkv + 3 * h * h, c_w1 = c_wo + h * h, c_w2 = c_w1 + f * h;
  const int64_t c_m = c_w2 + h * f;  // patch merging (mln_g, mln_b, w_m), unsharded
  int s = -1;
  for (int i = 0; i < kInitSlots; ++i)
    if (j >= L.off[i] && j < L.off[i] + L.n[i]) s = i;
  if (s < 0) return -1;
  const int64_t k = j - L.off[s];
  switch (s) {
    case 0: return c_ln1g + k;
    case 1: return c_ln1b + k;
    case 2: return c_ln2g + k;
    case 3: return c_ln2b + k;
    case 4: return c_bqkv + (k / ht) * h + tr * ht + k % ht;
    case 5: return c_bo + k;
    case 6: return c_b1 + tr * ft + k;
    case 7: return c_b2 + k;
    case 8: return c_wqkv + ((k / h) / ht * h + tr * ht + (k / h) % ht) * h + k % h;
    case 9: return c_wo + (k / ht) * h + tr * ht + k % ht;
    case 10: return c_w1 + (tr * ft + k / h) * h + k % h;
    case 11: return c_w2 + (k / ft) * f + tr * ft + k % ft;
    case 12: return c_m + k;
    case 13: return c_m + 2 * h + k;
    case 14: return c_m + 4 * h + k;
    // cross-attention (c_m is also its base: a layer merges or cross-attends, never both)
    case 15: return c_m + k;                                              // ln3_g
    case 16: return c_m + h + k;                                          // ln3_b
    case 17: return c_m + 2 * h + tr * ht + k;                            // b_q2
    case 18: return c_m + 3 * h + (k / ht) * h + tr * ht + k % ht;        // b_kv2
    case 19: return c_m + 5 * h + k;                                      // b_o2
    case 20: return c_m + 6 * h + (tr * ht + k / h) * h + k % h;          // w_q2
    case 21: return c_m + 6 * h + h * h + ((k / h) / ht * h + tr * ht + (k / h) % ht) * h + k % h;
    case 22: return c_m + 6 * h + 3 * h * h + (k / ht) * h + tr * ht + k % ht;  // w_o2
    // Swin relative-position bias, after w_2 (+ the merge block): this rank's heads contiguous
    case 23: return c_m + (L.extra == 1 ? 4 * h + 2 * h * h : 0) + tr * L.n[23] + k;
    // T5 relative attention bias, after w_2 (+ the cross block), this rank's heads contiguous
    default: return c_m + (L.extra == 2 ? 6 * h + 4 * h * h : 0) + tr * L.n[24] + k;
  }
}

__global__ void init_params_kernel(float* __restrict__ master, int64_t n, InitLayout L,
                                   uint64_t seed, uint64_t layer, float std_dev) {
  const int64_t h = L.h, f = L.f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = canon_of(L, L.lo + i);
    float v = 0.f;
    const int64_t c_m = 9 * h + f + 4 * h * h + 2 * h * f;  // first merge / cross element
    const int64_t gains = L.extra == 1 ? 2 * h : h;              // merge LN(2h) / LN3(h)
    const int64_t zeros = L.extra == 1 ? 4 * h : 6 * h;          // ... then shifts, biases
    if (c >= 0) {
      if (c < h || (c >= 2 * h && c < 3 * h) || (L.extra != 0 && c >= c_m && c < c_m + gains)) {
        v = 1.f;  // LayerNorm gains
      } else if (L.extra != 0 && c >= c_m && c < c_m + zeros) {
        v = 0.f;  // LayerNorm shifts and biases of the extra sublayer
      } else if (c >= 9 * h + f) {
        const Philox4 w = philox4x32_10(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32),
                                        static_cast<uint32_t>(layer), 0x5eedu,
                                        static_cast<uint32_t>(seed),
                                        static_cast<uint32_t>(seed >> 32));
        const float u1 = (static_cast<float>(w.x) + 1.f) * 2.3283064e-10f;
        const float u2 = static_cast<float>(w.y) * 2.3283064e-10f;
        v = std_dev * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
      }
    }
    master[i] = v;
  }
}

int init_params(float* master, int64_t n, const InitLayout& L, uint64_t seed, uint64_t layer,
                float std_dev, cudaStream_t st) {
  if (n <= 0) return kOk;
  int64_t blocks = (n + 255) / 256;
  if (blocks > num_sms() * 16) blocks = num_sms() * 16;
  init_params_kernel<<<static_cast<int>(blocks), 256, 0, st>>>(master, n, L, seed, layer, std_dev);
  return check_launch("init_params_kernel");
}

}  // namespace gx
