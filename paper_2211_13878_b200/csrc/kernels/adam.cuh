// adam.cuh — the AdamW update shared by the standalone optimizer kernel (norm_elementwise.cu)
// and the weight-gradient GEMM epilogue that consumes its accumulator in place (gemm.cu).
//   p <- p - lr * (m_hat / (sqrt(v_hat) + eps) + wd * p)
// restated with the bias corrections folded into two per-launch scalars (step_size = lr/bc1,
// 1/sqrt(bc2)), so the per-element work is FMAs, one sqrt and one fast divide.
#pragma once
#include <cuda_runtime.h>

namespace gx {

struct AdamScalars {
  float b1, b2, eps, step_size, inv_sqrt_bc2, lr_wd;
};
__device__ __forceinline__ AdamScalars adam_scalars(float lr, float b1, float b2, float eps,
                                                    float wd, float bc1, float bc2) {
  return AdamScalars{b1, b2, eps, lr / bc1, rsqrtf(bc2), lr * wd};
}
// scalars for device step counter t (t >= 1)
__device__ __forceinline__ AdamScalars adam_scalars_step(float lr, float b1, float b2, float eps,
                                                         float wd, const int64_t* step) {
  const float t = static_cast<float>(*step);
  return adam_scalars(lr, b1, b2, eps, wd, 1.f - powf(b1, t), 1.f - powf(b2, t));
}
__device__ __forceinline__ void adam1(const AdamScalars& c, float& p, float g, float& m, float& v) {
  m = c.b1 * m + (1.f - c.b1) * g;
  v = c.b2 * v + (1.f - c.b2) * g * g;
  const float denom = sqrtf(v) * c.inv_sqrt_bc2 + c.eps;
  p = p - c.step_size * __fdividef(m, denom) - c.lr_wd * p;
}
__device__ __forceinline__ void adam4(const AdamScalars& c, float4& p, const float4& g, float4& m,
                                      float4& v) {
  adam1(c, p.x, g.x, m.x, v.x);
  adam1(c, p.y, g.y, m.y, v.y);
  adam1(c, p.z, g.z, m.z, v.z);
  adam1(c, p.w, g.w, m.w, v.w);
}

}  // namespace gx
