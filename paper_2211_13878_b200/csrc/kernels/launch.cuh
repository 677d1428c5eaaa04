// launch.cuh — kernel launches with Programmatic Dependent Launch (PDL).
//
// Every executor kernel is launched with cudaLaunchAttributeProgrammaticStreamSerialization,
// and starts with pdl_enter(): griddepcontrol.wait (block until the previous kernel in the
// stream has completed and its writes are visible) followed by
// griddepcontrol.launch_dependents (let the next kernel's CTAs start their own prologue).
// Kernels with expensive prologues (the GEMMs: barrier init, TMEM allocation, tensor-map
// prefetch) do that work BEFORE pdl_enter, overlapping the predecessor's tail.  Inside a
// CUDA graph the programmatic edges are preserved, so back-to-back kernels of the step no
// longer pay a full launch gap each.  GX_PDL=0 disables it (plain stream ordering).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>

namespace gx {

__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GX_PDL");
    return e == nullptr || e[0] != '0';
  }();
  return on;
}

template <typename... Exp, typename... Act>
inline cudaError_t launch_k(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

// Same, with a thread-block cluster of `cluster_x` CTAs along x (grid.x must divide).
template <typename... Exp, typename... Act>
inline cudaError_t launch_k_cluster(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t st, unsigned cluster_x, Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

// Same, with a thread-block cluster of `cluster_y` CTAs along y (1: no cluster).
template <typename... Exp, typename... Act>
inline cudaError_t launch_k_cluster_y(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem,
                                      cudaStream_t st, unsigned cluster_y, Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster_y > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = 1;
    attr[n].val.clusterDim.y = cluster_y;
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
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

}  // namespace gx
