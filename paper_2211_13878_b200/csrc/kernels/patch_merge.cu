// patch_merge.cu — Swin patch merging as a row permutation between window-major layouts.
//
// A window layer stores a sample's G x G token grid window-major: token (y, x) sits at row
//   ((y / ws) * (G / ws) + x / ws) * ws^2 + (y % ws) * ws + x % ws.
// Merging maps the 2G grid (c channels) to the G grid (4c channels): output token (y, x)
// concatenates the inputs (2y + dy, 2x + dx) for (dy, dx) = (0,0) (1,0) (0,1) (1,1) -- Swin's
// x0 x1 x2 x3 order.  Forward gathers, backward scatters the gradient back; both move every
// byte once (HBM-bound: 2 * rows_out * 4c * 2 B), one 16-byte chunk per thread, coalesced
// along channels.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gx_internal.h"
#include "launch.cuh"

namespace gx {

namespace {

__device__ __forceinline__ int64_t wm_row(int y, int x, int g, int ws) {
  return static_cast<int64_t>((y / ws) * (g / ws) + x / ws) * ws * ws + (y % ws) * ws + x % ws;
}

__global__ void patch_merge_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                   int64_t total, int seq_out, int grid_out, int ws, int cv,
                                   bool backward) {
  pdl_enter();
  const int win = ws * ws;
  const int wpr = grid_out / ws;  // windows per grid row (output)
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // i = ((row_out * 4 + q) * cv + v): chunk v of quadrant q of output row row_out
    const int v = static_cast<int>(i % cv);
    const int64_t rq = i / cv;
    const int q = static_cast<int>(rq & 3);
    const int64_t row_out = rq >> 2;
    const int64_t b = row_out / seq_out;
    const int t = static_cast<int>(row_out % seq_out);
    const int w = t / win, p = t % win;
    const int y = (w / wpr) * ws + p / ws, x = (w % wpr) * ws + p % ws;
    const int64_t row_in =
        b * 4 * seq_out + wm_row(2 * y + (q & 1), 2 * x + (q >> 1), 2 * grid_out, ws);
    const int64_t merged = (row_out * 4 + q) * cv + v;  // [row_out][4c] chunk
    const int64_t single = row_in * cv + v;             // [row_in][c] chunk
    if (backward) {
      dst[single] = src[merged];
    } else {
      dst[merged] = src[single];
    }
  }
}

__global__ void window_roll_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                   int64_t total, int seq, int grid, int ws, int shift, int cv,
                                   bool inverse) {
  pdl_enter();
  const int win = ws * ws, wpr = grid / ws;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int v = static_cast<int>(i % cv);
    const int64_t row = i / cv;
    const int64_t b = row / seq;
    const int t = static_cast<int>(row % seq);
    const int w = t / win, p = t % win;
    const int y = (w / wpr) * ws + p / ws, x = (w % wpr) * ws + p % ws;
    // output token (y, x) takes the input token shifted by +shift (roll by -shift) or by
    // -shift (the inverse roll)
    const int d = inverse ? grid - shift : shift;
    const int64_t src_row = b * seq + wm_row((y + d) % grid, (x + d) % grid, grid, ws);
    dst[i] = src[src_row * cv + v];
  }
}

}  // namespace

int window_roll(const void* src, void* dst, int samples, int grid, int ws, int shift, int c,
                bool inverse, cudaStream_t st) {
  if (c % 8 != 0 || ws <= 0 || grid % ws != 0 || shift <= 0 || shift >= ws)
    return set_error(kErrConfig, "window_roll: channels % 8, grid tiled by windows, 0 < shift < side");
  const int seq = grid * grid;
  const int cv = c / 8;
  const int64_t total = static_cast<int64_t>(samples) * seq * cv;
  if (total == 0) return kOk;
  int64_t blocks = (total + 255) / 256;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  launch_k(window_roll_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st,
           static_cast<const uint4*>(src), static_cast<uint4*>(dst), total, seq, grid, ws, shift,
           cv, inverse);
  return check_launch("window_roll_kernel");
}

int patch_merge(const void* src, void* dst, int samples, int grid_out, int ws, int c,
                bool backward, cudaStream_t st) {
  if (c % 8 != 0 || ws <= 0 || grid_out % ws != 0)
    return set_error(kErrConfig, "patch_merge: channels must be a multiple of 8, grid tiled by windows");
  const int seq_out = grid_out * grid_out;
  const int cv = c / 8;
  const int64_t total = static_cast<int64_t>(samples) * seq_out * 4 * cv;
  if (total == 0) return kOk;
  int64_t blocks = (total + 255) / 256;
  if (blocks > num_sms() * 8) blocks = num_sms() * 8;
  launch_k(patch_merge_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, st,
           static_cast<const uint4*>(src), static_cast<uint4*>(dst), total, seq_out, grid_out, ws,
           cv, backward);
  return check_launch("patch_merge_kernel");
}

}  // namespace gx
