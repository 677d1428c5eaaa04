// philox.cuh — counter-based Philox4x32-10, shared bit-for-bit by every dropout site on the
// GPU and by the CPU oracle (oracle/layer_oracle.py::philox4x32).  Dropout element `i` of a
// site uses counter {i>>2 (lo), i>>34 (hi), site_lo, site_hi}, key {seed_lo, seed_hi}, and
// word (i & 3) of the output; the element is kept iff word >= threshold (= p * 2^32).
#pragma once
#include <cstdint>

namespace gx {

struct Philox4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                                         uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return Philox4{c0, c1, c2, c3};
}

// Four consecutive dropout words for elements [4q, 4q+4) of site `site` under `seed`.
__host__ __device__ __forceinline__ Philox4 dropout_words(uint64_t seed, uint64_t site,
                                                         uint64_t q) {
  return philox4x32_10(static_cast<uint32_t>(q), static_cast<uint32_t>(q >> 32),
                       static_cast<uint32_t>(site), static_cast<uint32_t>(site >> 32),
                       static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

// 16 keep bits (bit j = byte j >= thr8) of call `c` of a site.
__host__ __device__ __forceinline__ uint32_t keep16(uint64_t seed, uint64_t site, uint64_t c,
                                                    uint32_t thr8) {
  const Philox4 w = philox4x32_10(static_cast<uint32_t>(c), static_cast<uint32_t>(c >> 32),
                                  static_cast<uint32_t>(site), static_cast<uint32_t>(site >> 32),
                                  static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#ifdef __CUDA_ARCH__
  // SIMD byte compares: 0xFF per byte >= thr8, then one bit per byte (positions 0,8,16,24
  // folded to 0..3) -- identical bits to the scalar loop below
  const uint32_t t4 = thr8 * 0x01010101u;
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t x = __vcmpgeu4(words[k], t4) & 0x01010101u;
    x |= x >> 7;
    x |= x >> 14;
    bits |= (x & 0xFu) << (4 * k);
  }
  return bits;
#else
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint32_t b = (words[j >> 2] >> (8 * (j & 3))) & 0xFFu;
    bits |= (b >= thr8 ? 1u : 0u) << j;
  }
  return bits;
#endif
}

// keep16 of the four consecutive calls c, c+1, c+2, c+3 (the 64 keys of one attention key
// block): the four Philox streams share their round keys, so the key schedule is paid once.
// Bit-identical to four keep16 calls.
__device__ __forceinline__ void keep16x4(uint64_t seed, uint64_t site, uint64_t c,
                                         uint32_t thr8, uint32_t (&out)[4]) {
  uint32_t x0[4], x1[4], x2[4], x3[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint64_t ct = c + static_cast<uint64_t>(t);
    x0[t] = static_cast<uint32_t>(ct);
    x1[t] = static_cast<uint32_t>(ct >> 32);
    x2[t] = static_cast<uint32_t>(site);
    x3[t] = static_cast<uint32_t>(site >> 32);
  }
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * x0[t];
      const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * x2[t];
      const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ x1[t] ^ k0;
      const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ x3[t] ^ k1;
      x1[t] = static_cast<uint32_t>(p1);
      x3[t] = static_cast<uint32_t>(p0);
      x0[t] = n0;
      x2[t] = n2;
    }
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const uint32_t t4 = thr8 * 0x01010101u;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t words[4] = {x0[t], x1[t], x2[t], x3[t]};
    uint32_t bits = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t x = __vcmpgeu4(words[k], t4) & 0x01010101u;
      x |= x >> 7;
      x |= x >> 14;
      bits |= (x & 0xFu) << (4 * k);
    }
    out[t] = bits;
  }
}

}  // namespace gx
