// Dropout keep-masks from an in-kernel Philox4x32-10 stream (minGPT's embd /
// attn / resid dropout, the paper's profiled dropout layer).  Reading DESIGN.md
// R38: element i of one site tensor of one micro-batch takes 16-bit half i % 2 (0 = low) of word
// (i / 2) % 4 of Philox4x32-10(counter = (i / 8, site, layer, micro_step), key = (seed lo, seed hi));
// it is kept iff that half >= thr = floor(p * 2^16), kept elements are scaled by 1 / (1 - p).
// thr == 0 (p = 0, or p < 2^-16) is the identity.  Every kernel that applies a mask (the standalone
// dropout, the embedding, LayerNorm's residual read, the attention kernels) regenerates it here.
#pragma once
#include <stdint.h>

namespace atom {

enum DropSite : uint32_t { DS_EMBD = 0, DS_ATTN = 1, DS_RESID_ATTN = 2, DS_RESID_MLP = 3 };

struct Drop {
  uint32_t thr = 0;       // floor(p * 2^16); 0 = no dropout
  float scale = 1.f;      // fp32(1 / (1 - p))
  uint32_t site = 0, layer = 0, step = 0;
  uint32_t k0 = 0, k1 = 0;   // seed lo, hi
};

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// keep bits of the 8 elements of group g (bit j = element 8 g + j kept)
__device__ __forceinline__ uint32_t drop_keep8(const Drop& d, uint32_t g) {
  const uint4 w = philox4x32_10(make_uint4(g, d.site, d.layer, d.step), d.k0, d.k1);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  uint32_t bits = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    bits |= ((ws[j] & 0xFFFFu) >= d.thr ? 1u : 0u) << (2 * j);
    bits |= ((ws[j] >> 16) >= d.thr ? 1u : 0u) << (2 * j + 1);
  }
  return bits;
}
// multiplier of element i (0 or scale; 1 without dropout)
__device__ __forceinline__ float drop_mult(const Drop& d, uint64_t i) {
  if (d.thr == 0) return 1.f;
  return (drop_keep8(d, (uint32_t)(i >> 3)) >> (i & 7)) & 1u ? d.scale : 0.f;
}

}  // namespace atom
