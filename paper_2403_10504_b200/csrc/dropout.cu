// Dropout site multiplier y = x * keep(i) / (1 - p) with an in-kernel Philox4x32-10 stream
// (minGPT's embd / attn / resid dropout, the paper's profiled dropout layer,
// PAPER.md P:184).  Reading DESIGN.md R38: element i of one site tensor takes word i % 4 of
// Philox4x32-10(counter = (i / 4, site, layer, micro_step), key = (seed lo, seed hi)); it is kept
// iff that word >= thr = floor(p * 2^32) (computed on the host in double).  The same call is the
// backward (dx = dy * the same multiplier).
//
// HBM-bound: one thread per Philox group (4 elements, one 16 B fp32 / 8 B bf16 vector), grid
// stride over a grid of 16 CTAs x 148 SMs; algorithmic bytes 2 x sizeof(T) per element.
#include "../../include/atom_kernels.h"
#include "common.cuh"
#include "kernels.h"

namespace atom {

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

template <typename T> struct Quad;
template <> struct Quad<float> {
  static __device__ __forceinline__ void load(const float* p, float v[4]) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
  static __device__ __forceinline__ void store(float* p, const float v[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  }
};
template <> struct Quad<bf16> {
  static __device__ __forceinline__ void load(const bf16* p, float v[4]) {
    const uint2 q = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q.y));
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  static __device__ __forceinline__ void store(bf16* p, const float v[4]) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 q;
    q.x = *reinterpret_cast<uint32_t*>(&a);
    q.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(p) = q;
  }
};

template <typename T>
__global__ void __launch_bounds__(256) dropout_kernel(const T* x, T* y, long n, uint32_t thr,
                                                      float scale, uint32_t site, uint32_t layer, uint32_t step,
                                                      uint32_t k0, uint32_t k1) {
  const long groups = (n + 3) >> 2;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < groups; g += (long)gridDim.x * blockDim.x) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)g, site, layer, step), k0, k1);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    const long i0 = g << 2;
    float v[4];
    if (i0 + 4 <= n) {
      Quad<T>::load(x + i0, v);
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = ws[j] >= thr ? v[j] * scale : 0.f;
      Quad<T>::store(y + i0, v);
    } else {
      for (long i = i0; i < n; ++i) {
        const float xv = to_f(x[i]);
        y[i] = from_f<T>(ws[i - i0] >= thr ? xv * scale : 0.f);
      }
    }
  }
}

template <typename T>
bool dropout(const T* x, T* y, long n, double p, uint64_t seed, uint32_t site, uint32_t layer, uint32_t step,
             cudaStream_t st) {
  if (n <= 0) return true;
  const uint32_t thr = (uint32_t)floor(p * 4294967296.0);
  const float scale = (float)(1.0 / (1.0 - p));
  const long groups = (n + 3) >> 2;
  long g = (groups + 255) / 256;
  const int grid = (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
  dropout_kernel<T><<<grid, 256, 0, st>>>(x, y, n, thr, scale, site, layer, step, (uint32_t)seed,
                                          (uint32_t)(seed >> 32));
  count_launch();
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

}  // namespace atom

using namespace atom;

extern "C" int atom_k_dropout(int dtype, const void* x, void* y, long n, double p, unsigned long long seed, int site,
                              int layer, int micro_step, void* stream) {
  if (!(p >= 0.0 && p < 1.0) || n < 0 || (n > 0 && (!x || !y)) || site < 0 || layer < 0 || micro_step < 0) {
    set_error("atom_k_dropout: invalid arguments (need 0 <= p < 1, n >= 0, non-null buffers)");
    return ATOM_E_INVALID;
  }
  if (n > (4l << 32)) {
    set_error("atom_k_dropout: n > 2^34 (the Philox group index is one 32-bit counter word)");
    return ATOM_E_INVALID;
  }
  const size_t align = dtype == ATOM_FP32 ? 16 : 8;
  if (((uintptr_t)x % align) || ((uintptr_t)y % align)) {
    set_error("atom_k_dropout: x and y must be %zu-byte aligned", align);
    return ATOM_E_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  bool ok;
  if (dtype == ATOM_FP32)
    ok = dropout<float>((const float*)x, (float*)y, n, p, seed, site, layer, micro_step, st);
  else if (dtype == ATOM_BF16)
    ok = dropout<bf16>((const bf16*)x, (bf16*)y, n, p, seed, site, layer, micro_step, st);
  else {
    set_error("atom_k_dropout: dtype must be ATOM_FP32 or ATOM_BF16");
    return ATOM_E_INVALID;
  }
  return ok ? ATOM_OK : ATOM_E_CUDA;
}
