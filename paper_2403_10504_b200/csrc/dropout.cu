// Dropout site multiplier y = x * keep(i) / (1 - p) with an in-kernel Philox4x32-10 stream
// (minGPT's embd / attn / resid dropout, the paper's profiled dropout layer,
// PAPER.md P:184).  Reading DESIGN.md R38: element i of one site tensor takes 16-bit half i % 2
// (0 = low) of word (i / 2) % 4 of Philox4x32-10(counter = (i / 8, site, layer, micro_step),
// key = (seed lo, seed hi)); it is kept iff that half >= thr = floor(p * 2^16) (host double).
// The same call is the backward (dx = dy * the same multiplier).
//
// HBM-bound: one thread per Philox group (8 elements: two 16 B fp32 vectors / one 16 B bf16
// vector), grid stride over 16 CTAs x 148 SMs; algorithmic bytes 2 x sizeof(T) per element.  With
// 32-bit draws (4 elements per Philox call) the bf16 kernel was ALU-bound at 3.3-3.8 TB/s
// (profiles/r01k_dropout.txt); 16-bit halves halve the Philox work per element.
#include "../../include/atom_kernels.h"
#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace atom {

template <typename T> struct Oct;
template <> struct Oct<float> {
  static __device__ __forceinline__ void load(const float* p, float v[8]) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float v[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};
template <> struct Oct<bf16> {
  static __device__ __forceinline__ void load(const bf16* p, float v[8]) {
    const uint4 q = *reinterpret_cast<const uint4*>(p);
    const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[j]));
      v[2 * j] = f.x;
      v[2 * j + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void store(bf16* p, const float v[8]) {
    uint32_t u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      u[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(u[0], u[1], u[2], u[3]);
  }
};

template <typename T>
__global__ void __launch_bounds__(256) dropout_kernel(const T* x, T* y, long n, uint32_t thr,
                                                      float scale, uint32_t site, uint32_t layer, uint32_t step,
                                                      uint32_t k0, uint32_t k1) {
  const long groups = (n + 7) >> 3;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < groups; g += (long)gridDim.x * blockDim.x) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)g, site, layer, step), k0, k1);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    uint32_t r[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      r[2 * j] = ws[j] & 0xFFFFu;
      r[2 * j + 1] = ws[j] >> 16;
    }
    const long i0 = g << 3;
    float v[8];
    if (i0 + 8 <= n) {
      Oct<T>::load(x + i0, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = r[j] >= thr ? v[j] * scale : 0.f;
      Oct<T>::store(y + i0, v);
    } else {
      for (long i = i0; i < n; ++i) {
        const float xv = to_f(x[i]);
        y[i] = from_f<T>(r[i - i0] >= thr ? xv * scale : 0.f);
      }
    }
  }
}

template <typename T>
bool dropout(const T* x, T* y, long n, double p, uint64_t seed, uint32_t site, uint32_t layer, uint32_t step,
             cudaStream_t st) {
  if (n <= 0) return true;
  const uint32_t thr = (uint32_t)floor(p * 65536.0);
  const float scale = (float)(1.0 / (1.0 - p));
  const long groups = (n + 7) >> 3;
  long g = (groups + 255) / 256;
  const int grid = (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
  dropout_kernel<T><<<grid, 256, 0, st>>>(x, y, n, thr, scale, site, layer, step, (uint32_t)seed,
                                          (uint32_t)(seed >> 32));
  count_launch();
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

// y <- T(D(y) + r): a residual branch's dropout and the residual add in one pass (the MLP
// projection's output when dropout is on: minGPT h = x2 + D(fc2(GELU(u))))
template <typename T>
__global__ void __launch_bounds__(256) dropout_add_kernel(T* y, const T* r, long n, Drop d) {
  const long groups = (n + 7) >> 3;
  for (long g = blockIdx.x * (long)blockDim.x + threadIdx.x; g < groups; g += (long)gridDim.x * blockDim.x) {
    const uint32_t keep = drop_keep8(d, (uint32_t)g);
    const long i0 = g << 3;
    float v[8], a[8];
    if (i0 + 8 <= n) {
      Oct<T>::load(y + i0, v);
      Oct<T>::load(r + i0, a);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = round_t<T>(((keep >> j) & 1u ? v[j] * d.scale : 0.f) + a[j]);
      Oct<T>::store(y + i0, v);
    } else {
      for (long i = i0; i < n; ++i)
        y[i] = from_f<T>(((keep >> (i - i0)) & 1u ? to_f(y[i]) * d.scale : 0.f) + to_f(r[i]));
    }
  }
}

template <typename T>
bool dropout_add(T* y, const T* r, long n, const Drop& d, cudaStream_t st) {
  if (n <= 0) return true;
  const long groups = (n + 7) >> 3;
  long g = (groups + 255) / 256;
  const int grid = (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
  dropout_add_kernel<T><<<grid, 256, 0, st>>>(y, r, n, d);
  count_launch("dropout_add");
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}
template bool dropout_add<float>(float*, const float*, long, const Drop&, cudaStream_t);
template bool dropout_add<bf16>(bf16*, const bf16*, long, const Drop&, cudaStream_t);

template <typename T>
bool dropout(const T* x, T* y, long n, const Drop& d, cudaStream_t st) {
  if (n <= 0 || d.thr == 0) {
    if (x != y && n > 0) ATOM_CUDA_OK(cudaMemcpyAsync(y, x, n * sizeof(T), cudaMemcpyDeviceToDevice, st));
    return true;
  }
  const long groups = (n + 7) >> 3;
  long g = (groups + 255) / 256;
  const int grid = (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
  dropout_kernel<T><<<grid, 256, 0, st>>>(x, y, n, d.thr, d.scale, d.site, d.layer, d.step, d.k0, d.k1);
  count_launch("dropout");
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}
template bool dropout<float>(const float*, float*, long, const Drop&, cudaStream_t);
template bool dropout<bf16>(const bf16*, bf16*, long, const Drop&, cudaStream_t);

}  // namespace atom

using namespace atom;

extern "C" int atom_k_dropout(int dtype, const void* x, void* y, long n, double p, unsigned long long seed, int site,
                              int layer, int micro_step, void* stream) {
  if (!(p >= 0.0 && p < 1.0) || n < 0 || (n > 0 && (!x || !y)) || site < 0 || layer < 0 || micro_step < 0) {
    set_error("atom_k_dropout: invalid arguments (need 0 <= p < 1, n >= 0, non-null buffers)");
    return ATOM_E_INVALID;
  }
  if (n > (8l << 32)) {
    set_error("atom_k_dropout: n > 2^35 (the Philox group index is one 32-bit counter word)");
    return ATOM_E_INVALID;
  }
  const size_t align = 16;
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
