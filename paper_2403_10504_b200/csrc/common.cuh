// Shared device/host helpers for libatom's sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

namespace atom {

using bf16 = __nv_bfloat16;

// ---- element conversions (activation dtype T in {float, bf16}) ----
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(bf16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }
// round through T and back (what a store/load of T does to a value)
template <typename T> __device__ __forceinline__ float round_t(float x) { return to_f(from_f<T>(x)); }

// ---- GELU, tanh approximation (minGPT NewGELU) ----
constexpr float kGeluC = 0.7978845608028654f;   // sqrt(2/pi)
__device__ __forceinline__ float gelu_f(float u) {
  float th = tanhf(kGeluC * (u + 0.044715f * u * u * u));
  return 0.5f * u * (1.f + th);
}
__device__ __forceinline__ float gelu_grad_f(float u) {
  float th = tanhf(kGeluC * (u + 0.044715f * u * u * u));
  return 0.5f * (1.f + th) + 0.5f * u * (1.f - th * th) * kGeluC * (1.f + 3.f * 0.044715f * u * u);
}

// bf16 path: hardware tanh (MUFU.TANH, ~2^-11 relative error, far below bf16's 2^-8 rounding)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_fast(float u) {
  return 0.5f * u * (1.f + tanh_fast(kGeluC * (u + 0.044715f * u * u * u)));
}
__device__ __forceinline__ float gelu_grad_fast(float u) {
  const float th = tanh_fast(kGeluC * (u + 0.044715f * u * u * u));
  return 0.5f * (1.f + th) + 0.5f * u * (1.f - th * th) * kGeluC * (1.f + 3.f * 0.044715f * u * u);
}
// per activation dtype: exact for the fp32 parity path, hardware tanh for bf16
template <typename T> __device__ __forceinline__ float gelu_t(float u);
template <> __device__ __forceinline__ float gelu_t<float>(float u) { return gelu_f(u); }
template <> __device__ __forceinline__ float gelu_t<bf16>(float u) { return gelu_fast(u); }
template <typename T> __device__ __forceinline__ float gelu_grad_t(float u);
template <> __device__ __forceinline__ float gelu_grad_t<float>(float u) { return gelu_grad_f(u); }
template <> __device__ __forceinline__ float gelu_grad_t<bf16>(float u) { return gelu_grad_fast(u); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// kernel-launch accounting (how many of our kernels ran; bench "gpu_launches")
extern unsigned long long g_launch_count;
void count_launch_named(const char* name);
// name: the kernel family (and template width) for the launch log (atom_k_launch_log)
inline void count_launch(const char* name = "other") {
  ++g_launch_count;
  count_launch_named(name);
}

}  // namespace atom

#define ATOM_CUDA_OK(expr)                                                              \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess) {                                                            \
      ::atom::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorString(_e), __FILE__, \
                        __LINE__, #expr);                                               \
      return false;                                                                     \
    }                                                                                   \
  } while (0)

namespace atom {
void set_error(const char* fmt, ...);
}
