// Which pipe do MUFU.EX2 and F2FP.BF16.F32.PACK_AB share on sm_100a?  Each variant runs N
// independent chains per thread; the kernel time per warp-instruction tells the per-SM rate.
#include <cuda_bf16.h>
#include <cstdio>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned pack(float a, float b) { __nv_bfloat162 v = __floats2bfloat162_rn(a, b); return *(unsigned*)&v; }
template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8]; unsigned u[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i; u[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;                       // MUFU (+FADD)
      if (MODE == 1) u[i] += pack(a[i], __uint_as_float(u[i]));     // F2FP (+IADD)
      if (MODE == 2) { a[i] = ex2(a[i]) - 1.0f; u[i] += pack(a[i], __uint_as_float(u[i])); }
      if (MODE == 3) a[i] = fmaf(a[i], 1.0001f, 0.5f);              // FMA reference
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + u[i];
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* o; cudaMalloc(&o, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  const char* names[4] = {"ex2(+fadd)", "f2fp(+iadd)", "ex2+f2fp", "ffma"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(o, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(o, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(o, iters);
      if (mode == 3) k<3><<<blocks, threads>>>(o, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = (double)blocks * threads * iters * 8;   // per instruction kind
    double per_sm_clk = ops / sms / (ms * 1e-3 * clk * 1e3);
    printf("%-12s %.3f ms  %.1f lane-ops/clk/SM (of each kind, at the %d MHz rated clock)\n", names[mode], ms, per_sm_clk, clk / 1000);
  }
  return 0;
}
