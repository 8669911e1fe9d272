// GEMM epilogues shared by the tcgen05 GEMM (bf16) and the SIMT GEMM (fp32 / bf16).
//
// D[m, n] = sum_k A[m, k] * B[n, k]  (fp32 accumulate), then one of:
//   EPI_STORE     out = T(D)
//   EPI_BIAS      out = T(D + bias[n])                          (QKV projection)
//   EPI_BIAS_RES  out = T(D + bias[n] + res[m, n])              (attn proj / MLP proj + residual)
//   EPI_BIAS_GELU u = T(D + bias[n]); out = u; out2 = T(gelu(u)) (MLP fc: stash pre-act u, GELU(u) feeds fc2)
//   EPI_DGELU     out = T(D * gelu'(aux[m, n]))                 (fc2 dgrad fused with GELU backward)
//   EPI_ACC_F32   outf[m, n] += D                               (weight gradient, fp32 accumulate)
// (minGPT block; GELU = tanh approximation.)
#pragma once
#include "common.cuh"

namespace atom {

enum EpiMode : int { EPI_STORE = 0, EPI_BIAS = 1, EPI_BIAS_RES = 2, EPI_BIAS_GELU = 3, EPI_DGELU = 4, EPI_ACC_F32 = 5 };

struct Epi {
  int mode = EPI_STORE;
  void* out = nullptr;        // T [M, ldo]   (float for EPI_ACC_F32)
  long ldo = 0;
  void* out2 = nullptr;       // T [M, ldo2]  (EPI_BIAS_GELU)
  long ldo2 = 0;
  const void* bias = nullptr; // T [N]
  const void* res = nullptr;  // T [M, ldr]
  long ldr = 0;
  const void* aux = nullptr;  // T [M, ldx]   (EPI_DGELU: u)
  long ldx = 0;
};

// scalar epilogue for one element
template <typename T>
__device__ __forceinline__ void epi_scalar(const Epi& e, long m, long n, float acc) {
  switch (e.mode) {
    case EPI_ACC_F32: {
      float* o = (float*)e.out + m * e.ldo + n;
      *o += acc;
      return;
    }
    case EPI_STORE:
      ((T*)e.out)[m * e.ldo + n] = from_f<T>(acc);
      return;
    case EPI_BIAS:
      ((T*)e.out)[m * e.ldo + n] = from_f<T>(acc + to_f(((const T*)e.bias)[n]));
      return;
    case EPI_BIAS_RES:
      ((T*)e.out)[m * e.ldo + n] =
          from_f<T>(acc + to_f(((const T*)e.bias)[n]) + to_f(((const T*)e.res)[m * e.ldr + n]));
      return;
    case EPI_BIAS_GELU: {
      T u = from_f<T>(acc + to_f(((const T*)e.bias)[n]));
      ((T*)e.out)[m * e.ldo + n] = u;
      ((T*)e.out2)[m * e.ldo2 + n] = from_f<T>(gelu_t<T>(to_f(u)));
      return;
    }
    case EPI_DGELU:
      ((T*)e.out)[m * e.ldo + n] = from_f<T>(acc * gelu_grad_t<T>(to_f(((const T*)e.aux)[m * e.ldx + n])));
      return;
  }
}

// 8 consecutive columns n..n+7 of row m (bf16 path; 16-byte vectors; caller guarantees n+8 <= N
// and 16-byte alignment of every row pointer involved).
__device__ __forceinline__ void epi_vec8_bf16(const Epi& e, long m, long n, const float* acc) {
  if (e.mode == EPI_ACC_F32) {
    float4* o = (float4*)((float*)e.out + m * e.ldo + n);
    float4 a = o[0], b = o[1];
    a.x += acc[0]; a.y += acc[1]; a.z += acc[2]; a.w += acc[3];
    b.x += acc[4]; b.y += acc[5]; b.z += acc[6]; b.w += acc[7];
    o[0] = a; o[1] = b;
    return;
  }
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = acc[i];
  if (e.mode == EPI_BIAS || e.mode == EPI_BIAS_RES || e.mode == EPI_BIAS_GELU) {
    uint4 bb = *(const uint4*)((const bf16*)e.bias + n);
    const bf16* bp = (const bf16*)&bb;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += __bfloat162float(bp[i]);
  }
  if (e.mode == EPI_BIAS_RES) {
    uint4 rr = *(const uint4*)((const bf16*)e.res + m * e.ldr + n);
    const bf16* rp = (const bf16*)&rr;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += __bfloat162float(rp[i]);
  }
  if (e.mode == EPI_DGELU) {
    uint4 xx = *(const uint4*)((const bf16*)e.aux + m * e.ldx + n);
    const bf16* xp = (const bf16*)&xx;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] *= gelu_grad_fast(__bfloat162float(xp[i]));
  }
  uint4 ov;
  bf16* op = (bf16*)&ov;
#pragma unroll
  for (int i = 0; i < 8; ++i) op[i] = __float2bfloat16_rn(v[i]);
  *(uint4*)((bf16*)e.out + m * e.ldo + n) = ov;
  if (e.mode == EPI_BIAS_GELU) {
    uint4 gv;
    bf16* gp = (bf16*)&gv;
#pragma unroll
    for (int i = 0; i < 8; ++i) gp[i] = __float2bfloat16_rn(gelu_fast(__bfloat162float(op[i])));
    *(uint4*)((bf16*)e.out2 + m * e.ldo2 + n) = gv;
  }
}

// Same as epi_vec8_bf16 for the bf16-output modes, with its operands already in hand: bias8 the
// 8 bias values (shared memory), x8 the 8 residual (EPI_BIAS_RES) or pre-activation (EPI_DGELU)
// values prefetched by the caller one chunk ahead (the per-chunk global-load latency was what
// bounded the K = 2560 GEMMs' epilogues).
__device__ __forceinline__ void epi_vec8_bf16_pre(const Epi& e, long m, long n, const float* acc, uint4 bias8,
                                                  uint4 x8) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = acc[i];
  if (e.mode == EPI_BIAS || e.mode == EPI_BIAS_RES || e.mode == EPI_BIAS_GELU) {
    const bf16* bp = (const bf16*)&bias8;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += __bfloat162float(bp[i]);
  }
  if (e.mode == EPI_BIAS_RES) {
    const bf16* rp = (const bf16*)&x8;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += __bfloat162float(rp[i]);
  }
  if (e.mode == EPI_DGELU) {
    const bf16* xp = (const bf16*)&x8;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] *= gelu_grad_fast(__bfloat162float(xp[i]));
  }
  uint4 ov;
  bf16* op = (bf16*)&ov;
#pragma unroll
  for (int i = 0; i < 8; ++i) op[i] = __float2bfloat16_rn(v[i]);
  *(uint4*)((bf16*)e.out + m * e.ldo + n) = ov;
  if (e.mode == EPI_BIAS_GELU) {
    uint4 gv;
    bf16* gp = (bf16*)&gv;
#pragma unroll
    for (int i = 0; i < 8; ++i) gp[i] = __float2bfloat16_rn(gelu_fast(__bfloat162float(op[i])));
    *(uint4*)((bf16*)e.out2 + m * e.ldo2 + n) = gv;
  }
}

// The store / bias / bias+GELU modes' 8 outputs packed, not stored (TMA-store epilogue):
// ov = T(acc [+ bias]); gv = T(gelu(ov)) for EPI_BIAS_GELU.
__device__ __forceinline__ void epi_pack8_bf16(int mode, const float* acc, uint4 bias8, uint4* ov, uint4* gv) {
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = acc[i];
  if (mode == EPI_BIAS || mode == EPI_BIAS_GELU) {
    const bf16* bp = (const bf16*)&bias8;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += __bfloat162float(bp[i]);
  }
  bf16* op = (bf16*)ov;
#pragma unroll
  for (int i = 0; i < 8; ++i) op[i] = __float2bfloat16_rn(v[i]);
  if (mode == EPI_BIAS_GELU) {
    bf16* gp = (bf16*)gv;
#pragma unroll
    for (int i = 0; i < 8; ++i) gp[i] = __float2bfloat16_rn(gelu_fast(__bfloat162float(op[i])));
  }
}

}  // namespace atom
