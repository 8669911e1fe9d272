// Causal multi-head attention on CUDA cores (one warp per query / key row, online softmax),
// for the fp32 parity path (dtype T = float) and as a reference-quality fallback for head sizes
// the tensor-core kernel does not cover.  minGPT CausalSelfAttention:
//   S_ts = q_t . k_s / sqrt(dh) (s <= t); o_t = sum_s softmax_s(S)_ts v_s; lse_t = log sum_s exp(S_ts)
// Backward (exact, deterministic, no atomics):
//   D_t = do_t . o_t;  P_ts = exp(S_ts - lse_t);  dS_ts = P_ts (do_t . v_s - D_t)
//   dq_t = sum_{s<=t} dS_ts k_s / sqrt(dh);  dk_s = sum_{t>=s} dS_ts q_t / sqrt(dh);  dv_s = sum_{t>=s} P_ts do_t
// With attention dropout (multiplier m_ts of element ((b h + head) T + t) T + s, R38):
//   o_t = sum_s m_ts P_ts v_s / l;  dS_ts = P_ts (m_ts do_t . v_s - D_t);  dv_s = sum_t m_ts P_ts do_t
#include "common.cuh"
#include "kernels.h"

namespace atom {

constexpr int AMAX = 4;   // dh <= 128

template <typename T>
__device__ __forceinline__ void load_row(const T* p, int dh, float* r) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < AMAX; ++i) {
    int j = lane + 32 * i;
    r[i] = j < dh ? to_f(p[j]) : 0.f;
  }
}
__device__ __forceinline__ float dotw(const float* a, const float* b) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < AMAX; ++i) s = fmaf(a[i], b[i], s);
  return warp_sum(s);
}

template <typename T>
__global__ void attn_fwd_simt_kernel(const T* __restrict__ qkv, T* __restrict__ o, float* __restrict__ lse, int B,
                                     int T_, int h, int dh, Drop drop) {
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  if (gw >= (long)B * h * T_) return;
  const int t = (int)(gw % T_);
  const int hh = (int)((gw / T_) % h);
  const int b = (int)(gw / ((long)T_ * h));
  const int d = h * dh;
  const long ld = 3L * d;
  const T* base = qkv + (long)b * T_ * ld;
  const float sc = rsqrtf((float)dh);
  float q[AMAX], k[AMAX], v[AMAX], acc[AMAX];
  load_row(base + (long)t * ld + hh * dh, dh, q);
#pragma unroll
  for (int i = 0; i < AMAX; ++i) acc[i] = 0.f;
  float m = -INFINITY, l = 0.f;
  for (int s = 0; s <= t; ++s) {
    load_row(base + (long)s * ld + d + hh * dh, dh, k);
    const float sco = dotw(q, k) * sc;
    load_row(base + (long)s * ld + 2 * d + hh * dh, dh, v);
    const float mn = fmaxf(m, sco);
    const float corr = __expf(m - mn);
    const float p = __expf(sco - mn);
    l = l * corr + p;
    const float pm = p * drop_mult(drop, (((uint64_t)b * h + hh) * T_ + t) * (uint64_t)T_ + s);
#pragma unroll
    for (int i = 0; i < AMAX; ++i) acc[i] = fmaf(pm, v[i], acc[i] * corr);
    m = mn;
  }
  const int lane = threadIdx.x & 31;
  T* orow = o + ((long)b * T_ + t) * d + hh * dh;
#pragma unroll
  for (int i = 0; i < AMAX; ++i) {
    int j = lane + 32 * i;
    if (j < dh) orow[j] = from_f<T>(acc[i] / l);
  }
  if (lane == 0) lse[((long)b * h + hh) * T_ + t] = m + logf(l);
}

template <typename T>
__global__ void attn_dsum_kernel(const T* __restrict__ o, const T* __restrict__ dout, float* __restrict__ Dsum, int B,
                                 int T_, int h, int dh) {
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  if (gw >= (long)B * h * T_) return;
  const int t = (int)(gw % T_);
  const int hh = (int)((gw / T_) % h);
  const int b = (int)(gw / ((long)T_ * h));
  const long off = ((long)b * T_ + t) * h * dh + hh * dh;
  float a[AMAX], c[AMAX];
  load_row(o + off, dh, a);
  load_row(dout + off, dh, c);
  const float s = dotw(a, c);
  if ((threadIdx.x & 31) == 0) Dsum[((long)b * h + hh) * T_ + t] = s;
}

template <typename T>
__global__ void attn_dq_simt_kernel(const T* __restrict__ qkv, const T* __restrict__ dout,
                                    const float* __restrict__ lse, const float* __restrict__ Dsum,
                                    T* __restrict__ dqkv, int B, int T_, int h, int dh, Drop drop) {
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  if (gw >= (long)B * h * T_) return;
  const int t = (int)(gw % T_);
  const int hh = (int)((gw / T_) % h);
  const int b = (int)(gw / ((long)T_ * h));
  const int d = h * dh;
  const long ld = 3L * d;
  const T* base = qkv + (long)b * T_ * ld;
  const float sc = rsqrtf((float)dh);
  float q[AMAX], k[AMAX], v[AMAX], dq[AMAX], g[AMAX];
  load_row(base + (long)t * ld + hh * dh, dh, q);
  load_row(dout + ((long)b * T_ + t) * d + hh * dh, dh, g);
  const float L = lse[((long)b * h + hh) * T_ + t];
  const float Dt = Dsum[((long)b * h + hh) * T_ + t];
#pragma unroll
  for (int i = 0; i < AMAX; ++i) dq[i] = 0.f;
  for (int s = 0; s <= t; ++s) {
    load_row(base + (long)s * ld + d + hh * dh, dh, k);
    load_row(base + (long)s * ld + 2 * d + hh * dh, dh, v);
    const float p = __expf(dotw(q, k) * sc - L);
    const float m = drop_mult(drop, (((uint64_t)b * h + hh) * T_ + t) * (uint64_t)T_ + s);
    const float ds = p * (m * dotw(g, v) - Dt);
#pragma unroll
    for (int i = 0; i < AMAX; ++i) dq[i] = fmaf(ds, k[i], dq[i]);
  }
  const int lane = threadIdx.x & 31;
  T* row = dqkv + ((long)b * T_ + t) * ld + hh * dh;
#pragma unroll
  for (int i = 0; i < AMAX; ++i) {
    int j = lane + 32 * i;
    if (j < dh) row[j] = from_f<T>(dq[i] * sc);
  }
}

template <typename T>
__global__ void attn_dkv_simt_kernel(const T* __restrict__ qkv, const T* __restrict__ dout,
                                     const float* __restrict__ lse, const float* __restrict__ Dsum,
                                     T* __restrict__ dqkv, int B, int T_, int h, int dh, Drop drop) {
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  if (gw >= (long)B * h * T_) return;
  const int s = (int)(gw % T_);
  const int hh = (int)((gw / T_) % h);
  const int b = (int)(gw / ((long)T_ * h));
  const int d = h * dh;
  const long ld = 3L * d;
  const T* base = qkv + (long)b * T_ * ld;
  const float sc = rsqrtf((float)dh);
  float q[AMAX], k[AMAX], v[AMAX], dk[AMAX], dv[AMAX], g[AMAX];
  load_row(base + (long)s * ld + d + hh * dh, dh, k);
  load_row(base + (long)s * ld + 2 * d + hh * dh, dh, v);
#pragma unroll
  for (int i = 0; i < AMAX; ++i) dk[i] = dv[i] = 0.f;
  for (int t = s; t < T_; ++t) {
    load_row(base + (long)t * ld + hh * dh, dh, q);
    load_row(dout + ((long)b * T_ + t) * d + hh * dh, dh, g);
    const float L = lse[((long)b * h + hh) * T_ + t];
    const float Dt = Dsum[((long)b * h + hh) * T_ + t];
    const float p = __expf(dotw(q, k) * sc - L);
    const float m = drop_mult(drop, (((uint64_t)b * h + hh) * T_ + t) * (uint64_t)T_ + s);
    const float ds = p * (m * dotw(g, v) - Dt);
#pragma unroll
    for (int i = 0; i < AMAX; ++i) {
      dv[i] = fmaf(p * m, g[i], dv[i]);
      dk[i] = fmaf(ds, q[i], dk[i]);
    }
  }
  const int lane = threadIdx.x & 31;
  T* row = dqkv + ((long)b * T_ + s) * ld;
#pragma unroll
  for (int i = 0; i < AMAX; ++i) {
    int j = lane + 32 * i;
    if (j < dh) {
      row[d + hh * dh + j] = from_f<T>(dk[i] * sc);
      row[2 * d + hh * dh + j] = from_f<T>(dv[i]);
    }
  }
}

template <typename T>
bool attn_fwd_simt(const T* qkv, T* o, float* lse, int B, int T_, int h, int dh, cudaStream_t st, Drop drop) {
  if (dh > 32 * AMAX) { set_error("attention: head size %d > %d", dh, 32 * AMAX); return false; }
  const long warps = (long)B * h * T_;
  attn_fwd_simt_kernel<T><<<(warps + 7) / 8, 256, 0, st>>>(qkv, o, lse, B, T_, h, dh, drop);
  count_launch();
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

template <typename T>
bool attn_bwd_simt(const T* qkv, const T* o, const T* dout, const float* lse, float* Dsum, T* dqkv, int B, int T_,
                   int h, int dh, cudaStream_t st, Drop drop) {
  if (dh > 32 * AMAX) { set_error("attention: head size %d > %d", dh, 32 * AMAX); return false; }
  const long warps = (long)B * h * T_;
  const int grid = (int)((warps + 7) / 8);
  attn_dsum_kernel<T><<<grid, 256, 0, st>>>(o, dout, Dsum, B, T_, h, dh);
  count_launch();
  attn_dq_simt_kernel<T><<<grid, 256, 0, st>>>(qkv, dout, lse, Dsum, dqkv, B, T_, h, dh, drop);
  count_launch();
  attn_dkv_simt_kernel<T><<<grid, 256, 0, st>>>(qkv, dout, lse, Dsum, dqkv, B, T_, h, dh, drop);
  count_launch();
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

template bool attn_fwd_simt<float>(const float*, float*, float*, int, int, int, int, cudaStream_t, Drop);
template bool attn_fwd_simt<bf16>(const bf16*, bf16*, float*, int, int, int, int, cudaStream_t, Drop);
template bool attn_bwd_simt<float>(const float*, const float*, const float*, const float*, float*, float*, int, int,
                                   int, int, cudaStream_t, Drop);
template bool attn_bwd_simt<bf16>(const bf16*, const bf16*, const bf16*, const float*, float*, bf16*, int, int, int,
                                  int, cudaStream_t, Drop);

}  // namespace atom
