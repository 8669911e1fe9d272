// HBM-bound kernels of the GPT-3 training step (activation dtype T in {float, bf16}):
//   LayerNorm forward / re-apply / backward, column partial sums (bias, LN gain/shift grads),
//   cross-entropy forward+backward over the vocabulary, embedding gather and its
//   deterministic backward, GELU re-application, fused AdamW, casts, parameter init, loss sum.
// Every reduction has a fixed order (no floating-point atomics): swapped and resident runs are
// bit-identical (north star).
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"
#include "planner.h"

namespace atom {

constexpr float LN_EPS = 1e-5f;
constexpr int LN_THREADS = 128;
constexpr int LN_MAXE = 48;   // d <= 128 * 48 = 6144

// block-wide sum over LN_THREADS threads, fixed order
__device__ __forceinline__ float block_sum128(float v, float* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = sh[0] + sh[1] + sh[2] + sh[3];
  return t;
}

__device__ __forceinline__ float ln_out(float x, float mean, float rstd, float g, float b) {
  return __fmaf_rn(__fmul_rn(__fsub_rn(x, mean), rstd), g, b);
}

// 16-byte vectors of T (8 bf16 / 4 fp32); a row of d elements is d / VW chunks, chunk c of a row
// handled by thread c % 128 (coalesced), at most LN_MAXC chunks per thread kept in registers.
template <typename T> struct Vec { static constexpr int N = 16 / sizeof(T); };
constexpr int LN_MAXC = 6;   // 6 x 128 x 8 = 6144 bf16 (3072 fp32) elements per row

template <typename T>
__device__ __forceinline__ void load_vec(const T* p, float* f) {
  uint4 u = *(const uint4*)p;
  const T* e = (const T*)&u;
#pragma unroll
  for (int i = 0; i < Vec<T>::N; ++i) f[i] = to_f(e[i]);
}
template <typename T>
__device__ __forceinline__ void store_vec(T* p, const float* f) {
  uint4 u;
  T* e = (T*)&u;
#pragma unroll
  for (int i = 0; i < Vec<T>::N; ++i) e[i] = from_f<T>(f[i]);
  *(uint4*)p = u;
}

// y = LN(x) * g + b; stats[row] = (mean, rstd)                       (minGPT nn.LayerNorm)
// With res: x <- T(D(x) + res) first (written back; the residual add of the producing GEMM moved
// here; D = the residual-dropout mask of x's site, identity when drop.thr == 0)
template <typename T, int NC>
__global__ void __launch_bounds__(LN_THREADS) ln_fwd_kernel(const T* __restrict__ x, const T* __restrict__ g,
                                                            const T* __restrict__ b, T* __restrict__ y,
                                                            float* __restrict__ stats, int d,
                                                            const T* __restrict__ res, Drop drop) {
  constexpr int VW = Vec<T>::N;
  __shared__ float sh[4];
  const long row = blockIdx.x;
  const int nch = d / VW;
  const T* xr = x + row * d;
  float v[NC][VW];
  float s = 0.f;
  // every 16-byte load of the row in flight before any use (the in-place residual stores below
  // would otherwise keep the compiler from hoisting the next chunk's loads above them)
  uint4 xraw[NC], rraw[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = c * LN_THREADS + threadIdx.x;
    if (ch < nch) {
      xraw[c] = *(const uint4*)(xr + ch * VW);
      if (res) rraw[c] = *(const uint4*)(res + row * d + ch * VW);
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = c * LN_THREADS + threadIdx.x;
    if (ch < nch) {
      {
        const T* e = (const T*)&xraw[c];
#pragma unroll
        for (int i = 0; i < VW; ++i) v[c][i] = to_f(e[i]);
      }
      if (res) {
        float r[VW];
        const T* e = (const T*)&rraw[c];
#pragma unroll
        for (int i = 0; i < VW; ++i) r[i] = to_f(e[i]);
        if (drop.thr) {   // VW consecutive elements of the site tensor from one Philox group (VW <= 8)
          const uint64_t i0 = (uint64_t)row * d + (uint64_t)ch * VW;
          const uint32_t keep = drop_keep8(drop, (uint32_t)(i0 >> 3)) >> (i0 & 7);
#pragma unroll
          for (int i = 0; i < VW; ++i) v[c][i] = (keep >> i) & 1u ? v[c][i] * drop.scale : 0.f;
        }
#pragma unroll
        for (int i = 0; i < VW; ++i) v[c][i] = round_t<T>(v[c][i] + r[i]);
        store_vec<T>(const_cast<T*>(xr) + ch * VW, v[c]);
      }
#pragma unroll
      for (int i = 0; i < VW; ++i) s += v[c][i];
    }
  }
  const float mean = block_sum128(s, sh) / (float)d;
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c)
    if (c * LN_THREADS + threadIdx.x < nch)
#pragma unroll
      for (int i = 0; i < VW; ++i) {
        const float t = v[c][i] - mean;
        q = fmaf(t, t, q);
      }
  const float var = block_sum128(q, sh) / (float)d;
  const float rstd = rsqrtf(var + LN_EPS);
  T* yr = y + row * d;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = c * LN_THREADS + threadIdx.x;
    if (ch < nch) {
      float gg[VW], bb[VW], o[VW];
      load_vec<T>(g + ch * VW, gg);
      load_vec<T>(b + ch * VW, bb);
#pragma unroll
      for (int i = 0; i < VW; ++i) o[i] = ln_out(v[c][i], mean, rstd, gg[i], bb[i]);
      store_vec<T>(yr + ch * VW, o);
    }
  }
  if (threadIdx.x == 0) {
    stats[2 * row] = mean;
    stats[2 * row + 1] = rstd;
  }
}

// y = LN(x) from stored stats (bit-identical to the forward's y); one 16-byte chunk per thread
template <typename T>
__global__ void ln_apply_kernel(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b,
                                const float* __restrict__ stats, T* __restrict__ y, long rows, int d) {
  constexpr int VW = Vec<T>::N;
  const int nch = d / VW;
  const long n = rows * nch;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long r = i / nch;
    const int ch = (int)(i - r * nch);
    float xv[VW], gg[VW], bb[VW], o[VW];
    load_vec<T>(x + i * VW, xv);
    load_vec<T>(g + ch * VW, gg);
    load_vec<T>(b + ch * VW, bb);
    const float mean = stats[2 * r], rstd = stats[2 * r + 1];
#pragma unroll
    for (int k = 0; k < VW; ++k) o[k] = ln_out(xv[k], mean, rstd, gg[k], bb[k]);
    store_vec<T>(y + i * VW, o);
  }
}

// dx = dres + rstd * (dy*g - mean(dy*g) - xhat * mean(dy*g*xhat))
template <typename T, int NC>
__global__ void __launch_bounds__(LN_THREADS) ln_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ x,
                                                            const float* __restrict__ stats,
                                                            const T* __restrict__ g, const T* __restrict__ dres,
                                                            T* __restrict__ dx, int d) {
  constexpr int VW = Vec<T>::N;
  __shared__ float sh[4];
  const long row = blockIdx.x;
  const int nch = d / VW;
  const float mean = stats[2 * row], rstd = stats[2 * row + 1];
  float xh[NC][VW], dg[NC][VW];
  uint4 rraw[NC];   // the residual gradient, loaded with the rest (its latency off the second phase)
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = c * LN_THREADS + threadIdx.x;
    if (ch < nch && dres) rraw[c] = *(const uint4*)(dres + row * d + ch * VW);
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = c * LN_THREADS + threadIdx.x;
    if (ch < nch) {
      float gg[VW];
      load_vec<T>(x + row * d + ch * VW, xh[c]);
      load_vec<T>(dy + row * d + ch * VW, dg[c]);
      load_vec<T>(g + ch * VW, gg);
#pragma unroll
      for (int i = 0; i < VW; ++i) {
        xh[c][i] = (xh[c][i] - mean) * rstd;
        dg[c][i] *= gg[i];
        s1 += dg[c][i];
        s2 = fmaf(dg[c][i], xh[c][i], s2);
      }
    }
  }
  const float m1 = block_sum128(s1, sh) / (float)d;
  const float m2 = block_sum128(s2, sh) / (float)d;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = c * LN_THREADS + threadIdx.x;
    if (ch < nch) {
      float o[VW], r[VW];
      if (dres) {
        const T* e = (const T*)&rraw[c];
#pragma unroll
        for (int i = 0; i < VW; ++i) r[i] = to_f(e[i]);
      }
#pragma unroll
      for (int i = 0; i < VW; ++i) {
        o[i] = rstd * (dg[c][i] - m1 - xh[c][i] * m2);
        if (dres) o[i] += r[i];
      }
      store_vec<T>(dx + row * d + ch * VW, o);
    }
  }
}

// Column sums over rows in a fixed order (bias gradients, LN gain / shift gradients):
//   mode 0: out0[j] += sum_r a[r][j]
//   mode 1: out0[j] += sum_r a[r][j] * xhat[r][j],  out1[j] += sum_r a[r][j]
//   mode 2: a[r][j] <- T(a[r][j] * gelu'(x[r][j])) in place, out0[j] += sum_r of the stored values;
//           with gout, gout[r][j] <- T(GELU(x[r][j])) as well (same pitch as x)
// Grid (column blocks of 64 x VW columns) x (G row ranges), sized by the host to one wave of
// resident CTAs (CP_PER_SM per SM): a CTA's four thread groups sum contiguous quarters of its row range
// (UNR 16-byte loads in flight per thread), combined in group order into one partial per range.
// The last CTA of a column block to finish (atomic ticket; the ticket only picks who, never the
// order) adds the range partials in range order and resets the ticket: deterministic for a given
// (rows, columns, SM count).
constexpr int CP_GROUPS = 4, CP_TX = 64, CP_PER_SM = 3;
template <typename T, int MODE>
__global__ void __launch_bounds__(CP_TX * CP_GROUPS, CP_PER_SM) col_sums_kernel(const T* __restrict__ a, long lda,
                                                                        const T* __restrict__ x,
                                                                        const float* __restrict__ stats, long rows,
                                                                        int ncols, float* __restrict__ part0,
                                                                        float* __restrict__ part1,
                                                                        float* __restrict__ out0,
                                                                        float* __restrict__ out1,
                                                                        int* __restrict__ ticket,
                                                                        T* __restrict__ gout) {
  constexpr int VW = Vec<T>::N;
  constexpr int UNR = MODE == 0 ? 8 : 4;
  constexpr int NS = MODE == 1 ? 2 : 1;
  __shared__ float sh[CP_GROUPS][NS][CP_TX * VW];
  __shared__ int last;
  const int tx = threadIdx.x, g = threadIdx.y;
  const int j = (blockIdx.x * CP_TX + tx) * VW;
  const int c = blockIdx.y, nch = gridDim.y;
  float s0[VW], s1[VW];
#pragma unroll
  for (int i = 0; i < VW; ++i) s0[i] = s1[i] = 0.f;
  // this CTA's rows [c*R, (c+1)*R) in four contiguous group quarters
  const long R = (rows + nch - 1) / nch, Rg = (R + CP_GROUPS - 1) / CP_GROUPS;
  const long cr1 = min(rows, (long)(c + 1) * R);
  const long r0 = (long)c * R + g * Rg, r1 = min(cr1, r0 + Rg);
  if (j < ncols) {
    for (long rb = r0; rb < r1; rb += UNR) {
      // raw 16-byte loads first (all in flight), conversions after
      uint4 ra[UNR], rx[MODE != 0 ? UNR : 1];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const bool ok = rb + u < r1;
        ra[u] = ok ? *(const uint4*)(a + (rb + u) * lda + j) : make_uint4(0, 0, 0, 0);
        if constexpr (MODE != 0) rx[u] = ok ? *(const uint4*)(x + (rb + u) * ncols + j) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (rb + u < r1) {
          float v[VW];
          const T* ep = (const T*)&ra[u];
#pragma unroll
          for (int i = 0; i < VW; ++i) v[i] = to_f(ep[i]);
          if constexpr (MODE == 2) {
            const T* xp = (const T*)&rx[u];
            float o[VW];
#pragma unroll
            for (int i = 0; i < VW; ++i) {
              o[i] = round_t<T>(v[i] * gelu_grad_t<T>(to_f(xp[i])));
              s0[i] += o[i];
            }
            store_vec<T>(const_cast<T*>(a) + (rb + u) * lda + j, o);
            if (gout) {
              float gl[VW];
#pragma unroll
              for (int i = 0; i < VW; ++i) gl[i] = gelu_t<T>(to_f(xp[i]));
              store_vec<T>(gout + (rb + u) * ncols + j, gl);
            }
          } else if constexpr (MODE == 1) {
            const T* xp = (const T*)&rx[u];
            const float mean = stats[2 * (rb + u)], rstd = stats[2 * (rb + u) + 1];
#pragma unroll
            for (int i = 0; i < VW; ++i) {
              s0[i] = fmaf(v[i], (to_f(xp[i]) - mean) * rstd, s0[i]);
              s1[i] += v[i];
            }
          } else {
#pragma unroll
            for (int i = 0; i < VW; ++i) s0[i] += v[i];
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < VW; ++i) {
    sh[g][0][tx * VW + i] = s0[i];
    if constexpr (MODE == 1) sh[g][NS - 1][tx * VW + i] = s1[i];
  }
  __syncthreads();
  // combine the groups in group order: thread (tx, g) finishes columns tx * VW + e, e = g, g + CP_GROUPS, ...
  const long cb = (long)blockIdx.x * CP_TX * VW;
  for (int e = g; e < VW; e += CP_GROUPS) {
    const int col = tx * VW + e;
    if (cb + col < ncols) {
      float t0 = sh[0][0][col];
      for (int q = 1; q < CP_GROUPS; ++q) t0 += sh[q][0][col];
      part0[(long)c * ncols + cb + col] = t0;
      if constexpr (MODE == 1) {
        float t1 = sh[0][NS - 1][col];
        for (int q = 1; q < CP_GROUPS; ++q) t1 += sh[q][NS - 1][col];
        part1[(long)c * ncols + cb + col] = t1;
      }
    }
  }
  __threadfence();
  __syncthreads();
  if (tx == 0 && g == 0) last = atomicAdd(&ticket[blockIdx.x], 1) == nch - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // final reduction of this column block over the ranges: thread (tx, g) sums its VW columns over
  // ranges g, g + CP_GROUPS, ... (16-byte loads, several in flight), then the groups are added in
  // group order -- a fixed order, so the result is deterministic
  float q0[VW], q1[VW];
#pragma unroll
  for (int i = 0; i < VW; ++i) q0[i] = q1[i] = 0.f;
  if (j < ncols) {
#pragma unroll 4
    for (int q = g; q < nch; q += CP_GROUPS) {
#pragma unroll
      for (int i4 = 0; i4 < VW; i4 += 4) {
        const float4 a4 = __ldcg((const float4*)(part0 + (long)q * ncols + j + i4));
        q0[i4] += a4.x; q0[i4 + 1] += a4.y; q0[i4 + 2] += a4.z; q0[i4 + 3] += a4.w;
        if constexpr (MODE == 1) {
          const float4 b4 = __ldcg((const float4*)(part1 + (long)q * ncols + j + i4));
          q1[i4] += b4.x; q1[i4 + 1] += b4.y; q1[i4 + 2] += b4.z; q1[i4 + 3] += b4.w;
        }
      }
    }
  }
  __syncthreads();   // the group-combine reads of sh above are done
#pragma unroll
  for (int i = 0; i < VW; ++i) {
    sh[g][0][tx * VW + i] = q0[i];
    if constexpr (MODE == 1) sh[g][NS - 1][tx * VW + i] = q1[i];
  }
  __syncthreads();
  for (int e = g; e < VW; e += CP_GROUPS) {
    const int col = tx * VW + e;
    if (cb + col < ncols) {
      float t0 = sh[0][0][col];
      for (int q = 1; q < CP_GROUPS; ++q) t0 += sh[q][0][col];
      out0[cb + col] += t0;
      if constexpr (MODE == 1) {
        float t1 = sh[0][NS - 1][col];
        for (int q = 1; q < CP_GROUPS; ++q) t1 += sh[q][NS - 1][col];
        out1[cb + col] += t1;
      }
    }
  }
  if (tx == 0 && g == 0) ticket[blockIdx.x] = 0;
}

// Cross-entropy over one row of logits ("softmax" layer):
//   loss[row] = logsumexp(z) - z[y];  z <- (softmax(z) - onehot(y)) * scale   (in place)
template <typename T>
__global__ void __launch_bounds__(256) ce_kernel(T* __restrict__ logits, long ld, int V,
                                                 const int32_t* __restrict__ targets, long tstride, int T_,
                                                 float scale, float* __restrict__ loss) {
  __shared__ float sh[8];
  const long row = blockIdx.x;
  T* z = logits + row * ld;
  // pass 1: online max / sum-exp per thread
  float mx = -INFINITY, se = 0.f;
  for (int j = threadIdx.x; j < V; j += 256) {
    const float v = to_f(z[j]);
    if (v > mx) {
      se = se * __expf(mx - v) + 1.f;
      mx = v;
    } else {
      se += __expf(v - mx);
    }
  }
  // combine (fixed order): max first
  float m = warp_max(mx);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = m;
  __syncthreads();
  float gm = sh[0];
  for (int i = 1; i < 8; ++i) gm = fmaxf(gm, sh[i]);
  __syncthreads();
  float part = (mx == -INFINITY) ? 0.f : se * __expf(mx - gm);
  part = warp_sum(part);
  if (l == 0) sh[w] = part;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < 8; ++i) tot += sh[i];
  const float lse = gm + logf(tot);
  const long b = row / T_, t = row - b * T_;
  const int y = targets[b * tstride + t];
  const float zy = to_f(z[y]);
  __syncthreads();
  if (threadIdx.x == 0) loss[row] = lse - zy;
  const float inv = 1.f / tot;
  for (int j = threadIdx.x; j < V; j += 256) {
    float p = __expf(to_f(z[j]) - gm) * inv;
    if (j == y) p -= 1.f;
    z[j] = from_f<T>(p * scale);
  }
}

// bf16 cross-entropy, one HBM read and one write of the logits row: the row (V bf16, padded to
// 16 bytes) arrives in shared memory by one TMA bulk copy; three passes over shared memory (max,
// sum of exp, output) with 16-byte vectors; two CTAs per SM, so one CTA's copy overlaps the other's
// passes.  Same arithmetic as ce_kernel: fixed-order reductions (thread, warp, then warps in order).
constexpr int CE_THREADS = 256;
__device__ __forceinline__ float ce_block_reduce(float v, float* sh, bool is_max) {
  v = is_max ? warp_max(v) : warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = sh[0];
#pragma unroll
  for (int i = 1; i < CE_THREADS / 32; ++i) t = is_max ? fmaxf(t, sh[i]) : t + sh[i];
  return t;
}
__global__ void __launch_bounds__(CE_THREADS, 2) ce_bf16_kernel(bf16* __restrict__ logits, long ld, int V,
                                                                const int32_t* __restrict__ targets, long tstride,
                                                                int T_, float scale, float* __restrict__ loss) {
  extern __shared__ __align__(16) uint8_t ce_smem[];
  __shared__ float sh[CE_THREADS / 32];
  __shared__ __align__(8) uint64_t bar;
  const long row = blockIdx.x;
  bf16* z = logits + row * ld;
  const int nv = (V + 7) / 8;                       // 16-byte vectors (the last one partly padding)
  const uint32_t bytes = (uint32_t)nv * 16;
  const uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t sdst = (uint32_t)__cvta_generic_to_shared(ce_smem);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sdst),
                 "l"(z), "r"(bytes), "r"(sbar)
                 : "memory");
  }
  const long b = row / T_, t = row - b * T_;
  const int y = targets[b * tstride + t];
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done)
                   : "r"(sbar)
                   : "memory");
  }
  const uint4* sv = (const uint4*)ce_smem;
  auto vals = [&](int i, float* f) {
    const uint4 u = sv[i];
    const bf16* e = (const bf16*)&u;
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = (8 * i + k < V) ? __bfloat162float(e[k]) : -INFINITY;
  };
  float mx = -INFINITY;
  for (int i = threadIdx.x; i < nv; i += CE_THREADS) {
    float f[8];
    vals(i, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) mx = fmaxf(mx, f[k]);
  }
  const float gm = ce_block_reduce(mx, sh, true);
  float se = 0.f;
  for (int i = threadIdx.x; i < nv; i += CE_THREADS) {
    float f[8];
    vals(i, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) se += __expf(f[k] - gm);
  }
  const float tot = ce_block_reduce(se, sh, false);
  const float zy = __bfloat162float(((const bf16*)ce_smem)[y]);
  if (threadIdx.x == 0) loss[row] = gm + logf(tot) - zy;
  const float inv = 1.f / tot;
  for (int i = threadIdx.x; i < nv; i += CE_THREADS) {
    float f[8];
    vals(i, f);
    uint4 o;
    bf16* e = (bf16*)&o;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float p = __expf(f[k] - gm) * inv;
      if (8 * i + k == y) p -= 1.f;
      e[k] = __float2bfloat16_rn(p * scale);
    }
    if (8 * i + 8 <= V) {
      *(uint4*)(z + 8 * i) = o;
    } else {
      for (int k = 0; 8 * i + k < V; ++k) z[8 * i + k] = e[k];
    }
  }
}

// guarded averaging commit (R36): dst <- src only when the flag reduced over all ranks is 1
__global__ void commit_if_kernel(float* __restrict__ dst, const float* __restrict__ src, long n,
                                 const int* __restrict__ flag) {
  if (*flag != 1) return;
  const long n4 = n >> 2;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
  for (long i = (n4 << 2) + blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// h0[row] = wte[x] + wpe[t]   (P:295, P:307 embedding in sub-model 1)
template <typename T>
__global__ void embed_fwd_kernel(const int32_t* __restrict__ tok, long tstride, int T_, const T* __restrict__ wte,
                                 const T* __restrict__ wpe, T* __restrict__ h, int d) {
  const long row = blockIdx.x;
  const long b = row / T_, t = row - b * T_;
  const int id = tok[b * tstride + t];
  for (int j = threadIdx.x; j < d; j += blockDim.x)
    h[row * d + j] = from_f<T>(to_f(wte[(long)id * d + j]) + to_f(wpe[t * d + j]));
}

// dwpe[t] += sum_b dh[b, t]   (b ascending)
template <typename T>
__global__ void embed_bwd_pos_kernel(const T* __restrict__ dh, int B, int T_, int d, float* __restrict__ dwpe) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= (long)T_ * d) return;
  float s = 0.f;
  for (int b = 0; b < B; ++b) s += to_f(dh[(long)b * T_ * d + i]);
  dwpe[i] += s;
}

__global__ void tok_count_kernel(const int32_t* __restrict__ tok, long tstride, int T_, long M, int* __restrict__ cnt) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= M) return;
  const long b = i / T_, t = i - b * T_;
  atomicAdd(&cnt[tok[b * tstride + t]], 1);   // integer: order-independent
}

// exclusive scan of cnt[V] -> off[V+1] (one CTA of 1024 threads, fixed order)
__global__ void __launch_bounds__(1024) scan_kernel(const int* __restrict__ cnt, int V, int* __restrict__ off) {
  __shared__ int sh[1024];
  const int per = (V + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(V, lo + per);
  int s = 0;
  for (int i = lo; i < hi; ++i) s += cnt[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    int v = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += v;
    __syncthreads();
  }
  int base = threadIdx.x ? sh[threadIdx.x - 1] : 0;
  for (int i = lo; i < hi; ++i) {
    off[i] = base;
    base += cnt[i];
  }
  if (threadIdx.x == 1023) off[V] = sh[1023];
}

__global__ void tok_fill_kernel(const int32_t* __restrict__ tok, long tstride, int T_, long M,
                                const int* __restrict__ off, int* __restrict__ cur, int* __restrict__ perm) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= M) return;
  const long b = i / T_, t = i - b * T_;
  const int v = tok[b * tstride + t];
  perm[off[v] + atomicAdd(&cur[v], 1)] = (int)i;
}

// sort each bucket ascending (insertion sort; buckets are token positions of one vocab id)
__global__ void bucket_sort_kernel(const int* __restrict__ off, int V, int* __restrict__ perm) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int lo = off[v], hi = off[v + 1];
  for (int i = lo + 1; i < hi; ++i) {
    int key = perm[i], j = i - 1;
    while (j >= lo && perm[j] > key) {
      perm[j + 1] = perm[j];
      --j;
    }
    perm[j + 1] = key;
  }
}

// dwte[v] += sum over positions p with token v, ascending p, of dh[p]   (one warp per vocab row)
template <typename T>
__global__ void embed_bwd_tok_kernel(const T* __restrict__ dh, const int* __restrict__ off,
                                     const int* __restrict__ perm, int V, int d, float* __restrict__ dwte) {
  const int v = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (v >= V) return;
  const int lo = off[v], hi = off[v + 1];
  if (lo == hi) return;
  for (int j = lane; j < d; j += 32) {
    float s = 0.f;
    for (int p = lo; p < hi; ++p) s += to_f(dh[(long)perm[p] * d + j]);
    dwte[(long)v * d + j] += s;
  }
}

// n % VW == 0 (rows of 4d elements); 16-byte vectors
template <typename T>
__global__ void gelu_kernel(const T* __restrict__ u, T* __restrict__ g, long n) {
  constexpr int VW = Vec<T>::N;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n / VW; i += (long)gridDim.x * blockDim.x) {
    float v[VW];
    load_vec<T>(u + i * VW, v);
#pragma unroll
    for (int k = 0; k < VW; ++k) v[k] = gelu_t<T>(v[k]);
    store_vec<T>(g + i * VW, v);
  }
}

// Fused AdamW on a swapped-in segment (torch AdamW semantics, R19):
//   p <- p (1 - lr wd); m <- m + (1-b1)(g - m); v <- b2 v + (1-b2) g^2;
//   p <- p - (lr / bc1) m / (sqrt(v) / sqrt(bc2) + eps);  w <- T(p) (optional)
template <typename T>
__global__ void adamw_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, T* __restrict__ w, long n, AdamConsts c) {
  // every product and quotient rounded on its own (__fmul_rn / __fdiv_rn: no contraction), the
  // two explicit fmaf as written: cpu_adam.cpp applies the same operations in the same order
  const float omb1 = 1.f - c.b1, omb2 = 1.f - c.b2;
  auto upd = [&](float& pk, float gk, float& mk, float& vk) {
    gk = __fmul_rn(gk, c.gscale);
    const float pd = __fmul_rn(pk, c.decay);
    mk = fmaf(omb1, gk - mk, mk);
    vk = fmaf(c.b2, vk, __fmul_rn(__fmul_rn(omb2, gk), gk));
    const float den = __fadd_rn(__fdiv_rn(sqrtf(vk), c.sbc2), c.eps);
    pk = pd - __fdiv_rn(__fmul_rn(c.step, mk), den);
  };
  const long n4 = n / 4;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 pp = ((float4*)p)[i], gg = ((const float4*)g)[i], mm = ((float4*)m)[i], vv = ((float4*)v)[i];
    float* pa = &pp.x; const float* ga = &gg.x; float* ma = &mm.x; float* va = &vv.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) upd(pa[k], ga[k], ma[k], va[k]);
    ((float4*)p)[i] = pp; ((float4*)m)[i] = mm; ((float4*)v)[i] = vv;
    if (w) {
#pragma unroll
      for (int k = 0; k < 4; ++k) w[4 * i + k] = from_f<T>(pa[k]);
    }
  }
  for (long i = 4 * n4 + blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    float pk = p[i], mk = m[i], vk = v[i];
    upd(pk, g[i], mk, vk);
    p[i] = pk; m[i] = mk; v[i] = vk;
    if (w) w[i] = from_f<T>(pk);
  }
}

template <typename T>
__global__ void cast_kernel(const float* __restrict__ src, T* __restrict__ dst, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    dst[i] = from_f<T>(src[i]);
}

// minGPT init drawn on the device: normal(0, std) from a counter-based hash (splitmix64 +
// Box-Muller), constant `fill` when std == 0.
__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void init_normal_kernel(float* __restrict__ dst, long n, uint64_t seed, uint64_t base, float std,
                                   float fill) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    if (std == 0.f) {
      dst[i] = fill;
      continue;
    }
    const uint64_t r = splitmix(seed * 0x2545F4914F6CDD1Dull + base + (uint64_t)i);
    const float u1 = ((r >> 40) + 1) * (1.0f / 16777217.0f);
    const float u2 = ((r & 0xFFFFFF)) * (1.0f / 16777216.0f);
    dst[i] = std * sqrtf(-2.f * logf(u1)) * cospif(2.f * u2);
  }
}

// loss = sum(losses[0..n)) * scale, fixed order (one CTA)
__global__ void __launch_bounds__(1024) loss_sum_kernel(const float* __restrict__ l, long n, float scale,
                                                        float* __restrict__ out) {
  __shared__ float sh[32];
  float s = 0.f;
  for (long i = threadIdx.x; i < n; i += 1024) s += l[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < 32; ++i) t += sh[i];
    *out = t * scale;
  }
}

// ------------------------------------------------------------------ launchers
static inline int grid_for(long n, int threads = 256) {
  long g = (n + threads - 1) / threads;
  return (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

// row ranges of the column sums: one wave of resident CTAs (CP_PER_SM per SM) over the column blocks,
// at least 32 rows per range, and no more ranges than the partial buffer's ceil(rows / RED_ROWS)
static int cs_ranges(long rows, int col_blocks) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  long g = (long)sms * CP_PER_SM / (col_blocks > 0 ? col_blocks : 1);
  g = std::min(g, (rows + 31) / 32);
  g = std::min(g, (rows + RED_ROWS - 1) / RED_ROWS);
  return (int)std::max(1L, g);
}

#define LAUNCH_OK()                      \
  do {                                   \
    count_launch(__func__);              \
    ATOM_CUDA_OK(cudaGetLastError());    \
  } while (0)

template <typename T>
bool ln_fwd(const T* x, const T* g, const T* b, T* y, float* stats, long rows, int d, cudaStream_t st,
            const T* res, Drop drop) {
  if (d % Vec<T>::N || d > LN_THREADS * LN_MAXC * Vec<T>::N) {
    set_error("LayerNorm: d must be a multiple of %d and <= %d", Vec<T>::N, LN_THREADS * LN_MAXC * Vec<T>::N);
    return false;
  }
  switch ((d / Vec<T>::N + LN_THREADS - 1) / LN_THREADS) {   // chunks per thread (same order for any NC)
#define LN_FWD_CASE(NC) \
  case NC: ln_fwd_kernel<T, NC><<<rows, LN_THREADS, 0, st>>>(x, g, b, y, stats, d, res, drop); break;
    LN_FWD_CASE(1) LN_FWD_CASE(2) LN_FWD_CASE(3) LN_FWD_CASE(4) LN_FWD_CASE(5) LN_FWD_CASE(6)
#undef LN_FWD_CASE
  }
  LAUNCH_OK();
  return true;
}
template <typename T>
bool ln_apply(const T* x, const T* g, const T* b, const float* stats, T* y, long rows, int d, cudaStream_t st) {
  ln_apply_kernel<T><<<grid_for(rows * d / Vec<T>::N), 256, 0, st>>>(x, g, b, stats, y, rows, d);
  LAUNCH_OK();
  return true;
}
template <typename T>
bool ln_bwd(const T* dy, const T* x, const float* stats, const T* g, const T* dres, T* dx, float* dg, float* db,
            float* part, int* ticket, long rows, int d, cudaStream_t st) {
  if (d % Vec<T>::N || d > LN_THREADS * LN_MAXC * Vec<T>::N) {
    set_error("LayerNorm: d must be a multiple of %d and <= %d", Vec<T>::N, LN_THREADS * LN_MAXC * Vec<T>::N);
    return false;
  }
  switch ((d / Vec<T>::N + LN_THREADS - 1) / LN_THREADS) {
#define LN_BWD_CASE(NC) \
  case NC: ln_bwd_kernel<T, NC><<<rows, LN_THREADS, 0, st>>>(dy, x, stats, g, dres, dx, d); break;
    LN_BWD_CASE(1) LN_BWD_CASE(2) LN_BWD_CASE(3) LN_BWD_CASE(4) LN_BWD_CASE(5) LN_BWD_CASE(6)
#undef LN_BWD_CASE
  }
  LAUNCH_OK();
  constexpr int VW = Vec<T>::N;
  const int nb = (d / VW + CP_TX - 1) / CP_TX;
  if (nb > CS_TICKETS) {
    set_error("ln_bwd: %d columns exceed the column-sum ticket slots", d);
    return false;
  }
  const int nch = cs_ranges(rows, nb);
  col_sums_kernel<T, 1><<<dim3(nb, nch), dim3(CP_TX, CP_GROUPS), 0, st>>>(
      dy, d, x, stats, rows, d, part, part + (long)nch * d, dg, db, ticket, nullptr);
  LAUNCH_OK();
  return true;
}
// dy <- T(dy * gelu'(u)) in place (dy [rows, n] at pitch n, u likewise) and db += column sums of
// the result: the fc pre-activation gradient and its bias gradient in one pass
template <typename T>
bool dgelu_bias_grad(T* dy, const T* u, long rows, int n, float* db, float* part, int* ticket, cudaStream_t st,
                     T* gelu_out) {
  constexpr int VW = Vec<T>::N;
  const int nb = (n / VW + CP_TX - 1) / CP_TX;
  if (n % VW || nb > CS_TICKETS) {
    set_error("dgelu_bias_grad: %d columns (multiple of %d, at most %d blocks)", n, VW, CS_TICKETS);
    return false;
  }
  const int nch = cs_ranges(rows, nb);
  col_sums_kernel<T, 2><<<dim3(nb, nch), dim3(CP_TX, CP_GROUPS), 0, st>>>(
      dy, n, u, nullptr, rows, n, part, nullptr, db, nullptr, ticket, gelu_out);
  LAUNCH_OK();
  return true;
}
template <typename T>
bool bias_grad(const T* dy, long ld, long rows, int n, float* db, float* part, int* ticket, cudaStream_t st) {
  constexpr int VW = Vec<T>::N;
  if (n % VW || ld % VW) {
    set_error("bias_grad: columns and pitch must be multiples of %d", VW);
    return false;
  }
  const int nb = (n / VW + CP_TX - 1) / CP_TX;
  if (nb > CS_TICKETS) {
    set_error("bias_grad: %d columns exceed the column-sum ticket slots", n);
    return false;
  }
  const int nch = cs_ranges(rows, nb);
  col_sums_kernel<T, 0><<<dim3(nb, nch), dim3(CP_TX, CP_GROUPS), 0, st>>>(
      dy, ld, nullptr, nullptr, rows, n, part, nullptr, db, nullptr, ticket, nullptr);
  LAUNCH_OK();
  return true;
}
bool commit_if(float* dst, const float* src, long n, const int* flag, cudaStream_t st) {
  if (((uintptr_t)dst | (uintptr_t)src) & 15) {
    set_error("commit_if: 16-byte aligned buffers required");
    return false;
  }
  commit_if_kernel<<<grid_for(n / 4 + 1), 256, 0, st>>>(dst, src, n, flag);
  LAUNCH_OK();
  return true;
}

template <typename T>
bool cross_entropy(T* logits, long ld, int V, const int32_t* targets, long tstride, int T_, long rows, float scale,
                   float* loss, cudaStream_t st) {
  const size_t row_bytes = (size_t)(V + 7) / 8 * 16;
  if (std::is_same<T, bf16>::value && ld % 8 == 0 && ((uintptr_t)logits & 15) == 0 && row_bytes <= 112 * 1024) {
    static bool attr = false;
    if (!attr) {
      ATOM_CUDA_OK(cudaFuncSetAttribute(ce_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
      attr = true;
    }
    ce_bf16_kernel<<<rows, CE_THREADS, row_bytes, st>>>((bf16*)logits, ld, V, targets, tstride, T_, scale, loss);
  } else {
    ce_kernel<T><<<rows, 256, 0, st>>>(logits, ld, V, targets, tstride, T_, scale, loss);
  }
  LAUNCH_OK();
  return true;
}
template <typename T>
bool embed_fwd(const int32_t* tok, long tstride, int T_, long rows, const T* wte, const T* wpe, T* h, int d,
               cudaStream_t st) {
  embed_fwd_kernel<T><<<rows, 128, 0, st>>>(tok, tstride, T_, wte, wpe, h, d);
  LAUNCH_OK();
  return true;
}
template <typename T>
bool embed_bwd(const int32_t* tok, long tstride, int T_, int B, const T* dh, int V, int d, float* dwte, float* dwpe,
               int* scratch, cudaStream_t st) {
  const long M = (long)B * T_;
  int* cnt = scratch;
  int* off = cnt + V;
  int* cur = off + V + 1;
  int* perm = cur + V;
  ATOM_CUDA_OK(cudaMemsetAsync(cnt, 0, sizeof(int) * V, st));
  ATOM_CUDA_OK(cudaMemsetAsync(cur, 0, sizeof(int) * V, st));
  tok_count_kernel<<<(M + 255) / 256, 256, 0, st>>>(tok, tstride, T_, M, cnt);
  LAUNCH_OK();
  scan_kernel<<<1, 1024, 0, st>>>(cnt, V, off);
  LAUNCH_OK();
  tok_fill_kernel<<<(M + 255) / 256, 256, 0, st>>>(tok, tstride, T_, M, off, cur, perm);
  LAUNCH_OK();
  bucket_sort_kernel<<<(V + 255) / 256, 256, 0, st>>>(off, V, perm);
  LAUNCH_OK();
  embed_bwd_tok_kernel<T><<<(V + 7) / 8, 256, 0, st>>>(dh, off, perm, V, d, dwte);
  LAUNCH_OK();
  embed_bwd_pos_kernel<T><<<((long)T_ * d + 255) / 256, 256, 0, st>>>(dh, B, T_, d, dwpe);
  LAUNCH_OK();
  return true;
}
template <typename T>
bool gelu_apply(const T* u, T* g, long n, cudaStream_t st) {
  if (n % Vec<T>::N) {
    set_error("gelu: length must be a multiple of %d", Vec<T>::N);
    return false;
  }
  gelu_kernel<T><<<grid_for(n / Vec<T>::N), 256, 0, st>>>(u, g, n);
  LAUNCH_OK();
  return true;
}
template <typename T>
bool adamw(float* p, const float* g, float* m, float* v, T* w, long n, const AdamConsts& k, cudaStream_t st) {
  adamw_kernel<T><<<grid_for(n / 4 + 1), 256, 0, st>>>(p, g, m, v, w, n, k);
  LAUNCH_OK();
  return true;
}
template <typename T>
bool cast_params(const float* src, T* dst, long n, cudaStream_t st) {
  cast_kernel<T><<<grid_for(n), 256, 0, st>>>(src, dst, n);
  LAUNCH_OK();
  return true;
}
bool init_normal(float* dst, long n, uint64_t seed, uint64_t base, float std, float fill, cudaStream_t st) {
  init_normal_kernel<<<grid_for(n), 256, 0, st>>>(dst, n, seed, base, std, fill);
  LAUNCH_OK();
  return true;
}
bool loss_sum(const float* l, long n, float scale, float* out, cudaStream_t st) {
  loss_sum_kernel<<<1, 1024, 0, st>>>(l, n, scale, out);
  LAUNCH_OK();
  return true;
}

#define INST(T)                                                                                                 \
  template bool ln_fwd<T>(const T*, const T*, const T*, T*, float*, long, int, cudaStream_t, const T*, Drop);                   \
  template bool ln_apply<T>(const T*, const T*, const T*, const float*, T*, long, int, cudaStream_t);           \
  template bool ln_bwd<T>(const T*, const T*, const float*, const T*, const T*, T*, float*, float*, float*, int*, long, \
                          int, cudaStream_t);                                                                   \
  template bool bias_grad<T>(const T*, long, long, int, float*, float*, int*, cudaStream_t);                    \
  template bool dgelu_bias_grad<T>(T*, const T*, long, int, float*, float*, int*, cudaStream_t, T*);              \
  template bool cross_entropy<T>(T*, long, int, const int32_t*, long, int, long, float, float*, cudaStream_t);  \
  template bool embed_fwd<T>(const int32_t*, long, int, long, const T*, const T*, T*, int, cudaStream_t);       \
  template bool embed_bwd<T>(const int32_t*, long, int, int, const T*, int, int, float*, float*, int*,         \
                             cudaStream_t);                                                                     \
  template bool gelu_apply<T>(const T*, T*, long, cudaStream_t);                                                \
  template bool adamw<T>(float*, const float*, float*, float*, T*, long, const AdamConsts&, cudaStream_t);     \
  template bool cast_params<T>(const float*, T*, long, cudaStream_t);
INST(float)
INST(bf16)
#undef INST

}  // namespace atom
