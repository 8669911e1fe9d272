// Fused causal attention on tensor cores (bf16 in, fp32 accumulate), flash-attention style:
// scores never leave the SM (PAPER.md P:184 names the materialised T x T "dropout"/"softmax"
// tensors as GPT-3's peak-memory layers; here they are never materialised).
//   forward : per (b, h, 64-query block): S = Q K^T in registers, online softmax, O += P V; LSE
//   backward: deterministic, two passes without atomics:
//     dK/dV kernel per 64-key block (loops over query blocks >= it),
//     dQ kernel per 64-query block (loops over key blocks <= it)
// mma.sync.m16n8k16 bf16 (legacy tensor-core path; the tcgen05 version is the next step, see
// DESIGN.md §6).  qkv rows are tokens (b, t): [q | k | v], head j at columns j*dh .. j*dh+dh-1.
#include "common.cuh"
#include "kernels.h"

namespace atom {

namespace fa {

constexpr int BR = 64;   // queries per CTA (4 warps x 16)
constexpr int BC = 64;   // keys per iteration
constexpr int NT = 128;  // threads
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void ldsm_x4(uint32_t* r, const void* p) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t* r, const void* p) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *(uint32_t*)&v;
}

// Load a [64][DH] tile of rows r0.. (row stride ld elements) into smem [64][DH+8]; rows >= nrows -> 0.
template <int DH>
__device__ __forceinline__ void load_tile(bf16* sm, const bf16* g, long ld, int r0, int nrows) {
  constexpr int CH = DH / 8;  // 16-byte chunks per row
  for (int i = threadIdx.x; i < 64 * CH; i += NT) {
    const int r = i / CH, c = i % CH;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r0 + r < nrows) v = *(const uint4*)(g + (long)(r0 + r) * ld + c * 8);
    *(uint4*)(sm + r * (DH + 8) + c * 8) = v;
  }
}

// A fragments of a warp's 16 rows x DH from smem (row-major, stride DH+8)
template <int DH>
__device__ __forceinline__ void load_afrag(uint32_t (*a)[4], const bf16* sm, int row0) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) {
    // matrices: (rows 0-7, k 0-7), (rows 8-15, k 0-7), (rows 0-7, k 8-15), (rows 8-15, k 8-15)
    const int r = row0 + (lane & 7) + ((lane >> 3) & 1) * 8;
    const int c = kk * 16 + (lane >> 4) * 8;
    ldsm_x4(a[kk], sm + r * (DH + 8) + c);
  }
}

// acc[16 x 64] += A(16 x DH) * B^T where B rows are 64 "columns" stored [64][DH+8] (non-trans)
template <int DH>
__device__ __forceinline__ void mm_abt(float (*acc)[4], const uint32_t (*a)[4], const bf16* smB) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int nn = 0; nn < 8; nn += 2) {
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
      uint32_t b[4];
      // matrices: (n 0-7, k 0-7), (n 0-7, k 8-15), (n 8-15, k 0-7), (n 8-15, k 8-15)
      const int r = nn * 8 + (lane & 7) + (lane >> 4) * 8;
      const int c = kk * 16 + ((lane >> 3) & 1) * 8;
      ldsm_x4(b, smB + r * (DH + 8) + c);
      mma16816(acc[nn], a[kk], b);
      mma16816(acc[nn + 1], a[kk], b + 2);
    }
  }
}

// acc[16 x DH] += P(16 x 64, A fragments from C fragments) * Bm (64 x DH stored [64][DH+8], trans)
template <int DH>
__device__ __forceinline__ void mm_pb(float (*acc)[4], const float (*p)[4], const bf16* smB) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {  // 16 keys at a time
    uint32_t a[4];
    a[0] = pack_bf16(p[2 * kk][0], p[2 * kk][1]);
    a[1] = pack_bf16(p[2 * kk][2], p[2 * kk][3]);
    a[2] = pack_bf16(p[2 * kk + 1][0], p[2 * kk + 1][1]);
    a[3] = pack_bf16(p[2 * kk + 1][2], p[2 * kk + 1][3]);
#pragma unroll
    for (int nn = 0; nn < DH / 8; nn += 2) {
      uint32_t b[4];
      // matrices: (k 0-7, n 0-7), (k 8-15, n 0-7), (k 0-7, n 8-15), (k 8-15, n 8-15)
      const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      const int c = nn * 8 + (lane >> 4) * 8;
      ldsm_x4_t(b, smB + r * (DH + 8) + c);
      mma16816(acc[nn], a, b);
      mma16816(acc[nn + 1], a, b + 2);
    }
  }
}

// ---------------------------------------------------------------- forward
template <int DH>
__global__ void __launch_bounds__(NT) fa_fwd_kernel(const bf16* __restrict__ qkv, bf16* __restrict__ o,
                                                    float* __restrict__ lse, int T_, int h) {
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sQ = (bf16*)smraw;
  bf16* sK = sQ + 64 * (DH + 8);
  bf16* sV = sK + 64 * (DH + 8);
  const int qb = blockIdx.x, bh = blockIdx.y;
  const int b = bh / h, hh = bh % h;
  const int d = h * DH;
  const long ld = 3L * d;
  const bf16* base = qkv + (long)b * T_ * ld + hh * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const float sc = rsqrtf((float)DH) * LOG2E;
  const int q0 = qb * BR;
  load_tile<DH>(sQ, base, ld, q0, T_);
  __syncthreads();
  uint32_t qa[DH / 16][4];
  load_afrag<DH>(qa, sQ, warp * 16);
  float acc[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  const int nkb = min(qb + 1, (T_ + BC - 1) / BC);
  for (int kb = 0; kb < nkb; ++kb) {
    __syncthreads();
    load_tile<DH>(sK, base + d, ld, kb * BC, T_);
    load_tile<DH>(sV, base + 2 * d, ld, kb * BC, T_);
    __syncthreads();
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
    mm_abt<DH>(s, qa, sK);
    // scale, mask (causal + keys beyond T), row max
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nn = 0; nn < 8; ++nn)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = q0 + warp * 16 + g + (e >> 1) * 8;
        const int kj = kb * BC + nn * 8 + tig * 2 + (e & 1);
        float v = s[nn][e] * sc;
        if (kj > qi || kj >= T_) v = -INFINITY;
        s[nn][e] = v;
        mx[e >> 1] = fmaxf(mx[e >> 1], v);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float mnew[2], corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mnew[r] = fmaxf(m[r], mx[r]);
      corr[r] = (mnew[r] == -INFINITY) ? 1.f : exp2f(m[r] - mnew[r]);
    }
#pragma unroll
    for (int nn = 0; nn < 8; ++nn)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const float p = (mnew[r] == -INFINITY) ? 0.f : exp2f(s[nn][e] - mnew[r]);
        s[nn][e] = p;
        rs[r] += p;
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      l[r] = l[r] * corr[r] + rs[r];
      m[r] = mnew[r];
    }
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      acc[i][0] *= corr[0]; acc[i][1] *= corr[0];
      acc[i][2] *= corr[1]; acc[i][3] *= corr[1];
    }
    mm_pb<DH>(acc, s, sV);
  }
  // epilogue
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qi = q0 + warp * 16 + g + r * 8;
    if (qi >= T_) continue;
    const float inv = 1.f / l[r];
    bf16* orow = o + ((long)b * T_ + qi) * d + hh * DH;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i)
      *(__nv_bfloat162*)(orow + i * 8 + tig * 2) = __floats2bfloat162_rn(acc[i][2 * r] * inv, acc[i][2 * r + 1] * inv);
    if (tig == 0) lse[((long)b * h + hh) * T_ + qi] = (m[r] + log2f(l[r])) / LOG2E;
  }
}

// ---------------------------------------------------------------- backward: dK, dV
// Per warp: 16 keys.  S^T = K Q^T, P^T = exp(S^T - lse), dV += P^T dO, dP^T = V dO^T,
// dS^T = P^T (dP^T - D), dK += dS^T Q.
template <int DH>
__global__ void __launch_bounds__(NT) fa_bwd_dkv_kernel(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                        const float* __restrict__ lse, const float* __restrict__ Dsum,
                                                        bf16* __restrict__ dqkv, int T_, int h) {
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sK = (bf16*)smraw;
  bf16* sV = sK + 64 * (DH + 8);
  bf16* sQ = sV + 64 * (DH + 8);
  bf16* sO = sQ + 64 * (DH + 8);
  float* sL = (float*)(sO + 64 * (DH + 8));
  float* sD = sL + 64;
  const int kb = blockIdx.x, bh = blockIdx.y;
  const int b = bh / h, hh = bh % h;
  const int d = h * DH;
  const long ld = 3L * d;
  const bf16* base = qkv + (long)b * T_ * ld + hh * DH;
  const bf16* dob = dout + (long)b * T_ * d + hh * DH;
  const float* lrow = lse + ((long)b * h + hh) * T_;
  const float* drow = Dsum + ((long)b * h + hh) * T_;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const float sc = rsqrtf((float)DH);
  const int k0 = kb * BC;
  load_tile<DH>(sK, base + d, ld, k0, T_);
  load_tile<DH>(sV, base + 2 * d, ld, k0, T_);
  __syncthreads();
  uint32_t ka[DH / 16][4], va[DH / 16][4];
  load_afrag<DH>(ka, sK, warp * 16);
  load_afrag<DH>(va, sV, warp * 16);
  float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int nqb = (T_ + BR - 1) / BR;
  for (int qb = kb; qb < nqb; ++qb) {
    const int q0 = qb * BR;
    __syncthreads();
    load_tile<DH>(sQ, base, ld, q0, T_);
    load_tile<DH>(sO, dob, d, q0, T_);
    for (int i = threadIdx.x; i < 64; i += NT) {
      const bool ok = q0 + i < T_;
      sL[i] = ok ? lrow[q0 + i] * LOG2E : INFINITY;
      sD[i] = ok ? drow[q0 + i] : 0.f;
    }
    __syncthreads();
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
    mm_abt<DH>(s, ka, sQ);    // S^T [16 keys x 64 queries]
    mm_abt<DH>(dp, va, sO);   // dP^T = V dO^T
#pragma unroll
    for (int nn = 0; nn < 8; ++nn)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kj = k0 + warp * 16 + g + (e >> 1) * 8;
        const int qc = nn * 8 + tig * 2 + (e & 1);
        const int qi = q0 + qc;
        float p = exp2f(s[nn][e] * sc * LOG2E - sL[qc]);
        if (qi < kj || kj >= T_) p = 0.f;
        s[nn][e] = p;
        dp[nn][e] = p * (dp[nn][e] - sD[qc]);
      }
    mm_pb<DH>(dv, s, sO);     // dV += P^T dO
    mm_pb<DH>(dk, dp, sQ);    // dK += dS^T Q
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int kj = k0 + warp * 16 + g + r * 8;
    if (kj >= T_) continue;
    bf16* row = dqkv + ((long)b * T_ + kj) * ld + hh * DH;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      *(__nv_bfloat162*)(row + d + i * 8 + tig * 2) = __floats2bfloat162_rn(dk[i][2 * r] * sc, dk[i][2 * r + 1] * sc);
      *(__nv_bfloat162*)(row + 2 * d + i * 8 + tig * 2) = __floats2bfloat162_rn(dv[i][2 * r], dv[i][2 * r + 1]);
    }
  }
}

// ---------------------------------------------------------------- backward: dQ
template <int DH>
__global__ void __launch_bounds__(NT) fa_bwd_dq_kernel(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                       const float* __restrict__ lse, const float* __restrict__ Dsum,
                                                       bf16* __restrict__ dqkv, int T_, int h) {
  extern __shared__ __align__(16) uint8_t smraw[];
  bf16* sQ = (bf16*)smraw;
  bf16* sO = sQ + 64 * (DH + 8);
  bf16* sK = sO + 64 * (DH + 8);
  bf16* sV = sK + 64 * (DH + 8);
  const int qb = blockIdx.x, bh = blockIdx.y;
  const int b = bh / h, hh = bh % h;
  const int d = h * DH;
  const long ld = 3L * d;
  const bf16* base = qkv + (long)b * T_ * ld + hh * DH;
  const bf16* dob = dout + (long)b * T_ * d + hh * DH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const float sc = rsqrtf((float)DH);
  const int q0 = qb * BR;
  load_tile<DH>(sQ, base, ld, q0, T_);
  load_tile<DH>(sO, dob, d, q0, T_);
  __syncthreads();
  uint32_t qa[DH / 16][4], oa[DH / 16][4];
  load_afrag<DH>(qa, sQ, warp * 16);
  load_afrag<DH>(oa, sO, warp * 16);
  float Lr[2], Dr[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qi = q0 + warp * 16 + g + r * 8;
    const bool ok = qi < T_;
    Lr[r] = ok ? lse[((long)b * h + hh) * T_ + qi] * LOG2E : INFINITY;
    Dr[r] = ok ? Dsum[((long)b * h + hh) * T_ + qi] : 0.f;
  }
  float dq[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
  const int nkb = min(qb + 1, (T_ + BC - 1) / BC);
  for (int kb = 0; kb < nkb; ++kb) {
    __syncthreads();
    load_tile<DH>(sK, base + d, ld, kb * BC, T_);
    load_tile<DH>(sV, base + 2 * d, ld, kb * BC, T_);
    __syncthreads();
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
    mm_abt<DH>(s, qa, sK);
    mm_abt<DH>(dp, oa, sV);   // dP = dO V^T
#pragma unroll
    for (int nn = 0; nn < 8; ++nn)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = e >> 1;
        const int qi = q0 + warp * 16 + g + r * 8;
        const int kj = kb * BC + nn * 8 + tig * 2 + (e & 1);
        float p = exp2f(s[nn][e] * sc * LOG2E - Lr[r]);
        if (kj > qi || kj >= T_) p = 0.f;
        s[nn][e] = p * (dp[nn][e] - Dr[r]);   // dS
      }
    mm_pb<DH>(dq, s, sK);      // dQ += dS K
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qi = q0 + warp * 16 + g + r * 8;
    if (qi >= T_) continue;
    bf16* row = dqkv + ((long)b * T_ + qi) * ld + hh * DH;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i)
      *(__nv_bfloat162*)(row + i * 8 + tig * 2) = __floats2bfloat162_rn(dq[i][2 * r] * sc, dq[i][2 * r + 1] * sc);
  }
}

__global__ void dsum_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout, float* __restrict__ Dsum,
                            int B, int T_, int h, int dh) {
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  if (gw >= (long)B * h * T_) return;
  const int lane = threadIdx.x & 31;
  const int t = (int)(gw % T_);
  const int hh = (int)((gw / T_) % h);
  const int b = (int)(gw / ((long)T_ * h));
  const long off = ((long)b * T_ + t) * h * dh + hh * dh;
  float s = 0.f;
  for (int j = lane; j < dh; j += 32) s = fmaf(__bfloat162float(o[off + j]), __bfloat162float(dout[off + j]), s);
  s = warp_sum(s);
  if (lane == 0) Dsum[((long)b * h + hh) * T_ + t] = s;
}

template <int DH>
bool fwd(const bf16* qkv, bf16* o, float* lse, int B, int T_, int h, cudaStream_t st) {
  const int smem = 3 * 64 * (DH + 8) * 2;
  static bool once = false;
  if (!once) {
    ATOM_CUDA_OK(cudaFuncSetAttribute(fa_fwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    once = true;
  }
  dim3 grid((T_ + BR - 1) / BR, B * h);
  fa_fwd_kernel<DH><<<grid, NT, smem, st>>>(qkv, o, lse, T_, h);
  count_launch();
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

template <int DH>
bool bwd(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, float* Dsum, bf16* dqkv, int B, int T_,
         int h, cudaStream_t st) {
  const long warps = (long)B * h * T_;
  dsum_kernel<<<(warps + 7) / 8, 256, 0, st>>>(o, dout, Dsum, B, T_, h, DH);
  count_launch();
  const int smem_kv = 4 * 64 * (DH + 8) * 2 + 2 * 64 * 4;
  const int smem_q = 4 * 64 * (DH + 8) * 2;
  static bool once = false;
  if (!once) {
    ATOM_CUDA_OK(cudaFuncSetAttribute(fa_bwd_dkv_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv));
    ATOM_CUDA_OK(cudaFuncSetAttribute(fa_bwd_dq_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q));
    once = true;
  }
  dim3 grid((T_ + 63) / 64, B * h);
  fa_bwd_dkv_kernel<DH><<<grid, NT, smem_kv, st>>>(qkv, dout, lse, Dsum, dqkv, T_, h);
  count_launch();
  fa_bwd_dq_kernel<DH><<<grid, NT, smem_q, st>>>(qkv, dout, lse, Dsum, dqkv, T_, h);
  count_launch();
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

}  // namespace fa

bool attn_fa_supported(int dh) { return dh == 16 || dh == 64 || dh == 80 || dh == 128; }

bool attn_fwd_fa(const bf16* qkv, bf16* o, float* lse, int B, int T_, int h, int dh, cudaStream_t st) {
  switch (dh) {
    case 16: return fa::fwd<16>(qkv, o, lse, B, T_, h, st);
    case 64: return fa::fwd<64>(qkv, o, lse, B, T_, h, st);
    case 80: return fa::fwd<80>(qkv, o, lse, B, T_, h, st);
    case 128: return fa::fwd<128>(qkv, o, lse, B, T_, h, st);
  }
  set_error("attention: unsupported head size %d", dh);
  return false;
}

bool attn_bwd_fa(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, float* Dsum, bf16* dqkv, int B,
                 int T_, int h, int dh, cudaStream_t st) {
  switch (dh) {
    case 16: return fa::bwd<16>(qkv, o, dout, lse, Dsum, dqkv, B, T_, h, st);
    case 64: return fa::bwd<64>(qkv, o, dout, lse, Dsum, dqkv, B, T_, h, st);
    case 80: return fa::bwd<80>(qkv, o, dout, lse, Dsum, dqkv, B, T_, h, st);
    case 128: return fa::bwd<128>(qkv, o, dout, lse, Dsum, dqkv, B, T_, h, st);
  }
  set_error("attention: unsupported head size %d", dh);
  return false;
}

}  // namespace atom
