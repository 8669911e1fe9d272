/*
 * atom_kernels.h -- per-kernel C-ABI of libatom, for the GPU parity tests.
 *
 * Each entry runs one hand-written sm_100a kernel on caller-owned DEVICE buffers on the given
 * CUDA stream (NULL = legacy default stream) and returns atom_status (see atom.h).  Nothing is
 * synchronised; the caller synchronises before reading results.  Layouts are row-major.
 */
#ifndef ATOM_KERNELS_H
#define ATOM_KERNELS_H

#include "atom.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { ATOM_IMPL_TC = 0, ATOM_IMPL_SIMT = 1 };
/* GEMM epilogue modes (see csrc/epilogue.cuh) */
enum { ATOM_EPI_STORE = 0, ATOM_EPI_BIAS = 1, ATOM_EPI_BIAS_RES = 2, ATOM_EPI_BIAS_GELU = 3, ATOM_EPI_DGELU = 4,
       ATOM_EPI_ACC_F32 = 5 };

/* D[m,n] = sum_k A[m,k] B[n,k] (fp32 accumulate), then the epilogue `mode`:
 *   STORE out = D; BIAS out = D + bias[n]; BIAS_RES out = D + bias[n] + res[m,n];
 *   BIAS_GELU out = u = D + bias[n], out2 = gelu_tanh(u); DGELU out = D * gelu_tanh'(aux[m,n]);
 *   ACC_F32 out(fp32)[m,n] += D.       (nn.Linear of the minGPT block)
 * A is [M, lda] (K-major) or, with a_mn, [K, lda] (M contiguous); B likewise with N.
 * impl = ATOM_IMPL_TC: tcgen05/TMEM/TMA kernel, dtype must be ATOM_BF16, lda/ldb % 8 == 0;
 * impl = ATOM_IMPL_SIMT: CUDA-core kernel, dtype ATOM_FP32 or ATOM_BF16.
 * force_bn: 0 = automatic tile width, else 128 or 256 (TC only). */
int atom_k_gemm(int impl, int dtype, int M, int N, int K, const void* A, long lda, int a_mn, const void* B, long ldb,
                int b_mn, int mode, void* out, long ldo, void* out2, long ldo2, const void* bias, const void* res,
                long ldr, const void* aux, long ldx, int force_bn, void* stream);

/* Causal attention (minGPT CausalSelfAttention).  qkv: [B*T, 3*h*dh] rows (b, t) =
 * [q | k | v], head j at columns j*dh; o: [B*T, h*dh]; lse: fp32 [B, h, T] (natural log of the
 * softmax normaliser of scores q.k/sqrt(dh)).  impl: ATOM_ATTN_TC (tcgen05/TMEM, dh in {64, 80, 128};
 * the backward's dQ kernel recomputes S and dP), ATOM_ATTN_TC_DS (backward only: the dK/dV kernel
 * writes dS^T to a [B h][T][T] bf16 buffer and dQ = dS K runs over it -- the step's path when
 * T % 128 == 0, else as ATOM_ATTN_TC; here the buffer is allocated on first use and kept, growing
 * only, for later calls on the device), ATOM_ATTN_MMA (mma.sync flash attention, dh in
 * {16, 64, 80, 128}), ATOM_ATTN_SIMT (CUDA cores, dh <= 128).  dtype ATOM_FP32 always uses SIMT.
 * Backward: dout [B*T, h*dh] -> dqkv [B*T, 3*h*dh]; dsum fp32 [B, h, T] is scratch (rowsum(dout*o)). */
enum { ATOM_ATTN_TC = 0, ATOM_ATTN_MMA = 1, ATOM_ATTN_SIMT = 2, ATOM_ATTN_TC_DS = 3 };
int atom_k_attn_fwd(int impl, int dtype, const void* qkv, void* o, float* lse, int B, int T, int h, int dh,
                    void* stream);
int atom_k_attn_bwd(int impl, int dtype, const void* qkv, const void* o, const void* dout, const float* lse,
                    float* dsum, void* dqkv, int B, int T, int h, int dh, void* stream);

/* The CPU AdamW of the host update placement ("CPU AdamW"; R37) on host fp32
 * arrays p, m, v (updated in place) and g (read, scaled by gscale first): lr_t the step's learning
 * rate, t the 1-based update count, threads 0 = all cores.  Pure host code: runs without a GPU. */
int atom_k_cpu_adamw(float* p, const float* g, float* m, float* v, long n, float lr_t, float b1, float b2, float eps,
                     float wd, long t, float gscale, int threads);

/* Dropout site multiplier, in place allowed (x == y): y[i] = x[i] * keep(i) / (1 - p) on n
 * elements of dtype ATOM_FP32 or ATOM_BF16 (x, y 16-byte aligned), fp32 math.
 * keep(i) = (16-bit half i % 2 (0 = low) of word (i / 2) % 4 of Philox4x32-10(counter =
 * (i / 8, site, layer, micro_step), key = (seed & 0xffffffff, seed >> 32))) >= floor(p * 2^16).  SURVEY §8 NEXT-4 (minGPT's embd /
 * attn / resid dropout, the paper's profiled dropout layer); R38.  The
 * backward of a site is the same call on dy.  Requires 0 <= p < 1, n <= 2^35, else
 * ATOM_E_INVALID. */
int atom_k_dropout(int dtype, const void* x, void* y, long n, double p, unsigned long long seed, int site, int layer,
                   int micro_step, void* stream);

/* Number of kernels libatom launched in this process. */
unsigned long long atom_k_launch_count(void);

/* Launches per kernel family since the library was loaded, as text: one "<family> <count>" line
 * per family (e.g. "gemm_tc2<0,1> 12", "attn_fwd3<80> 4"), written NUL-terminated into the
 * caller-owned buf of cap bytes; *len = text length.  ATOM_E_INVALID if cap <= *len (nothing
 * written; call again with a larger buffer).  Tests use it to prove which kernels a step ran. */
int atom_k_launch_log(char* buf, int64_t cap, int64_t* len);

#ifdef __cplusplus
}
#endif
#endif /* ATOM_KERNELS_H */
