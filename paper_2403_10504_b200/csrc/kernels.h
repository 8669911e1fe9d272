// Internal (C++) declarations of libatom's kernel launchers.  The C-ABI lives in
// include/atom.h (training step) and include/atom_kernels.h (per-kernel test entry points).
#pragma once
#include <string>
#include "adam.h"
#include "common.cuh"
#include "epilogue.cuh"
#include "philox.cuh"

namespace atom {

const char* last_error();
std::string launch_log_text();

// dropout site multiplier y = D(x) (in place allowed; dropout.cu; R38)
template <typename T>
bool dropout(const T* x, T* y, long n, double p, uint64_t seed, uint32_t site, uint32_t layer, uint32_t step,
             cudaStream_t st);
template <typename T> bool dropout(const T* x, T* y, long n, const Drop& d, cudaStream_t st);
// y <- T(D(y) + r) (a residual branch's dropout fused with the residual add)
template <typename T> bool dropout_add(T* y, const T* r, long n, const Drop& d, cudaStream_t st);

// GEMM: D[m,n] = sum_k A[m,k] B[n,k] + epilogue.  *_mn = operand stored MN-major ([K][ld]).
bool gemm_tc(int M, int N, int K, const bf16* A, long lda, bool a_mn, const bf16* B, long ldb, bool b_mn,
             const Epi& e, cudaStream_t st, int force_bn = 0);
template <typename T>
bool gemm_simt(int M, int N, int K, const T* A, long lda, bool a_mn, const T* B, long ldb, bool b_mn, const Epi& e,
               cudaStream_t st);

// elementwise / reductions (elementwise.cu)
// res != NULL: x <- T(D(x) + res) in place first (a producing GEMM's residual add, moved here; D the
// residual-dropout mask of x's site, the identity when drop.thr == 0)
template <typename T> bool ln_fwd(const T* x, const T* g, const T* b, T* y, float* stats, long rows, int d, cudaStream_t st,
                                  const T* res = nullptr, Drop drop = Drop());
template <typename T> bool ln_apply(const T* x, const T* g, const T* b, const float* stats, T* y, long rows, int d, cudaStream_t st);
// part: fp32 range partials (at most 2 x ceil(rows / RED_ROWS) x d for ln_bwd); ticket: CS_TICKETS zeroed
// ints, one per block of 64 x (16 / sizeof(T)) columns, returned to zero by the kernel
constexpr int CS_TICKETS = 48;
template <typename T> bool ln_bwd(const T* dy, const T* x, const float* stats, const T* g, const T* dres, T* dx, float* dg,
                                  float* db, float* part, int* ticket, long rows, int d, cudaStream_t st);
template <typename T> bool bias_grad(const T* dy, long ld, long rows, int n, float* db, float* part, int* ticket,
                                     cudaStream_t st);
// gelu_out != NULL: also writes T(GELU(u)) there (the backward's re-apply of the fc activation)
template <typename T> bool dgelu_bias_grad(T* dy, const T* u, long rows, int n, float* db, float* part, int* ticket,
                                           cudaStream_t st, T* gelu_out = nullptr);
template <typename T> bool cross_entropy(T* logits, long ld, int V, const int32_t* targets, long tstride, int T_, long rows,
                                         float scale, float* loss, cudaStream_t st);
template <typename T> bool embed_fwd(const int32_t* tok, long tstride, int T_, long rows, const T* wte, const T* wpe, T* h,
                                     int d, cudaStream_t st);
template <typename T> bool embed_bwd(const int32_t* tok, long tstride, int T_, int B, const T* dh, int V, int d, float* dwte,
                                     float* dwpe, int* scratch, cudaStream_t st);
template <typename T> bool gelu_apply(const T* u, T* g, long n, cudaStream_t st);
template <typename T> bool adamw(float* p, const float* g, float* m, float* v, T* w, long n, const AdamConsts& k,
                                 cudaStream_t st);
template <typename T> bool cast_params(const float* src, T* dst, long n, cudaStream_t st);
bool init_normal(float* dst, long n, uint64_t seed, uint64_t base, float std, float fill, cudaStream_t st);
bool loss_sum(const float* l, long n, float scale, float* out, cudaStream_t st);
// dst <- src (n fp32) iff *flag == 1 (the guarded averaging commit, R36)
bool commit_if(float* dst, const float* src, long n, const int* flag, cudaStream_t st);

// attention (attn_simt.cu: fp32/bf16 CUDA cores; attn_fa.cu: bf16 tensor cores)
// qkv [B*T, 3d] rows (b,t): [q | k | v], head j at columns j*dh; o [B*T, d]; lse [B, h, T]
// drop: attention-probability dropout (site DS_ATTN; element index ((b h + head) T + q) T + k);
// the softmax normaliser and LSE use the undropped probabilities
template <typename T> bool attn_fwd_simt(const T* qkv, T* o, float* lse, int B, int T_, int h, int dh, cudaStream_t st,
                                         Drop drop = Drop());
template <typename T> bool attn_bwd_simt(const T* qkv, const T* o, const T* dout, const float* lse, float* Dsum, T* dqkv,
                                         int B, int T_, int h, int dh, cudaStream_t st, Drop drop = Drop());
bool attn_fwd_fa(const bf16* qkv, bf16* o, float* lse, int B, int T_, int h, int dh, cudaStream_t st);
bool attn_bwd_fa(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, float* Dsum, bf16* dqkv, int B,
                 int T_, int h, int dh, cudaStream_t st);
bool attn_fa_supported(int dh);
// tcgen05 / TMEM forward (attn_tc.cu)
bool attn_tc_supported(int dh, int d);
bool attn_fwd_tc(const bf16* qkv, bf16* o, float* lse, int B, int T_, int h, int dh, cudaStream_t st,
                 Drop drop = Drop());
// dsT != NULL: [B h][T][T] bf16 scratch: the dK/dV kernel also writes dS^T there and dQ = dS K runs
// as a separate kernel over it (no recomputation of S and dP); NULL: the dQ kernel recomputes them
bool attn_bwd_tc(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, float* Dsum, bf16* dqkv, int B,
                 int T_, int h, int dh, cudaStream_t st, cudaStream_t st2 = nullptr, Drop drop = Drop(),
                 bf16* dsT = nullptr);

}  // namespace atom
