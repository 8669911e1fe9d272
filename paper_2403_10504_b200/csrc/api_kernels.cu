// C-ABI per-kernel entry points (include/atom_kernels.h): used by the GPU parity tests to
// check each kernel against a plain fp32 reference on the same inputs.
#include "../../include/atom_kernels.h"
#include "kernels.h"
#include <string.h>

#include <map>
#include <mutex>

using namespace atom;

extern "C" {

int atom_k_gemm(int impl, int dtype, int M, int N, int K, const void* A, long lda, int a_mn, const void* B, long ldb,
                int b_mn, int mode, void* out, long ldo, void* out2, long ldo2, const void* bias, const void* res,
                long ldr, const void* aux, long ldx, int force_bn, void* stream) {
  Epi e;
  e.mode = mode;
  e.out = out; e.ldo = ldo; e.out2 = out2; e.ldo2 = ldo2;
  e.bias = bias; e.res = res; e.ldr = ldr; e.aux = aux; e.ldx = ldx;
  cudaStream_t st = (cudaStream_t)stream;
  bool ok;
  if (impl == ATOM_IMPL_TC) {
    if (dtype != ATOM_BF16) { set_error("tcgen05 GEMM is bf16 only"); return ATOM_E_INVALID; }
    ok = gemm_tc(M, N, K, (const bf16*)A, lda, a_mn, (const bf16*)B, ldb, b_mn, e, st, force_bn);
  } else if (dtype == ATOM_FP32) {
    ok = gemm_simt<float>(M, N, K, (const float*)A, lda, a_mn, (const float*)B, ldb, b_mn, e, st);
  } else {
    ok = gemm_simt<bf16>(M, N, K, (const bf16*)A, lda, a_mn, (const bf16*)B, ldb, b_mn, e, st);
  }
  if (ok) return ATOM_OK;
  return strncmp(last_error(), "CUDA", 4) == 0 ? ATOM_E_CUDA : ATOM_E_INVALID;
}

int atom_k_attn_fwd(int impl, int dtype, const void* qkv, void* o, float* lse, int B, int T, int h, int dh,
                    void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  bool ok;
  if (dtype == ATOM_FP32) {
    ok = attn_fwd_simt<float>((const float*)qkv, (float*)o, lse, B, T, h, dh, st);
  } else if (impl == ATOM_ATTN_TC) {
    ok = attn_fwd_tc((const bf16*)qkv, (bf16*)o, lse, B, T, h, dh, st);
  } else if (impl == ATOM_ATTN_MMA) {
    ok = attn_fwd_fa((const bf16*)qkv, (bf16*)o, lse, B, T, h, dh, st);
  } else {
    ok = attn_fwd_simt<bf16>((const bf16*)qkv, (bf16*)o, lse, B, T, h, dh, st);
  }
  if (ok) return ATOM_OK;
  return strncmp(last_error(), "CUDA", 4) == 0 ? ATOM_E_CUDA : ATOM_E_INVALID;
}

int atom_k_attn_bwd(int impl, int dtype, const void* qkv, const void* o, const void* dout, const float* lse,
                    float* dsum, void* dqkv, int B, int T, int h, int dh, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  bool ok;
  if (dtype == ATOM_FP32)
    ok = attn_bwd_simt<float>((const float*)qkv, (const float*)o, (const float*)dout, lse, dsum, (float*)dqkv, B, T,
                              h, dh, st);
  else if (impl == ATOM_ATTN_TC)
    ok = attn_bwd_tc((const bf16*)qkv, (const bf16*)o, (const bf16*)dout, lse, dsum, (bf16*)dqkv, B, T, h, dh, st);
  else if (impl == ATOM_ATTN_TC_DS) {
    // the dS^T scratch (an executor-owned buffer inside atom_step) is kept across calls here and
    // only grows, so back-to-back calls stay stream-ordered (no allocation or sync per call)
    static std::mutex mu;
    static std::map<int, std::pair<bf16*, size_t>> pool;   // device -> (buffer, bytes)
    const size_t need = (size_t)B * h * T * T * sizeof(bf16);
    int dev = 0;
    cudaGetDevice(&dev);
    bf16* dsT = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto& e = pool[dev];
      if (e.second < need) {
        if (e.first) {
          cudaDeviceSynchronize();
          cudaFree(e.first);
        }
        e = {nullptr, 0};
        if (cudaMalloc((void**)&e.first, need) != cudaSuccess) {
          set_error("CUDA: dS^T buffer allocation failed");
          return ATOM_E_CUDA;
        }
        e.second = need;
      }
      dsT = e.first;
    }
    ok = attn_bwd_tc((const bf16*)qkv, (const bf16*)o, (const bf16*)dout, lse, dsum, (bf16*)dqkv, B, T, h, dh, st,
                     nullptr, Drop(), dsT);
  }
  else if (impl == ATOM_ATTN_MMA)
    ok = attn_bwd_fa((const bf16*)qkv, (const bf16*)o, (const bf16*)dout, lse, dsum, (bf16*)dqkv, B, T, h, dh, st);
  else
    ok = attn_bwd_simt<bf16>((const bf16*)qkv, (const bf16*)o, (const bf16*)dout, lse, dsum, (bf16*)dqkv, B, T, h,
                             dh, st);
  if (ok) return ATOM_OK;
  return strncmp(last_error(), "CUDA", 4) == 0 ? ATOM_E_CUDA : ATOM_E_INVALID;
}

unsigned long long atom_k_launch_count(void) { return g_launch_count; }

int atom_k_launch_log(char* buf, int64_t cap, int64_t* len) {
  const std::string t = launch_log_text();
  if (len) *len = (int64_t)t.size();
  if (!buf || cap <= (int64_t)t.size()) {
    set_error("atom_k_launch_log: buffer of %lld bytes, need %zu", (long long)cap, t.size() + 1);
    return ATOM_E_INVALID;
  }
  memcpy(buf, t.c_str(), t.size() + 1);
  return ATOM_OK;
}

int atom_k_cpu_adamw(float* p, const float* g, float* m, float* v, long n, float lr_t, float b1, float b2, float eps,
                     float wd, long t, float gscale, int threads) {
  if (!p || !g || !m || !v || n < 0 || t < 1) {
    set_error("atom_k_cpu_adamw: invalid arguments");
    return ATOM_E_INVALID;
  }
  cpu_adamw(p, g, m, v, n, adam_consts(lr_t, b1, b2, eps, wd, t, gscale), threads);
  return ATOM_OK;
}

}  // extern "C"
