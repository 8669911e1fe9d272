// SIMT GEMM (CUDA cores, fp32 accumulate) with the same operand conventions and fused
// epilogues as the tcgen05 GEMM.  It is the contraction of the fp32 parity path
// (north star: fp32 results within 1e-4 of the oracle; tcgen05 kind::tf32 would not meet
// that bound), and never runs on the bf16 performance path.
#include "common.cuh"
#include "epilogue.cuh"

namespace atom {

constexpr int ST = 64;   // tile edge
constexpr int SK = 16;   // k step

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int M, int N, int K, const T* __restrict__ A, long lda,
                                                        int a_mn, const T* __restrict__ B, long ldb, int b_mn,
                                                        Epi e) {
  __shared__ float As[SK][ST + 1];
  __shared__ float Bs[SK][ST + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const long m0 = (long)blockIdx.y * ST, n0 = (long)blockIdx.x * ST;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += SK) {
    for (int i = threadIdx.x; i < SK * ST; i += 256) {
      int kk, rr;
      if (a_mn) { kk = i / ST; rr = i % ST; } else { rr = i / SK; kk = i % SK; }
      long m = m0 + rr, k = k0 + kk;
      As[kk][rr] = (m < M && k < K) ? to_f(a_mn ? A[k * lda + m] : A[m * lda + k]) : 0.f;
      if (b_mn) { kk = i / ST; rr = i % ST; } else { rr = i / SK; kk = i % SK; }
      long n = n0 + rr;
      k = k0 + kk;
      Bs[kk][rr] = (n < N && k < K) ? to_f(b_mn ? B[k * ldb + n] : B[n * ldb + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      long m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) epi_scalar<T>(e, m, n, acc[i][j]);
    }
}

template <typename T>
bool gemm_simt(int M, int N, int K, const T* A, long lda, bool a_mn, const T* B, long ldb, bool b_mn, const Epi& e,
               cudaStream_t st) {
  if (M <= 0 || N <= 0) return true;
  dim3 grid((N + ST - 1) / ST, (M + ST - 1) / ST);
  gemm_simt_kernel<T><<<grid, 256, 0, st>>>(M, N, K, A, lda, a_mn, B, ldb, b_mn, e);
  count_launch();
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

template bool gemm_simt<float>(int, int, int, const float*, long, bool, const float*, long, bool, const Epi&,
                               cudaStream_t);
template bool gemm_simt<bf16>(int, int, int, const bf16*, long, bool, const bf16*, long, bool, const Epi&,
                              cudaStream_t);

}  // namespace atom
