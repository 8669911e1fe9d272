// tcgen05 / TMEM / TMA GEMM for sm_100a (bf16 x bf16 -> fp32 accumulate in TMEM) with the
// fused epilogues of epilogue.cuh.  This is the contraction behind every nn.Linear of the
// GPT-3 block and the lm_head:
//
//   D[m, n] = sum_k A[m, k] B[n, k]
//
// A and B are each either K-major (row-major [rows][ld], K contiguous) or MN-major
// ([K][ld], M or N contiguous), which covers forward (K,K), dgrad (K,MN) and wgrad (MN,MN)
// without transposes.
//
// Structure (persistent, warp-specialised, one CTA per SM):
//   warp 0      TMA producer: 128B-swizzled tiles of A (128 x 64) and B (BN x 64) into a
//               STAGES-deep shared-memory ring (full/empty mbarriers)
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.cta_group::1.kind::f16
//               (M=128, N=BN, K=16) into a double-buffered TMEM accumulator and commits
//               to the ring's empty barrier / the accumulator's full barrier
//   warp 2      TMEM allocator (2*BN columns)
//   warps 4..7  epilogue: tcgen05.ld 32x32b.x32 -> registers -> fused epilogue -> global
#include <cuda.h>
#include <map>
#include <mutex>
#include <string>

#include "common.cuh"
#include "epilogue.cuh"

namespace atom {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// tcgen05.ld without the wait (the caller overlaps it with other work, then tmem_wait_ld())
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, 128-byte swizzle (sm100 encoding: version 1 at bit 46,
// layout type SWIZZLE_128B = 2 at bits 61..63; LBO / SBO in 16-byte units).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// One lane of a converged warp (elect.sync). MMAs issued under this predicate compile to
// back-to-back UTCHMMA; under `lane == 0` ptxas wraps every tcgen05.mma in its own
// ELECT / BRA.U.ANY loop, which limited issue to ~100 cycles per MMA (tools/tmem_bw.cu).
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(p));
  return p != 0;
}
// Instruction descriptor, kind::f16: D fp32 (bit 4), A/B bf16 (bits 7, 10), major bits 15/16,
// N>>3 at bit 17, M>>4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int BM = 128;
constexpr int BK = 64;

// Grouped raster: consecutive tiles walk GROUP_M m-blocks down before moving right, so the
// ~148 tiles in flight cover a GROUP_M x (148 / GROUP_M) block of the output and re-read A and
// B from L2 instead of DRAM.
// GROUP_M adapts to K (host side, group_m_for): the A row panels of a group must stay in L2
// next to B; with a fixed 16 the K = 10240 projection GEMM read A from DRAM 2.5x over.
constexpr int GROUP_M = 16;
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int* mb, int* nb, int group_m) {
  const int per_group = group_m * num_n;
  const int g = tile / per_group;
  const int first = g * group_m;
  const int gsz = min(num_m - first, group_m);
  const int r = tile - g * per_group;
  *mb = first + r % gsz;
  *nb = r / gsz;
}

template <int BN>
struct TcCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int EPI_BIAS_BYTES = 4 * BN * 2;   // one bias row per epilogue warp
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + EPI_BIAS_BYTES;
};

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(256, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, Epi epi, int group_m) {
  using Cfg = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = (uint64_t*)(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  bf16* sbias = (bf16*)(smem + Cfg::STAGES * Cfg::STAGE_BYTES + 256);   // [4][BN]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(tile, num_m, num_n, &mb, &nb, group_m);
        const int m0 = mb * BM;
        const int n0 = nb * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
          const int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d(sa + j * 8192, &tmA, &full[stage], m0 + 64 * j, k0);
          } else {
            tma_load_2d(sa, &tmA, &full[stage], k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(sb + j * 8192, &tmB, &full[stage], n0 + 64 * j, k0);
          } else {
            tma_load_2d(sb, &tmB, &full[stage], k0, n0);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
    const bool elected = elect_one();
    // stage-0 descriptors; stage s and K step kk only add constants to the address field
    const uint64_t a_desc0 = A_MN ? desc_sw128(smem_u32(smem), 8192, 1024) : desc_sw128(smem_u32(smem), 16, 1024);
    const uint64_t b_desc0 = B_MN ? desc_sw128(smem_u32(smem) + Cfg::A_BYTES, 8192, 1024)
                                  : desc_sw128(smem_u32(smem) + Cfg::A_BYTES, 16, 1024);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elected) {
          const uint64_t sofs = (uint64_t)((stage * Cfg::STAGE_BYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = a_desc0 + sofs + (A_MN ? kk * 128 : kk * 2);
            const uint64_t bd = b_desc0 + sofs + (B_MN ? kk * 128 : kk * 2);
            tc_mma(tmem_d, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (kb == num_kb - 1) tc_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == Cfg::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      int mb, nb;
      tile_coords(tile, num_m, num_n, &mb, &nb, group_m);
      const int m0 = mb * BM;
      const int n0 = nb * BN;
      const long m = m0 + 32 * q + lane;
      // fast path: interior tiles of the modes without per-row global operands (the residual /
      // pre-activation prefetch of EPI_BIAS_RES / EPI_DGELU measured slower than the plain loop)
      const bool fast = (epi.mode == EPI_STORE || epi.mode == EPI_BIAS || epi.mode == EPI_BIAS_GELU) &&
                        m0 + BM <= M && n0 + BN <= N;
      const bool has_bias = epi.mode == EPI_BIAS || epi.mode == EPI_BIAS_RES || epi.mode == EPI_BIAS_GELU;
      bf16* sb = sbias + q * BN;
      if (fast && has_bias) {   // this tile's bias row into the warp's smem row (before the wait)
        __syncwarp();
        if (8 * lane < BN) *(uint4*)(sb + 8 * lane) = *(const uint4*)((const bf16*)epi.bias + n0 + 8 * lane);
        __syncwarp();
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t trow = tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN;
      if (fast) {
        // interior tile: TMEM chunk c + 1 and its residual / pre-activation operands are in flight
        // while chunk c is finished and stored
        const bf16* xrow = epi.mode == EPI_BIAS_RES ? (const bf16*)epi.res + m * epi.ldr
                         : epi.mode == EPI_DGELU   ? (const bf16*)epi.aux + m * epi.ldx : nullptr;
        uint32_t va[32], vb[32];
        uint4 xa[4], xb[4];
        // chunk c's operands in (vc, xc); chunk c + 1's are loaded into (vn, xn) meanwhile
        auto chunk = [&](int c, uint32_t (&vc)[32], uint4 (&xc)[4], uint32_t (&vn)[32], uint4 (&xn)[4]) {
          if (c + 1 < BN / 32) {
            tmem_ld32_nw(trow + 32 * (c + 1), vn);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              xn[j] = xrow ? *(const uint4*)(xrow + n0 + 32 * (c + 1) + 8 * j) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float a[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a[i] = __uint_as_float(vc[8 * j + i]);
            const uint4 b8 = has_bias ? *(const uint4*)(sb + 32 * c + 8 * j) : make_uint4(0, 0, 0, 0);
            epi_vec8_bf16_pre(epi, m, n0 + 32 * c + 8 * j, a, b8, xc[j]);
          }
          if (c + 1 < BN / 32) tmem_wait_ld();
        };
        tmem_ld32_nw(trow, va);
#pragma unroll
        for (int j = 0; j < 4; ++j) xa[j] = xrow ? *(const uint4*)(xrow + n0 + 8 * j) : make_uint4(0, 0, 0, 0);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < BN / 32; c += 2) {
          chunk(c, va, xa, vb, xb);
          chunk(c + 1, vb, xb, va, xa);
        }
      } else {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(trow + c0, v);
          const int nb = n0 + c0;
          if (m < M && nb < N) {
            if (nb + 32 <= N) {
#pragma unroll
              for (int j = 0; j < 4; ++j) epi_vec8_bf16(epi, m, nb + 8 * j, v + 8 * j);
            } else {
              for (int j = 0; j < 32 && nb + j < N; ++j) epi_scalar<bf16>(epi, m, nb + j, v[j]);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ 2-CTA variant
// A CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile with tcgen05.mma.cta_group::2:
// each CTA stages its 128 rows of A and its 128 rows of B (half the operand bytes per SM of the
// 1-CTA kernel), the leader CTA issues the M=256 MMAs, each CTA's TMEM holds its 128 x 256
// accumulator half and its own epilogue drains it.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// remote arrive on a peer CTA's mbarrier.  Default (CTA-scope) release: an explicit
// .release.cluster compiles to MEMBAR.ALL.GPU, which made every arrive wait for the thread's
// outstanding global stores (profiles/r01: 2-CTA GEMM at 34% tensor-pipe activity).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                 int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

struct Tc2Cfg {
  static constexpr int BN = 256;         // cluster tile N (each CTA stages BN/2 rows of B)
  static constexpr int HB = BN / 2;
  static constexpr int STAGES = 6;
  static constexpr int A_BYTES = BM * BK * 2;  // this CTA's 128 rows of A
  static constexpr int B_BYTES = HB * BK * 2;  // this CTA's 128 rows of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int EPI_BIAS_BYTES = 4 * BN * 2;   // one bias row per epilogue warp
  // TMA-store staging: per epilogue warp one 32 x 32 bf16 box per output (64B-swizzled rows)
  static constexpr int STG_BOX = 32 * 32 * 2;
  static constexpr int STG_BYTES = 4 * 2 * STG_BOX;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256 + EPI_BIAS_BYTES + STG_BYTES;
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t smem, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Stream-K tail of the fp32-accumulating (weight-gradient) GEMMs: the last partial wave of tiles
// (num_tiles % clusters of them) would leave most CTA pairs idle, so each of those tiles is split
// into P parts along K, one work unit each, run by different pairs. A part writes its fp32 partial
// tile to a workspace; the last part of a tile to finish (atomic ticket: who, never the order)
// adds the P partials in part order to the output -- deterministic. No unit ever waits for another.
struct SplitK {
  int base = 0;          // tiles processed whole (units 0 .. base-1)
  int P = 1;             // parts per tail tile (1: no split)
  float* ws = nullptr;   // [tail * P][2 CTAs][BM][BN] fp32 partials
  int* ticket = nullptr; // [tail][2], zero between launches
};
struct Unit {
  int tile, kb0, kb1, part, tail;
};
__device__ __forceinline__ Unit unit_of(int u, int num_kb, const SplitK& sk) {
  Unit w;
  if (sk.P <= 1 || u < sk.base) {
    w.tile = u; w.kb0 = 0; w.kb1 = num_kb; w.part = -1; w.tail = -1;
  } else {
    const int v = u - sk.base;
    w.tail = v / sk.P;
    w.part = v % sk.P;
    w.tile = sk.base + w.tail;
    w.kb0 = (int)((long)w.part * num_kb / sk.P);
    w.kb1 = (int)((long)(w.part + 1) * num_kb / sk.P);
  }
  return w;
}

template <bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2, int M, int N,
                    int K, Epi epi, int group_m, SplitK sk) {
  using Cfg = Tc2Cfg;
  constexpr int BN = Cfg::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sstage = smem + Cfg::STAGES * Cfg::STAGE_BYTES;   // 1024-aligned: [4 warps][2 outputs] boxes
  uint64_t* full = (uint64_t*)(smem + Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::STG_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* tfull = empty + Cfg::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  bf16* sbias = (bf16*)(smem + Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::STG_BYTES + 256);   // [4][BN]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int num_m = (M + 2 * BM - 1) / (2 * BM);
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + BK - 1) / BK;
  const int cluster_id = blockIdx.x >> 1;
  const int num_clusters = gridDim.x >> 1;
  const int num_units = sk.P <= 1 ? num_tiles : sk.base + (num_tiles - sk.base) * sk.P;
  __shared__ int sk_last;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 2);   // leader arrive.expect_tx + peer's remote arrive
      mbar_init(&empty[s], 1);  // one multicast MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // one arrive per epilogue warp of both CTAs (used in the leader)
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cluster_id; u < num_units; u += num_clusters) {
        const Unit w = unit_of(u, num_kb, sk);
        int mb, nb;
        tile_coords(w.tile, num_m, num_n, &mb, &nb, group_m);
        const int m0 = mb * 2 * BM + rank * BM;
        const int n0 = nb * BN + rank * Cfg::HB;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          const uint32_t lbar = mapa_shared(smem_u32(&full[stage]), 0);
          if (leader)
            mbar_expect_tx(&full[stage], 2 * Cfg::STAGE_BYTES);
          else
            mbar_arrive_cluster(lbar);
          const int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair(sa + j * 8192, &tmA, lbar, m0 + 64 * j, k0);
          } else {
            tma_load_2d_pair(sa, &tmA, lbar, k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < Cfg::HB / 64; ++j) tma_load_2d_pair(sb + j * 8192, &tmB, lbar, n0 + 64 * j, k0);
          } else {
            tma_load_2d_pair(sb, &tmB, lbar, k0, n0);
          }
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader only)
    if (leader) {
      constexpr uint32_t idesc = idesc_bf16(2 * BM, BN, A_MN, B_MN);
      const bool elected = elect_one();
      const uint64_t a_desc0 =
          A_MN ? desc_sw128(smem_u32(smem), 8192, 1024) : desc_sw128(smem_u32(smem), 16, 1024);
      const uint64_t b_desc0 = B_MN ? desc_sw128(smem_u32(smem) + Cfg::A_BYTES, 8192, 1024)
                                    : desc_sw128(smem_u32(smem) + Cfg::A_BYTES, 16, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = cluster_id; u < num_units; u += num_clusters, ++it) {
        const Unit w = unit_of(u, num_kb, sk);
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elected) {
            const uint64_t sofs = (uint64_t)((stage * Cfg::STAGE_BYTES) >> 4);
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ad = a_desc0 + sofs + (A_MN ? kk * 128 : kk * 2);
              const uint64_t bd = b_desc0 + sofs + (B_MN ? kk * 128 : kk * 2);
              tc_mma_pair(tmem_d, ad, bd, idesc, (kb != w.kb0 || kk != 0) ? 1u : 0u);
            }
            tc_commit_pair(&empty[stage]);
            if (kb == w.kb1 - 1) tc_commit_pair(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == Cfg::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;
    int it = 0;
    for (int u = cluster_id; u < num_units; u += num_clusters, ++it) {
      const Unit w = unit_of(u, num_kb, sk);
      const int tile = w.tile;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      int mb, nb;
      tile_coords(tile, num_m, num_n, &mb, &nb, group_m);
      const int m0 = mb * 2 * BM + rank * BM;
      const int n0 = nb * BN;
      const long m = m0 + 32 * q + lane;
      // fast path: interior tiles of the modes without per-row global operands (the residual /
      // pre-activation prefetch of EPI_BIAS_RES / EPI_DGELU measured slower than the plain loop)
      const bool fast = (epi.mode == EPI_STORE || epi.mode == EPI_BIAS || epi.mode == EPI_BIAS_GELU) &&
                        m0 + BM <= M && n0 + BN <= N && w.part < 0;
      const bool has_bias = epi.mode == EPI_BIAS || epi.mode == EPI_BIAS_RES || epi.mode == EPI_BIAS_GELU;
      bf16* sb = sbias + q * BN;
      if (fast && has_bias) {   // this tile's bias row into the warp's smem row (before the wait)
        __syncwarp();
        if (8 * lane < BN) *(uint4*)(sb + 8 * lane) = *(const uint4*)((const bf16*)epi.bias + n0 + 8 * lane);
        __syncwarp();
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t trow = tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN;
      if (w.part >= 0) {
        // stream-K tail unit (fp32 accumulate): this part's partial tile to the workspace; the last
        // part of this CTA's half-tile to finish adds all parts in part order to the output
        const int r = 32 * q + lane;
        float* wsp = sk.ws + ((long)(w.tail * sk.P + w.part) * 2 + rank) * (BM * BN) + (long)r * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(trow + c0, v);
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            __stcg((float4*)(wsp + c0 + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]));
        }
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (q == 0 && lane == 0) sk_last = atomicAdd(&sk.ticket[2 * w.tail + rank], 1) == sk.P - 1;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (sk_last) {
          __threadfence();
          const float* w0 = sk.ws + ((long)(w.tail * sk.P) * 2 + rank) * (BM * BN) + (long)r * BN;
          const long pstride = 2L * BM * BN;
          float* orow = (float*)epi.out + m * epi.ldo;
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 4) {
            const int n = n0 + c0;
            if (m >= M || n >= N) continue;
            float4 t = __ldcg((const float4*)(w0 + c0));
            for (int p = 1; p < sk.P; ++p) {
              const float4 x = __ldcg((const float4*)(w0 + p * pstride + c0));
              t.x += x.x; t.y += x.y; t.z += x.z; t.w += x.w;
            }
            const float tv[4] = {t.x, t.y, t.z, t.w};
            for (int j = 0; j < 4 && n + j < N; ++j) orow[n + j] += tv[j];
          }
          if (q == 0 && lane == 0) sk.ticket[2 * w.tail + rank] = 0;
        }
      } else if (fast) {
        // interior tile, TMEM chunk c + 1 in flight while chunk c is finished.
        // TMA-store epilogue: each warp packs its 32 rows x 32 columns of a chunk into a 64B-swizzled
        // smem box per output and one lane stores the box (full-line writes instead of 32 scattered
        // 16-byte pieces per instruction)
        const bool gelu2 = epi.mode == EPI_BIAS_GELU;
        uint8_t* stg = sstage + q * 2 * Cfg::STG_BOX;
        const uint32_t stg0 = smem_u32(stg), stg1 = stg0 + Cfg::STG_BOX;
        const uint32_t row_off = (uint32_t)lane * 64;
        const uint32_t swz = (uint32_t)((lane >> 1) & 3);
        const int mrow = m0 + 32 * q;
        uint32_t va[32], vb[32];
        auto chunk = [&](int c, uint32_t (&vc)[32], uint32_t (&vn)[32]) {
          if (c + 1 < BN / 32) tmem_ld32_nw(trow + 32 * (c + 1), vn);
          uint4 ov[4], gv[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float a8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) a8[i] = __uint_as_float(vc[8 * j + i]);
            const uint4 b8 = has_bias ? *(const uint4*)(sb + 32 * c + 8 * j) : make_uint4(0, 0, 0, 0);
            epi_pack8_bf16(epi.mode, a8, b8, &ov[j], &gv[j]);
          }
          if (lane == 0) bulk_wait_read0();   // the previous chunk's boxes have been read out
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t off = row_off + ((((uint32_t)j) ^ swz) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg0 + off), "r"(ov[j].x), "r"(ov[j].y),
                         "r"(ov[j].z), "r"(ov[j].w)
                         : "memory");
            if (gelu2)
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(stg1 + off), "r"(gv[j].x), "r"(gv[j].y),
                           "r"(gv[j].z), "r"(gv[j].w)
                           : "memory");
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmO, stg0, n0 + 32 * c, mrow);
            if (gelu2) tma_store_2d(&tmO2, stg1, n0 + 32 * c, mrow);
            bulk_commit();
          }
          if (c + 1 < BN / 32) tmem_wait_ld();
        };
        tmem_ld32_nw(trow, va);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < BN / 32; c += 2) {
          chunk(c, va, vb);
          chunk(c + 1, vb, va);
        }
      } else {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(trow + c0, v);
          const int nb = n0 + c0;
          if (m < M && nb < N) {
            if (nb + 32 <= N) {
#pragma unroll
              for (int j = 0; j < 4; ++j) epi_vec8_bf16(epi, m, nb + 8 * j, v + 8 * j);
            } else {
              for (int j = 0; j < 32 && nb + j < N; ++j) epi_scalar<bf16>(epi, m, nb + j, v[j]);
            }
          }
        }
      }

      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
    }
  }
  if (warp >= 4 && lane == 0) bulk_wait_all();   // TMA stores complete before the CTA retires
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  });
  return fn;
}

// 2-D bf16 tensor map: inner dimension `inner` (contiguous), `outer` rows of pitch ld elements.
static bool make_map(CUtensorMap* map, const void* base, long inner, long outer, long ld, int box_inner,
                     int box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%ld outer=%ld ld=%ld", (int)r, inner, outer, ld);
    return false;
  }
  return true;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// m-blocks per raster group: keep ~40 MB of A row panels (group_m x rows x K bf16) live in L2
// Data-gradient GEMMs (B MN-major, A K-major) run faster with half the footprint: measured on B200
// (tools/gpu_run55.sh, interleaved A/B) QKV data gradient +6.8 %, fc +1 %, fc2 +2.7 %; the forward
// and weight-gradient GEMMs showed no gain
#ifndef ATOM_GEMM_GROUP_MB
#define ATOM_GEMM_GROUP_MB 40
#endif
#ifndef ATOM_GEMM_GROUP_MB_DGRAD
#define ATOM_GEMM_GROUP_MB_DGRAD 20
#endif
static int group_m_for(int K, int ctas_per_tile, bool dgrad) {
  const long panel = (long)BM * ctas_per_tile * K * 2;
  long g = ((long)(dgrad ? ATOM_GEMM_GROUP_MB_DGRAD : ATOM_GEMM_GROUP_MB) << 20) / (panel > 0 ? panel : 1);
  return (int)(g < 2 ? 2 : g > GROUP_M ? GROUP_M : g);
}

template <int BN, bool A_MN, bool B_MN>
static bool launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const Epi& e,
                      cudaStream_t st) {
  using Cfg = TcCfg<BN>;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    ATOM_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr_set = true;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  kern<<<grid, 256, Cfg::SMEM, st>>>(ta, tb, M, N, K, e, group_m_for(K, 1, !A_MN && B_MN));
  static const std::string name = "gemm_tc<" + std::to_string(BN) + "," + std::to_string((int)A_MN) + "," +
                                  std::to_string((int)B_MN) + ">";
  count_launch(name.c_str());
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

// stream-K workspace per stream (a split GEMM only ever overlaps split GEMMs of other streams):
// room for one partial tile per CTA pair (tail * P <= clusters) and the tickets, zeroed once
struct SplitWs {
  float* ws = nullptr;
  int* ticket = nullptr;
};
// Off by default: in the 2.7B step the weight-gradient GEMMs run on a side stream whose tails the
// main stream's kernels already fill, and the split's workspace traffic and final sums cost more
// than the idle pairs it recovers (interleaved A/B on B200, tools/gpu_run60.sh: 53.4K tokens/s
// with the split vs 55.1K without). ATOM_GEMM_SPLITK=1 turns it on (tests cover both).
static bool splitk_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("ATOM_GEMM_SPLITK");
    on = v && v[0] == '1';
  }
  return on == 1;
}
static SplitWs* splitk_ws(cudaStream_t st, int clusters) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SplitWs> pool;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  SplitWs& w = pool[{dev, st}];
  if (!w.ws) {
    clusters = num_sms() / 2;   // the most any launch uses
    const size_t nws = (size_t)clusters * 2 * BM * Tc2Cfg::BN;
    if (cudaMalloc((void**)&w.ws, nws * sizeof(float)) != cudaSuccess ||
        cudaMalloc((void**)&w.ticket, (size_t)clusters * 2 * sizeof(int)) != cudaSuccess ||
        cudaMemset(w.ticket, 0, (size_t)clusters * 2 * sizeof(int)) != cudaSuccess) {
      set_error("gemm_tc: stream-K workspace allocation failed");
      return nullptr;
    }
  }
  return &w;
}

template <bool A_MN, bool B_MN>
static bool launch_tc2(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const Epi& e,
                       cudaStream_t st) {
  // output boxes for the TMA-store epilogue (store / bias / bias+GELU modes): 32 x 32, 64B swizzle
  CUtensorMap to, to2;
  memset(&to, 0, sizeof to);
  memset(&to2, 0, sizeof to2);
  const bool tma_out = e.mode == EPI_STORE || e.mode == EPI_BIAS || e.mode == EPI_BIAS_GELU;
  if (tma_out) {
    if (!make_map(&to, e.out, N, M, e.ldo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)) return false;
    if (e.mode == EPI_BIAS_GELU && !make_map(&to2, e.out2, N, M, e.ldo2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
      return false;
  }
  auto kern = gemm_tc2_kernel<A_MN, B_MN>;
  static bool attr_set = false;
  if (!attr_set) {
    ATOM_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Tc2Cfg::SMEM));
    attr_set = true;
  }
  const int tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + Tc2Cfg::BN - 1) / Tc2Cfg::BN);
  int clusters = std::min(tiles, num_sms() / 2);
  SplitK sk;
  if (e.mode == EPI_ACC_F32 && splitk_enabled()) {
    // stream-K tail: split the last partial wave's tiles along K so that it fills the CTA pairs
    const int tail = tiles % clusters, num_kb = (K + BK - 1) / BK;
    if (tiles > clusters && tail > 0) {
      const int P = std::min(std::min(clusters / tail, 16), num_kb / 4);
      if (P >= 2) {
        SplitWs* w = splitk_ws(st, clusters);
        if (!w) return false;
        sk.base = tiles - tail;
        sk.P = P;
        sk.ws = w->ws;
        sk.ticket = w->ticket;
      }
    }
  }
  kern<<<2 * clusters, 256, Tc2Cfg::SMEM, st>>>(ta, tb, to, to2, M, N, K, e, group_m_for(K, 2, !A_MN && B_MN), sk);
  static const std::string name = "gemm_tc2<" + std::to_string((int)A_MN) + "," + std::to_string((int)B_MN) + ">";
  static const std::string name_sk = "gemm_tc2_splitk<" + std::to_string((int)A_MN) + "," + std::to_string((int)B_MN) + ">";
  count_launch(sk.P > 1 ? name_sk.c_str() : name.c_str());
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

// Kernel choice by estimated time: waves x per-SM tile work / relative speed
// (2-CTA 256x256 > 1-CTA 128x256 > 1-CTA 128x128 in per-SM efficiency).  Returns 512 for the
// 2-CTA kernel, else the 1-CTA tile width.
static bool g_allow_2cta = true;
static int pick_bn(int M, int N) {
  const int sms = num_sms();
  struct V { int code; long tiles; int slots; double work, speed; };
  // relative per-SM speeds measured on B200 (tools/gemm_perf.py): 128-wide tiles ~0.6x of 256-wide
  V vs[3] = {{512, (long)((M + 255) / 256) * ((N + 255) / 256), sms / 2, 128.0 * 256, 1.0},
             {256, (long)((M + 127) / 128) * ((N + 255) / 256), sms, 128.0 * 256, 0.9},
             {128, (long)((M + 127) / 128) * ((N + 127) / 128), sms, 128.0 * 128, 0.6}};
  double best = 1e300;
  int code = 256;
  for (auto& v : vs) {
    if (v.code == 512 && (!g_allow_2cta || M < 256)) continue;
    const double t = (double)((v.tiles + v.slots - 1) / v.slots) * v.work / v.speed;
    if (t < best * 0.999) {
      best = t;
      code = v.code;
    }
  }
  return code;
}

// (legacy chooser kept for reference by force_bn = 1)
static int pick_bn_1cta(int M, int N) {
  const int sms = num_sms();
  double best = -1;
  int bn_best = 256;
  for (int bn : {256, 128}) {
    long tiles = (long)((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    long waves = (tiles + sms - 1) / sms;
    double eff = (double)tiles / (double)(waves * sms) * (bn == 256 ? 1.0 : 0.93);
    if (eff > best + 1e-9) {
      best = eff;
      bn_best = bn;
    }
  }
  return bn_best;
}

bool gemm_tc(int M, int N, int K, const bf16* A, long lda, bool a_mn, const bf16* B, long ldb, bool b_mn,
             const Epi& e, cudaStream_t st, int force_bn) {
  if (M <= 0 || N <= 0 || K <= 0) return true;
  if ((lda % 8) || (ldb % 8) || ((uintptr_t)A & 15) || ((uintptr_t)B & 15)) {
    set_error("gemm_tc: operands need 16-byte aligned rows (lda=%ld ldb=%ld)", lda, ldb);
    return false;
  }
  const int bn = force_bn ? force_bn : pick_bn(M, N);
  CUtensorMap ta, tb;
  bool ok = a_mn ? make_map(&ta, A, M, K, lda, 64, 64) : make_map(&ta, A, K, M, lda, 64, BM);
  if (!ok) return false;
  // the 2-CTA kernel stages 128 rows of B per CTA
  ok = b_mn ? make_map(&tb, B, N, K, ldb, 64, 64) : make_map(&tb, B, K, N, ldb, 64, bn == 512 ? 128 : bn);
  if (!ok) return false;
  if (bn == 512) {
    if (!a_mn && !b_mn) return launch_tc2<false, false>(ta, tb, M, N, K, e, st);
    if (!a_mn && b_mn) return launch_tc2<false, true>(ta, tb, M, N, K, e, st);
    if (a_mn && b_mn) return launch_tc2<true, true>(ta, tb, M, N, K, e, st);
    return launch_tc2<true, false>(ta, tb, M, N, K, e, st);
  }
#define ATOM_TC_CASE(BN_, AM, BMN) \
  if (bn == BN_ && a_mn == AM && b_mn == BMN) return launch_tc<BN_, AM, BMN>(ta, tb, M, N, K, e, st);
  ATOM_TC_CASE(256, false, false)
  ATOM_TC_CASE(256, false, true)
  ATOM_TC_CASE(256, true, true)
  ATOM_TC_CASE(256, true, false)
  ATOM_TC_CASE(128, false, false)
  ATOM_TC_CASE(128, false, true)
  ATOM_TC_CASE(128, true, true)
  ATOM_TC_CASE(128, true, false)
#undef ATOM_TC_CASE
  set_error("gemm_tc: unsupported tile width %d", bn);
  return false;
}

}  // namespace atom
