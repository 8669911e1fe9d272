// Causal attention on 5th-gen tensor cores (tcgen05 / TMEM / TMA), flash style.
// minGPT CausalSelfAttention: o_t = sum_{s<=t} softmax_s(q_t.k_s/sqrt(dh)) v_s,
// LSE stashed for the backward.
//   forward   attn_fwd3_tc_kernel: persistent, one CTA per SM over (b h, query pair) items; two
//             128-query tiles ping-pong between two softmax warpgroups (thread = query row = TMEM
//             lane), P written back over S in TMEM as the A operand of O += P V
//   backward  dsum_tc_kernel (D = rowsum(dO o)), attn_bwd_dkv4_kernel (dK, dV per 128-key block;
//             optionally writes dS^T), then attn_bwd_dq_ds_kernel (dQ = dS K from dS^T) or, without
//             the dS^T buffer, attn_bwd_dq2_kernel (dQ recomputing S and dP)
// K / V / Q tiles are loaded by TMA in [rows, 64 features] 128B-swizzled panels; V (and Q, dO in the
// backward's second products) are read by the MMA as MN-major B operands, so no transpose is
// materialised.  Head sizes 64, 80, 128 (80 = two 64-wide panels, the MMAs use K = N = 80).
#include <cuda.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>
#include <stdlib.h>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace atom {
namespace atc {

constexpr int BQ = 128, BKV = 128;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_THRESHOLD = 8.f;   // log2 units

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, size % 16 == 0), completing on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
// one lane of a converged warp: tcgen05.mma under this predicate issues back to back (see gemm_tc.cu)
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// single MUFU.EX2 (exp2f adds denormal range fix-ups around it); ex2(-inf) = 0
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
// A-operand rows into TMEM: thread = lane = row, DH bf16 of `src` (or zeros) as DH / 2 columns
template <int DH>
__device__ __forceinline__ void row_to_tmem(uint32_t taddr, const bf16* src, bool valid) {
  uint32_t v[DH / 2];
#pragma unroll
  for (int c = 0; c < DH / 8; ++c) {
    const uint4 q = valid ? *(const uint4*)(src + 8 * c) : make_uint4(0, 0, 0, 0);
    v[4 * c] = q.x;
    v[4 * c + 1] = q.y;
    v[4 * c + 2] = q.z;
    v[4 * c + 3] = q.w;
  }
#pragma unroll
  for (int c = 0; c < DH / 2; c += 16) {
    if (c + 16 <= DH / 2) tmem_st16(taddr + c, v + c);
    else tmem_st8(taddr + c, v + c);
  }
}
// D[tmem] (+)= A[tmem] * B[smem]: A is M x 16 bf16 at lanes 0..M-1, 8 columns (two bf16 per
// 32-bit column, even k in the low half) -- the "TS" form of tcgen05.mma.
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// 2^x on the FMA pipe (x <= 0 finite): round-to-nearest split x = n + f, f in [-1/2, 1/2],
// minimax cubic for 2^f (max relative error 7.5e-5, below bf16's 2^-9), n added to the exponent
// field. Used for a fraction of the softmax exponentials so MUFU.EX2 is not the bottleneck.
__device__ __forceinline__ float exp2_poly(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;   // 1.5 * 2^23: n sits in the low mantissa bits of t
  const float f = x - (t - 12582912.f);
  float p = fmaf(0.05517132f, f, 0.24261054f);
  p = fmaf(p, f, 0.69326097f);
  p = fmaf(p, f, 0.99992812f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
// packed fp32 pairs (FFMA2 / FADD2 on sm_100a)
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// exp2_poly on a packed pair (same arithmetic, two lanes per instruction)
// which exponential pairs (of every 8) go to the FMA-pipe polynomial: K of them, spread evenly.
// Measured on B200 (tools/gpu_run51-53.sh, B=8 T=2048): the d_h = 80 forward is fastest with 3 of
// 8 (616 -> 631 TF/s); both backward kernels with none (2.7B 992 -> 915 us, XL 617 -> 589 us):
// their MUFU pipe is not the limit, the polynomial's extra FMA issue is
__host__ __device__ constexpr bool poly_pick(int p, int K) { return K > 0 && ((p & 7) * K) % 8 < K; }
#ifndef ATOM_BWD_POLY_KV
#define ATOM_BWD_POLY_KV 0
#endif
#ifndef ATOM_BWD_POLY_Q
#define ATOM_BWD_POLY_Q 0
#endif

__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  float x0, x1;
  f2unpack(x2, x0, x1);
  x2 = f2pack(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
  const uint64_t magic = f2pack(12582912.f, 12582912.f);
  const uint64_t t = fadd2(x2, magic);
  const uint64_t f = fsub2(x2, fsub2(t, magic));
  uint64_t p = ffma2(f2pack(0.05517132f, 0.05517132f), f, f2pack(0.24261054f, 0.24261054f));
  p = ffma2(p, f, f2pack(0.69326097f, 0.69326097f));
  p = ffma2(p, f, f2pack(0.99992812f, 0.99992812f));
  float p0, p1, t0, t1;
  f2unpack(p, p0, p1);
  f2unpack(t, t0, t1);
  return f2pack(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
                __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}

// ======================================================================================
// Forward v3: persistent, two 128-query tiles per work item, ping-pong between two softmax
// warpgroups so the tensor core works on one tile while the other tile's exponentials run.
// A work item is (b h, query pair qp): tile t covers queries [128 (2 qp + t), +128) and sees key
// blocks 0 .. 2 qp + t.  One CTA per SM walks its items (heavy-first order, dealt out in a snake
// over the CTAs: within ~2 % of a greedy schedule on the GPT-3 shapes), and the next item's
// start overlaps the current one's end: the producer loads Q_t of the next item as soon as the
// last S_t MMA of the current one has read Q_t, and the MMA issuer starts S_t(next, 0) right
// after the current item's last P_t V MMA -- so the next item's first tile runs under the other
// tile's last (unpaired, diagonal) block and both tiles' output epilogues.  (One CTA per item
// paid ~6.5 us of fill / drain per item: 30 % of the d_h = 80 forward at T = 2048.)
//   warp 0      TMA producer: per item Q0, K_0, Q1, then V_0, K_1, V_1, ... through a ring of
//               NSLOT tile slots (K_j of an item at ring position base + 2j, V_j at base + 2j + 1)
//   warp 1      MMA issuer, per key block j:  PV0(j) S0(j+1) PV1(j) S1(j+1)
//   warp 2      TMEM allocator (512 columns: S0/P0 | S1/P1 | O0 | O1)
//   warps 4-7   softmax of tile 0, warps 8-11 softmax of tile 1 (thread = query row = TMEM lane)
// P is written back into TMEM over its own S columns (bf16 pairs) and is the A operand of the
// O += P V MMA (tcgen05 "TS" form): no shared-memory round trip for P. The MMAs of one tile
// execute in issue order, so S_t(j+1) overwrites P_t(j) only after PV_t(j) has read it, and
// the commit that publishes S_t(j+1) also certifies that PV_t(j) finished (O_t is stable for
// the lazy rescale).  The first P V of an item overwrites O_t (accumulate off); it is issued
// only after the softmax warpgroup has published that item's first P, i.e. after it finished
// reading the previous item's O_t.
// ======================================================================================
template <int DH>
struct Cfg2 {
  static constexpr int NP = (DH + 63) / 64;
  static constexpr int PANEL = 128 * 128;
  static constexpr int SLOT = NP * PANEL;             // one K or V tile of 128 keys
  static constexpr int Q_BYTES = 2 * NP * PANEL;      // two query tiles
  static constexpr int NSLOT_FIT = (232448 - Q_BYTES - 2048) / SLOT;
  static constexpr int NSLOT = NSLOT_FIT > 8 ? 8 : NSLOT_FIT;
  static constexpr int SMEM = Q_BYTES + NSLOT * SLOT + 1024 + 512;
  static constexpr uint32_t S_COL = 0, O_COL = 256;  // tile t: S/P at 128t, O at 256 + 128t
  static_assert(NSLOT >= 4, "the item hand-over keeps four ring slots in flight");
};

// Work items in groups of `grp` heads (the host picks grp, fwd_group): within a group, heavy-first
// by query pair, then by head -- the items running at the same time share the K / V of a few heads
// in L2, and the lightest items of a group fill the idle tail of the CTAs.  Item i of the ordered
// list goes to CTA c in a snake deal: round r = i / G, CTA c takes the c-th (r even) or the
// (G - 1 - c)-th (r odd) item of the round.
__device__ __forceinline__ int fwd_item(int r, int c, int G) { return r * G + ((r & 1) ? G - 1 - c : c); }
struct FwdItem {
  int bh, qb0, nkb0, nkb1, nkb;
};
__host__ __device__ inline void fwd_item_pos(int i, int BH, int npair, int grp, int* bh, int* qp) {
  const int g0 = i / (grp * npair) * grp, rem = i - g0 * npair;
  const int gs = BH - g0 < grp ? BH - g0 : grp;
  *qp = npair - 1 - rem / gs;
  *bh = g0 + rem % gs;
}
__device__ __forceinline__ FwdItem fwd_decode(int i, int BH, int npair, int grp, int nkb_all, int T_) {
  FwdItem it;
  int qp;
  fwd_item_pos(i, BH, npair, grp, &it.bh, &qp);
  it.qb0 = 2 * qp;
  it.nkb0 = min(it.qb0 + 1, nkb_all);
  it.nkb1 = (it.qb0 + 1) * BQ < T_ ? min(it.qb0 + 2, nkb_all) : 0;
  it.nkb = max(it.nkb0, it.nkb1);
  return it;
}

// DROP: attention-probability dropout (R38): the P stored for P V is D(P) (one Philox call
// per 8 keys of the thread's query row), the normaliser l and the LSE keep the undropped P
template <int DH, bool DROP>
__global__ void __launch_bounds__(384, 1)
    attn_fwd3_tc_kernel(const __grid_constant__ CUtensorMap tm, bf16* __restrict__ o, float* __restrict__ lse, int T_,
                        int h, int BH, int grp, const Drop drop) {
  using C = Cfg2<DH>;
  constexpr int NS = C::NSLOT;
  (void)drop;
  // of 8 pairs on the FMA pipe: MUFU.EX2 (16/clk/SM) keeps pace with the MMAs at d_h = 128 but
  // not with the shorter MMAs of d_h = 80 / 64
#ifndef ATOM_FWD_POLY80
#define ATOM_FWD_POLY80 3
#endif
  constexpr int POLY = DH >= 128 ? 0 : (DH >= 80 ? ATOM_FWD_POLY80 : 2);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint8_t* sQ = sm;                        // tile t at + t * NP * PANEL
  uint8_t* sR = sQ + C::Q_BYTES;           // ring slot s at + s * SLOT
  uint64_t* bars = (uint64_t*)(sR + NS * C::SLOT);
  uint64_t* r_full = bars;                 // [NS]
  uint64_t* r_empty = bars + NS;           // [NS]
  uint64_t* q_full = bars + 2 * NS;        // [2]
  uint64_t* q_empty = q_full + 2;          // [2]
  uint64_t* s_full = q_empty + 2;          // [2]
  uint64_t* p_full = s_full + 2;           // [2]
  uint64_t* o_full = p_full + 2;           // [2]
  uint32_t* tmem_slot = (uint32_t*)(o_full + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npair = (T_ + 2 * BQ - 1) / (2 * BQ);
  const int n_items = npair * BH, G = gridDim.x, c = blockIdx.x;
  const int d = h * DH;
  const int nkb_all = (T_ + BKV - 1) / BKV;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&r_full[s], 1);
      mbar_init(&r_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&q_full[t], 1);
      mbar_init(&q_empty[t], 1);
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 128);
      mbar_init(&o_full[t], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp < 4) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
      int pos = 0;
      uint32_t qn[2] = {0, 0};   // Q loads per tile so far
      auto ring = [&](int col, int row) {
        const int s = pos % NS, use = pos / NS;
        mbar_wait(&r_empty[s], (use & 1) ^ 1);
        uint8_t* dst = sR + s * C::SLOT;
        mbar_expect_tx(&r_full[s], C::SLOT);
        for (int p = 0; p < C::NP; ++p) tma_load(dst + p * C::PANEL, &tm, &r_full[s], col + 64 * p, row);
        ++pos;
      };
      auto load_q = [&](int t, int col, int row) {
        mbar_wait(&q_empty[t], (qn[t] & 1) ^ 1);   // the previous item's S_t MMAs have read Q_t
        ++qn[t];
        mbar_expect_tx(&q_full[t], C::NP * C::PANEL);
        for (int p = 0; p < C::NP; ++p) tma_load(sQ + (t * C::NP + p) * C::PANEL, &tm, &q_full[t], col + 64 * p, row);
      };
      for (int r = 0;; ++r) {
        const int i = fwd_item(r, c, G);
        if (i >= n_items) break;
        const FwdItem it = fwd_decode(i, BH, npair, grp, nkb_all, T_);
        const int row0 = (it.bh / h) * T_, hh = it.bh % h;
        const int kc = d + hh * DH, vc = 2 * d + hh * DH;
        // Q0, K_0, Q1, then V_0, K_1, V_1, ...: the next item's first S needs only its Q_t and K_0
        load_q(0, hh * DH, row0 + it.qb0 * BQ);
        ring(kc, row0);
        if (it.nkb1 > 0) load_q(1, hh * DH, row0 + (it.qb0 + 1) * BQ);
        for (int j = 0; j < it.nkb; ++j) {
          ring(vc, row0 + j * BKV);
          if (j + 1 < it.nkb) ring(kc, row0 + (j + 1) * BKV);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t id_s = idesc_bf16(128, BKV, false, false);  // S = Q K^T (both K-major)
    constexpr uint32_t id_o = idesc_bf16(128, DH, false, true);    // O += P V (P in TMEM, V MN-major)
    const bool elected = elect_one();
    const uint64_t dq0 = desc_sw128(smem_u32(sQ), 16, 1024);          // Q tiles, K-major
    const uint64_t dk0 = desc_sw128(smem_u32(sR), 16, 1024);          // ring slots as K (K-major)
    const uint64_t dv0 = desc_sw128(smem_u32(sR), C::PANEL, 1024);    // ring slots as V (MN-major)
    uint32_t qc[2] = {0, 0}, pc[2] = {0, 0};   // Q tiles / P tiles consumed per tile
    auto wait_pos = [&](int pos) {
      mbar_wait(&r_full[pos % NS], (pos / NS) & 1);
      fence_after();
    };
    auto release = [&](int pos) {
      if (elected) commit(&r_empty[pos % NS]);
      __syncwarp();
    };
    auto issue_s = [&](int t, int kpos, bool last) {   // S_t = Q_t K^T, K at ring position kpos (resident)
      if (elected) {
        const uint64_t q = dq0 + (uint64_t)((t * C::NP * C::PANEL) >> 4);
        const uint64_t k = dk0 + (uint64_t)(((kpos % NS) * C::SLOT) >> 4);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * C::PANEL + (kk & 3) * 32) >> 4;
          mma(tbase + C::S_COL + 128 * t, q + off, k + off, id_s, kk > 0);
        }
        commit(&s_full[t]);
        if (last) commit(&q_empty[t]);   // Q_t may be replaced once these MMAs are done
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t, int vpos, bool first) {   // O_t (+)= P_t V, V at ring position vpos
      mbar_wait(&p_full[t], pc[t] & 1);
      ++pc[t];
      fence_after();
      if (elected) {
        const uint64_t v = dv0 + (uint64_t)(((vpos % NS) * C::SLOT) >> 4);
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          mma_ts(tbase + C::O_COL + 128 * t, tbase + C::S_COL + 128 * t + 8 * kk, v + kk * 128, id_o,
                 (!first || kk > 0) ? 1u : 0u);
      }
      __syncwarp();
    };
    // S_t(0) of an item: its Q_t and K_0 resident; K_0 released once every tile of the item has it
    int base = 0, s0_cur = 0, s0_next = 0;
    auto issue_s0 = [&](int t, const FwdItem& it, int kpos, int* done) {
      mbar_wait(&q_full[t], qc[t] & 1);
      ++qc[t];
      wait_pos(kpos);
      issue_s(t, kpos, (t ? it.nkb1 : it.nkb0) == 1);
      if (++*done == (it.nkb1 > 0 ? 2 : 1)) release(kpos);
    };
    bool pre[2] = {false, false};   // S_t(0) of the current item issued at the end of the previous one
    for (int r = 0;; ++r) {
      const int i = fwd_item(r, c, G);
      if (i >= n_items) break;
      const FwdItem it = fwd_decode(i, BH, npair, grp, nkb_all, T_);
      const int ni = fwd_item(r + 1, c, G);
      const bool has_next = ni < n_items;
      FwdItem nx = it;
      if (has_next) nx = fwd_decode(ni, BH, npair, grp, nkb_all, T_);
      const int nbase = base + 2 * it.nkb;
      s0_cur = s0_next;
      s0_next = 0;
      if (!pre[0]) issue_s0(0, it, base, &s0_cur);
      if (it.nkb1 > 0 && !pre[1]) issue_s0(1, it, base, &s0_cur);
      pre[0] = pre[1] = false;
      for (int j = 0; j < it.nkb; ++j) {
        wait_pos(base + 2 * j + 1);   // V_j
        const bool more = j + 1 < it.nkb;
        if (more) wait_pos(base + 2 * j + 2);   // K_{j+1}
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int nk = t ? it.nkb1 : it.nkb0;
          if (j < nk) {
            issue_pv(t, base + 2 * j + 1, j == 0);
            if (j + 1 < nk) {
              issue_s(t, base + 2 * j + 2, j + 2 == nk);
            } else {
              if (elected) commit(&o_full[t]);
              __syncwarp();
              // the next item's S_t(0) under this item's remaining blocks / epilogues
              if (has_next && (t == 0 || nx.nkb1 > 0)) {
                issue_s0(t, nx, nbase, &s0_next);
                pre[t] = true;
              }
            }
          }
        }
        release(base + 2 * j + 1);
        if (more) release(base + 2 * j + 2);
      }
      base = nbase;
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;\n" ::: "memory");
    // ------------------------------------------------------------ softmax, tile t
    const int t = (warp - 4) >> 2;
    const int qw = warp & 3;
    const int r = 32 * qw + lane;
    const uint32_t lane_addr = tbase + ((uint32_t)(32 * qw) << 16);
    const uint32_t s_addr = lane_addr + C::S_COL + 128 * t, o_addr = lane_addr + C::O_COL + 128 * t;
    const float sc = rsqrtf((float)DH) * LOG2E;
    uint32_t sn = 0, on = 0;   // S tiles / O results consumed
    for (int rr = 0;; ++rr) {
      const int i = fwd_item(rr, c, G);
      if (i >= n_items) break;
      const FwdItem it = fwd_decode(i, BH, npair, grp, nkb_all, T_);
      const int my_nkb = t ? it.nkb1 : it.nkb0;
      if (my_nkb == 0) continue;
      const int bh = it.bh, b = bh / h, hh = bh % h;
      const int qb = it.qb0 + t;
      const int qi = qb * BQ + r;
      float m_ref = -INFINITY, l = 0.f;
      for (int j = 0; j < my_nkb; ++j) {
        mbar_wait(&s_full[t], sn & 1);
        ++sn;
        fence_after();
        uint32_t raw[BKV];
#pragma unroll
        for (int cc = 0; cc < BKV; cc += 32) tmem_ld32(s_addr + cc, raw + cc);
        tmem_wait_ld();
        const bool masked = j == qb || (j + 1) * BKV > T_;
        if (masked) {   // keys j BKV + cc > min(qi, T_ - 1): one compare-select per score
          const int lim = min(qi, T_ - 1) - j * BKV;
#pragma unroll
          for (int cc = 0; cc < BKV; ++cc)
            if (cc > lim) raw[cc] = __float_as_uint(-INFINITY);
        }
        // row max of the raw scores (sc > 0, so max and scaling commute), four independent chains
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int cc = 0; cc < BKV; cc += 8)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            m4[q] = fmaxf(m4[q], fmaxf(__uint_as_float(raw[cc + 2 * q]), __uint_as_float(raw[cc + 2 * q + 1])));
        const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * sc;
        const bool need = mx > m_ref + RESCALE_THRESHOLD;
        const float new_ref = need ? mx : m_ref;
        const float alpha = (m_ref == -INFINITY) ? 0.f : fast_exp2(m_ref - new_ref);
        // PV_t(j-1) completed before s_full[t] fired for S_t(j): O_t is stable here
        if (__any_sync(0xffffffffu, need) && j > 0) {
#pragma unroll
          for (int cc = 0; cc < DH; cc += 16) {
            uint32_t ov[16];
            tmem_ld16(o_addr + cc, ov);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 16; ++q) ov[q] = __float_as_uint(__uint_as_float(ov[q]) * alpha);
            tmem_st16(o_addr + cc, ov);
          }
        }
        l *= alpha;
        m_ref = new_ref;
        // P = 2^(raw sc - m_ref) on packed fp32 pairs -> bf16 pairs into TMEM over S (16 columns =
        // 32 keys per store). Unmasked blocks send POLY of every 8 pairs to the FMA-pipe exponential;
        // the two variants are separate code paths (a shared, predicated loop issued both).
        const uint64_t sc2 = f2pack(sc, sc), nref2 = f2pack(-m_ref, -m_ref);
        auto p_block = [&](auto use_poly) {
          uint64_t rs2[4] = {0, 0, 0, 0};
#pragma unroll
          for (int c16 = 0; c16 < BKV / 32; ++c16) {
            uint32_t keep = 0xFFFFFFFFu;   // bit c: key j BKV + 32 c16 + c kept
            (void)keep;
            if constexpr (DROP) {
              const uint64_t g0 = ((((uint64_t)bh * T_ + qi) * T_) >> 3) + (uint64_t)(j * BKV + 32 * c16) / 8;
              keep = 0;
#pragma unroll
              for (int q = 0; q < 4; ++q) keep |= drop_keep8(drop, (uint32_t)(g0 + q)) << (8 * q);
            }
            uint32_t pk[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const int cc = c16 * 32 + 2 * q;
              const uint64_t x2 = ffma2(f2pack(__uint_as_float(raw[cc]), __uint_as_float(raw[cc + 1])), sc2, nref2);
              uint64_t p2;
              if (decltype(use_poly)::value && (q & 7) < POLY) {
                p2 = exp2_poly2(x2);
              } else {
                float x0, x1;
                f2unpack(x2, x0, x1);
                p2 = f2pack(fast_exp2(x0), fast_exp2(x1));
              }
              rs2[q & 3] = fadd2(rs2[q & 3], p2);
              float p0, p1;
              f2unpack(p2, p0, p1);
              if constexpr (DROP) {
                p0 = (keep >> (2 * q)) & 1u ? p0 * drop.scale : 0.f;
                p1 = (keep >> (2 * q + 1)) & 1u ? p1 * drop.scale : 0.f;
              }
              __nv_bfloat162 v2 = __floats2bfloat162_rn(p0, p1);
              pk[q] = *(uint32_t*)&v2;
            }
            tmem_st16(s_addr + 16 * c16, pk);
          }
          const uint64_t rsum = fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3]));
          float r0, r1;
          f2unpack(rsum, r0, r1);
          return r0 + r1;
        };
        if (POLY == 0 || masked) l += p_block(std::false_type{});
        else l += p_block(std::true_type{});
        tmem_wait_st();
        fence_before();
        mbar_arrive(&p_full[t]);
      }
      mbar_wait(&o_full[t], on & 1);
      ++on;
      fence_after();
      const float inv = 1.f / l;
      bf16* orow = o + ((long)b * T_ + qi) * d + hh * DH;
      uint32_t ov[DH];   // all loads in flight, one wait
#pragma unroll
      for (int cc = 0; cc < DH; cc += 16) tmem_ld16(o_addr + cc, ov + cc);
      tmem_wait_ld();
      if (qi < T_) {
#pragma unroll
        for (int cc = 0; cc < DH; cc += 16) {
          uint32_t pk[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            __nv_bfloat162 v2 = __floats2bfloat162_rn(__uint_as_float(ov[cc + 2 * q]) * inv,
                                                      __uint_as_float(ov[cc + 2 * q + 1]) * inv);
            pk[q] = *(uint32_t*)&v2;
          }
          *(uint4*)(orow + cc) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *(uint4*)(orow + cc + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
        lse[((long)b * h + hh) * T_ + qi] = (m_ref + log2f(l)) / LOG2E;
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

// ======================================================================================
// Backward (deterministic, no atomics), P and dS recomputed from the stashed LSE:
//   dK/dV kernel, one CTA per (b, h, 128-key block), loops over 64-query blocks i >= it:
//     S^T = K Q_i^T, dP^T = V dO_i^T (TMEM); thread = key row: P^T = exp(S^T/sqrt(dh) - lse_q),
//     dS^T = P^T (dP^T - D_q); dV += P^T dO_i, dK += dS^T Q_i (TMEM); optionally dS^T -> HBM
//   dQ kernel: dQ = dS K from that dS^T (attn_bwd_dq_ds_kernel), or, without the dS^T buffer,
//     one CTA per (b, h, 128-query block) looping over 64-key blocks j <= it:
//     S = Q K_j^T, dP = dO V_j^T; thread = query row: dS = P (dP - D); dQ += dS K_j
// D = rowsum(dO * O) comes from dsum_tc_kernel.
// ======================================================================================
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// ======================================================================================
// Recomputing dQ kernel (the path without the dS^T buffer), organised for the tensor core:
//   * dS goes back into TMEM over the S / dP columns it was computed from and feeds dQ += dS K as
//     the TMEM A operand (no smem round trip);
//   * 4-stage TMA rings for the streamed K, V tiles (a 2-stage ring left TMA latency exposed);
//   * two elementwise warpgroups, each on half of the 64 columns of a block (warps w and w+4
//     share TMEM lanes; a 64-thread named barrier per lane quarter orders their loads before
//     the in-place stores);
//   * the causal mask is applied only on the blocks that straddle the diagonal.
// Query rows beyond T_ produce values that are never stored; every result row depends only on
// its own TMEM lane.
// ======================================================================================
constexpr int BW_NST = 4;   // ring stages

template <int DH, bool TSA_ = false>
struct BCfg2 {
  static constexpr int NP = (DH + 63) / 64;
  static constexpr int P128 = 128 * 128, P64 = 64 * 128;
  static constexpr int FIX = 2 * NP * P128;          // Q, dO of the CTA's 128 queries
  static constexpr int STG = 2 * NP * P64;           // K_j, V_j: 64 rows each
  static constexpr int SMEM = FIX + BW_NST * STG + BW_NST * 2 * 64 * 4 + 1024 + 512;
  // d_h <= 80: the per-CTA fixed operands (Q, dO) live in TMEM as A operands of S / dP (TS MMAs:
  // no shared-memory A reads, which bound the SS MMAs); d_h = 128 has no TMEM room
  static constexpr bool TSA = TSA_ && DH <= 80;
  static constexpr uint32_t AL16(uint32_t x) { return (x + 15) / 16 * 16; }
  static constexpr uint32_t ST_COL = 0, DPT_COL = 64, ACC0 = 256;   // buffer u: +128u
  static constexpr uint32_t FA_COL = ACC0 + AL16(DH);               // fixed operand A (K or Q)
  static constexpr uint32_t FB_COL = FA_COL + AL16(DH / 2);         // fixed operand B (V or dO)
  static constexpr uint32_t ACC1 = TSA ? FB_COL + AL16(DH / 2) : 384;
  static_assert(!TSA || ACC1 + DH <= 512, "TMEM budget");
};

// keep bits of 32 queries (q0 .. q0 + 31) at this lane's key: the mask's 8-key Philox groups run
// along keys, but here a thread is a key row.  Lane l8 = lane % 8 of an 8-lane group (8 consecutive
// keys) draws the groups of queries l8, l8 + 8, l8 + 16, l8 + 24 (byte m of w: query l8 + 8 m, bit =
// key offset); an 8 x 8 bit-matrix transpose per byte across the group's lanes (three xor shuffles)
// leaves bit c of the result = query q0 + c at this lane's key
__device__ __forceinline__ uint32_t drop_keep_keyrow(const Drop& dr, uint64_t rowbase, int q0, int T_, int kj) {
  const int lane = threadIdx.x & 31, l8 = lane & 7;
  const uint32_t kg = (uint32_t)(kj >> 3);
  uint32_t w = 0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const uint64_t q = (uint64_t)(q0 + l8 + 8 * m);
    const uint32_t g = (uint32_t)(((rowbase + q) * (uint64_t)T_ >> 3) + kg);
    w |= drop_keep8(dr, g) << (8 * m);
  }
  const uint32_t lo[3] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu};
#pragma unroll
  for (int st = 0; st < 3; ++st) {
    const int sft = 1 << st;
    const uint32_t pv = __shfl_xor_sync(0xffffffffu, w, sft);
    if ((l8 & sft) == 0) w = (w & lo[st]) | ((pv & lo[st]) << sft);
    else w = (w & ~lo[st]) | ((pv & ~lo[st]) >> sft);
  }
  return w;
}

// ======================================================================================
// dK / dV kernel v4: the two elementwise warpgroups ping-pong over the 64-query blocks instead of
// splitting each block: warpgroup u owns TMEM buffer u (S^T | dP^T, 64 + 64 columns) and takes the
// blocks it with it % 2 == u, each thread (= key row = TMEM lane) all 64 queries of the block in
// two halves of 32.  One warpgroup's exponentials run while the other's block is on the tensor
// core, with no barrier between them (v2 split each block across both warpgroups, which had to
// meet at a named barrier before writing P^T / dS^T over the shared columns).  The MMA issuer
// keeps the in-order accumulation of dV, dK (block order; deterministic): per block it waits for
// that block's P^T / dS^T, issues dV += P^T dO and dK += dS^T Q, then S^T / dP^T of the block two
// ahead into the freed buffer.  dS^T (store_ds) leaves through a per-warp 32-key x 64-query smem
// box and a TMA store, staged at the top of the warpgroup's next block.
// ======================================================================================
#ifndef ATOM_DKV_NST
#define ATOM_DKV_NST 3
#endif
#ifndef ATOM_DKV_DSBOX
#define ATOM_DKV_DSBOX 1
#endif
constexpr int BW4_NST = ATOM_DKV_NST;   // ring stages (the dS^T staging takes the fourth one's room)
#ifdef ATOM_DKV_TRACE   // timing experiment only: per-warp clock64 stamps of the first CTAs' pipeline events
__device__ unsigned long long g_dkv_trace[8][12][64][4];
#define DKV_STAMP(it, ev)                                                                               \
  do {                                                                                                  \
    if (blockIdx.x == 0 && blockIdx.y < 8 && (threadIdx.x & 31) == 0 && (it) < 64)                      \
      g_dkv_trace[blockIdx.y][threadIdx.x >> 5][(it)][(ev)] = clock64();                                \
  } while (0)
#else
#define DKV_STAMP(it, ev) \
  do {                    \
  } while (0)
#endif
template <int DH>
struct BCfg4 {
  static constexpr int NP = (DH + 63) / 64;
  static constexpr int P128 = 128 * 128, P64 = 64 * 128;
  static constexpr int FIX = 2 * NP * P128;          // K, V of the CTA's 128 keys
  static constexpr int STG = 2 * NP * P64;           // Q_i, dO_i: 64 rows each
  static constexpr int DS_STG = ATOM_DKV_DSBOX * 8 * 32 * 128;   // per elementwise warp: 32 keys x 64 queries bf16
  static constexpr uint32_t ST_COL = 0, DPT_COL = 64, ACC0 = 256, ACC1 = 384;   // buffer u: +128u
  // d_h <= 80: K and V are also copied from shared memory into TMEM (tcgen05.cp, after the dV / dK
  // accumulators) and S^T = K Q^T, dP^T = V dO^T run as TS MMAs: an SS MMA at N = 64 reads 6 KB of
  // shared memory per 128 x 64 x 16 product and is bound by it (74 cycles, tools/tmem_bw.cu), the
  // TS form reads 2 KB (42 cycles) -- these products set this kernel's pace (clock64 trace,
  // tools/dkv_trace.py: ~1100 tensor-pipe cycles per 64-query block)
  static constexpr bool KVT = DH <= 80;
  static constexpr uint32_t FA_COL = ACC0 + (DH + 15) / 16 * 16, FB_COL = ACC1 + (DH + 15) / 16 * 16;
  static_assert(!KVT || FB_COL + DH / 2 <= 512, "TMEM budget");
  // ring stages: BW4_NST after the fixed K, V tiles; with K, V in TMEM the fixed tiles' room becomes
  // FIX / STG more stages once the copies have read it (a 3-stage ring left the TMA latency of the
  // Q / dO refill, ~1600 cycles under this kernel's dS^T stores, on the critical path)
  static constexpr int NST_X = KVT ? FIX / STG : 0;
  static constexpr int NST = BW4_NST + NST_X;
  static constexpr int SMEM = FIX + BW4_NST * STG + DS_STG + NST * 2 * 64 * 4 + 1024 + 512;
  static_assert(SMEM <= 232448, "shared memory");
};

// smem -> TMEM copy of a 128-row x 32-byte slab (16 bf16 of each row, as an MMA A-operand K step)
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

template <int DH, bool DROP>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkv4_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_do, const float* __restrict__ lse,
                         const float* __restrict__ Dsum, bf16* __restrict__ dqkv, int T_, int h, const Drop drop,
                         const bool store_ds, const __grid_constant__ CUtensorMap tm_dsw) {
  using C = BCfg4<DH>;
  constexpr int NST = C::NST;
  constexpr int POLY = DH < 128;   // the FMA-pipe share (ATOM_BWD_POLY_KV of 8 pairs) applies when the MMAs are short
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint8_t* sK = sm;
  uint8_t* sV = sK + C::NP * C::P128;
  uint8_t* sS = sm + C::FIX;                           // stage s < BW4_NST: Q at + s*STG, dO at + NP*P64
  // stage s >= BW4_NST (K, V in TMEM): in the fixed tiles' room, free once the copies have read it
  auto stage_ptr = [&](int s) { return s < BW4_NST ? sS + s * C::STG : sm + (s - BW4_NST) * C::STG; };
  uint8_t* sDS = sS + BW4_NST * C::STG;                // dS^T staging, 4 KB per elementwise warp (1024-aligned)
  float* sLD = (float*)(sDS + C::DS_STG);              // stage s: L[64] at + 128 s, D[64] at + 128 s + 64
  uint64_t* bars = (uint64_t*)(sLD + NST * 128);
  uint64_t* kv_full = bars;
  uint64_t* st_full = bars + 1;           // [NST]  TMA tx + 32 producer lanes
  uint64_t* st_empty = st_full + NST;     // [NST]
  uint64_t* s_full = st_empty + NST;      // [2]
  uint64_t* p_full = s_full + 2;          // [2]
  uint64_t* done = p_full + 2;
  uint64_t* kv_free = done + 1;           // the K, V copies into TMEM have read the fixed tiles
  uint32_t* tmem_slot = (uint32_t*)(kv_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x;
  const int bh = blockIdx.y, b = bh / h, hh = bh % h;
  const int d = h * DH;
  const int k0 = kb * 128;
  const int nq = (T_ + 63) / 64;
  const int i0 = k0 / 64;
  const int nblk = nq - i0;
  const int row0 = b * T_;

  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&st_full[s], 33);
      mbar_init(&st_empty[s], 1);
    }
    for (int u = 0; u < 2; ++u) {
      mbar_init(&s_full[u], 1);
      mbar_init(&p_full[u], 128);
    }
    mbar_init(done, 1);
    mbar_init(kv_free, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    const float* lrow = lse + ((long)b * h + hh) * T_;
    const float* drow = Dsum + ((long)b * h + hh) * T_;
    if (lane == 0) {
      mbar_expect_tx(kv_full, C::FIX);
      for (int p = 0; p < C::NP; ++p) {
        tma_load(sK + p * C::P128, &tm_kv, kv_full, d + hh * DH + 64 * p, row0 + k0);
        tma_load(sV + p * C::P128, &tm_kv, kv_full, 2 * d + hh * DH + 64 * p, row0 + k0);
      }
    }
    // the L / D values of a block (raw LSE; queries beyond T_ get L = +inf, so P and dS are exactly
    // 0): with T % 64 == 0 two 256-byte bulk copies on the stage's barrier, else this warp's lanes
    // (their global-load latency, ~900 cycles, in every stage's fill made this warp the pacer)
    const bool bulk_ld = T_ % 64 == 0;
    for (int it = 0; it < nblk; ++it) {
      const int s = it % NST, q0 = (i0 + it) * 64;
      DKV_STAMP(it, 0);
      mbar_wait(&st_empty[s], ((it / NST) & 1) ^ 1);
      if (C::NST_X > 0 && it == BW4_NST) mbar_wait(kv_free, 0);   // first use of the fixed tiles' room
      DKV_STAMP(it, 1);
      float* L = sLD + 128 * s;
      if (lane == 0) {
        uint8_t* q = stage_ptr(s);
        uint8_t* g = q + C::NP * C::P64;
        mbar_expect_tx(&st_full[s], C::STG + (bulk_ld ? 512 : 0));
        for (int p = 0; p < C::NP; ++p) {
          tma_load(q + p * C::P64, &tm_q, &st_full[s], hh * DH + 64 * p, row0 + q0);
          tma_load(g + p * C::P64, &tm_do, &st_full[s], hh * DH + 64 * p, row0 + q0);
        }
        if (bulk_ld) {
          bulk_load(L, lrow + q0, 256, &st_full[s]);
          bulk_load(L + 64, drow + q0, 256, &st_full[s]);
        }
      }
      if (!bulk_ld) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int qi = q0 + lane + 32 * e;
          L[lane + 32 * e] = qi < T_ ? lrow[qi] : INFINITY;
          L[64 + lane + 32 * e] = qi < T_ ? drow[qi] : 0.f;
        }
      }
      mbar_arrive(&st_full[s]);
      DKV_STAMP(it, 2);
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16(128, 64, false, false);   // S^T = K Q^T, dP^T = V dO^T
    constexpr uint32_t id_g = idesc_bf16(128, DH, false, true);    // dV += P^T dO, dK += dS^T Q
    mbar_wait(kv_full, 0);
    const bool elected = elect_one();
    const uint64_t dk = desc_sw128(smem_u32(sK), 16, 1024), dv = desc_sw128(smem_u32(sV), 16, 1024);
    auto ds_k = [&](int s) { return desc_sw128(smem_u32(stage_ptr(s)), 16, 1024); };       // stage tiles, K-major
    auto ds_mn = [&](int s) { return desc_sw128(smem_u32(stage_ptr(s)), C::P64, 1024); };  // stage tiles, MN-major
    if constexpr (C::KVT) {   // K, V into TMEM; executes before the MMAs issued after it
      if (elected) {
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t oa = ((kk >> 2) * C::P128 + (kk & 3) * 32) >> 4;
          tmem_cp_128x256b(tbase + C::FA_COL + 8 * kk, dk + oa);
          tmem_cp_128x256b(tbase + C::FB_COL + 8 * kk, dv + oa);
        }
        commit(kv_free);   // arrives when the copies (and nothing after them) are done
      }
      __syncwarp();
    }
    auto issue_s = [&](int it) {   // S^T / dP^T of block it into buffer it % 2
      const int s = it % NST, u = it & 1;
      mbar_wait(&st_full[s], (it / NST) & 1);
      fence_after();
      if (elected) {
        const uint64_t q = ds_k(s), g = q + ((C::NP * C::P64) >> 4);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t oa = ((kk >> 2) * C::P128 + (kk & 3) * 32) >> 4;
          const uint32_t ob = ((kk >> 2) * C::P64 + (kk & 3) * 32) >> 4;
          if constexpr (C::KVT) {
            mma_ts(tbase + C::ST_COL + 128 * u, tbase + C::FA_COL + 8 * kk, q + ob, id_s, kk > 0);
            mma_ts(tbase + C::DPT_COL + 128 * u, tbase + C::FB_COL + 8 * kk, g + ob, id_s, kk > 0);
          } else {
            mma(tbase + C::ST_COL + 128 * u, dk + oa, q + ob, id_s, kk > 0);
            mma(tbase + C::DPT_COL + 128 * u, dv + oa, g + ob, id_s, kk > 0);
          }
        }
        commit(&s_full[u]);
      }
      __syncwarp();
    };
    issue_s(0);
    if (nblk > 1) issue_s(1);
    for (int it = 0; it < nblk; ++it) {
      const int s = it % NST, u = it & 1;
      DKV_STAMP(it, 0);
      mbar_wait(&p_full[u], (it >> 1) & 1);
      DKV_STAMP(it, 1);
      fence_after();
      if (elected) {
        const uint64_t q = ds_mn(s), g = q + ((C::NP * C::P64) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {   // 64 queries = 4 x 16
          const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
          mma_ts(tbase + C::ACC0, tbase + C::ST_COL + 128 * u + 8 * kk, g + kk * 128, id_g, acc);
          mma_ts(tbase + C::ACC1, tbase + C::DPT_COL + 128 * u + 8 * kk, q + kk * 128, id_g, acc);
        }
        commit(&st_empty[s]);
        if (it == nblk - 1) commit(done);
      }
      __syncwarp();
      // buffer u is free once these products have read it (in-order execution)
      if (it + 2 < nblk) issue_s(it + 2);
      DKV_STAMP(it, 2);
    }
  } else if (warp >= 4) {
    const int wg = (warp - 4) >> 2, qw = warp & 3;
    const int r = 32 * qw + lane, kj = k0 + r;
    const uint32_t la = tbase + ((uint32_t)(32 * qw) << 16);
    const uint32_t st_col = la + C::ST_COL + 128 * wg, dp_col = la + C::DPT_COL + 128 * wg;
    const float sc = rsqrtf((float)DH) * LOG2E;
    const uint64_t sc2 = f2pack(sc, sc);
    const uint32_t box = smem_u32(sDS) + (uint32_t)(warp - 4) * 4096u;
    uint32_t pend[32];   // dS^T of the warpgroup's previous block (64 queries, bf16 pairs)
    int pend_q = -1;
    auto flush_ds = [&]() {
      if (!store_ds || pend_q < 0) return;
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      const uint32_t swz = (uint32_t)(lane & 7);   // 128B swizzle: 16-byte chunk i of row l at i ^ (l % 8)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(box + (uint32_t)lane * 128 + ((((uint32_t)i) ^ swz) << 4)),
                     "r"(pend[4 * i]), "r"(pend[4 * i + 1]), "r"(pend[4 * i + 2]), "r"(pend[4 * i + 3])
                     : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                         reinterpret_cast<uint64_t>(&tm_dsw)),
                     "r"(box), "r"(pend_q), "r"(bh * T_ + k0 + 32 * qw)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      pend_q = -1;
    };
    for (int it = wg; it < nblk; it += 2) {
      const int s = it % NST, q0 = (i0 + it) * 64;
      flush_ds();
      DKV_STAMP(it, 0);
      mbar_wait(&st_full[s], (it / NST) & 1);   // L / D of this stage visible
      DKV_STAMP(it, 1);
      mbar_wait(&s_full[wg], (it >> 1) & 1);
      DKV_STAMP(it, 2);
      fence_after();
      const bool masked = q0 < k0 + 128;   // block straddles the diagonal
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {   // queries q0 + 32 hf .. + 31
        uint32_t sv[32], dv[32];
        tmem_ld32(st_col + 32 * hf, sv);
        tmem_ld32(dp_col + 32 * hf, dv);
        tmem_wait_ld();
        const float* L = sLD + 128 * s + 32 * hf;   // raw LSE (x = s sc - L log2 e)
        const float* D = L + 64;
        const uint64_t nlog2e2 = f2pack(-LOG2E, -LOG2E);
        uint32_t pk[16], dk[16];
        uint32_t keep = 0xFFFFFFFFu;   // bit c: query q0 + 32 hf + c kept at this key
        (void)keep;
        if constexpr (DROP) keep = drop_keep_keyrow(drop, (uint64_t)bh * T_, q0 + 32 * hf, T_, kj);
        const int lim = kj - q0 - 32 * hf;   // masked block: query c of this half is visible iff c >= lim
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 l4 = *(const float4*)(L + 4 * c4);
          const float4 d4 = *(const float4*)(D + 4 * c4);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int c = 4 * c4 + 2 * h2;
            const uint64_t nl2 = fmul2(h2 ? f2pack(l4.z, l4.w) : f2pack(l4.x, l4.y), nlog2e2);
            const uint64_t d2 = h2 ? f2pack(d4.z, d4.w) : f2pack(d4.x, d4.y);
            const uint64_t x2 = ffma2(f2pack(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sc2, nl2);
            uint64_t p2;
            if (!masked && POLY && poly_pick(2 * c4 + h2, ATOM_BWD_POLY_KV)) {
              p2 = exp2_poly2(x2);
            } else {
              float x0, x1;
              f2unpack(x2, x0, x1);
              float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
              if (masked) {
                if (c < lim) p0 = 0.f;
                if (c + 1 < lim) p1 = 0.f;
              }
              p2 = f2pack(p0, p1);
            }
            float e0 = __uint_as_float(dv[c]), e1 = __uint_as_float(dv[c + 1]);
            float m0 = 1.f, m1 = 1.f;
            if constexpr (DROP) {
              m0 = (keep >> c) & 1u ? drop.scale : 0.f;
              m1 = (keep >> (c + 1)) & 1u ? drop.scale : 0.f;
              e0 *= m0;
              e1 *= m1;
            }
            const uint64_t ds2 = fmul2(p2, fsub2(f2pack(e0, e1), d2));
            float p0, p1, g0, g1;
            f2unpack(p2, p0, p1);
            f2unpack(ds2, g0, g1);
            if constexpr (DROP) {   // dV takes D(P)^T
              p0 *= m0;
              p1 *= m1;
            }
            __nv_bfloat162 a2 = __floats2bfloat162_rn(p0, p1), b2 = __floats2bfloat162_rn(g0, g1);
            pk[2 * c4 + h2] = *(uint32_t*)&a2;
            dk[2 * c4 + h2] = *(uint32_t*)&b2;
          }
        }
        // packed over this thread's own fp32 columns (read above; the other half's lie beyond)
        tmem_st16(st_col + 16 * hf, pk);
        tmem_st16(dp_col + 16 * hf, dk);
        if (store_ds) {
#pragma unroll
          for (int i = 0; i < 16; ++i) pend[16 * hf + i] = dk[i];
        }
      }
      if (store_ds) pend_q = q0;   // staged and stored at the top of this warpgroup's next block
      tmem_wait_st();
      fence_before();
      mbar_arrive(&p_full[wg]);
      DKV_STAMP(it, 3);
    }
    flush_ds();
    if (store_ds && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    mbar_wait(done, 0);
    fence_after();
    // warpgroup 0 writes dV, warpgroup 1 writes dK (scaled by 1/sqrt(dh))
    const float scale = wg ? rsqrtf((float)DH) : 1.f;
    bf16* row = dqkv + ((long)row0 + kj) * 3 * d + (wg ? d : 2 * d) + hh * DH;
    const uint32_t acc = la + (wg ? C::ACC1 : C::ACC0);
    uint32_t gv[DH];   // all loads in flight, one wait
#pragma unroll
    for (int c = 0; c < DH; c += 16) tmem_ld16(acc + c, gv + c);
    tmem_wait_ld();
    if (kj < T_) {
#pragma unroll
      for (int c = 0; c < DH; c += 16) {
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          __nv_bfloat162 v2 = __floats2bfloat162_rn(__uint_as_float(gv[c + 2 * i]) * scale,
                                                    __uint_as_float(gv[c + 2 * i + 1]) * scale);
          pk[i] = *(uint32_t*)&v2;
        }
        *(uint4*)(row + c) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *(uint4*)(row + c + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

// DROP: dS = P (D(dP) - D_row) with the forward's mask regenerated (thread = query row, natural order)
template <int DH, bool TSA, bool DROP>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq2_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                        const __grid_constant__ CUtensorMap tm_kv, const bf16* __restrict__ qkv,
                        const bf16* __restrict__ dout, const float* __restrict__ lse,
                        const float* __restrict__ Dsum, bf16* __restrict__ dqkv, int T_, int h, const Drop drop) {
  using C = BCfg2<DH, TSA>;
  constexpr int NST = BW_NST;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
  uint8_t* sQ = sm;
  uint8_t* sO = sQ + C::NP * C::P128;
  uint8_t* sS = sm + C::FIX;   // stage s: K_j at + s*STG, V_j at + NP*P64
  uint64_t* bars = (uint64_t*)(sS + NST * C::STG + NST * 512);
  uint64_t* qo_full = bars;
  uint64_t* st_full = bars + 1;           // [NST]
  uint64_t* st_empty = bars + 1 + NST;    // [NST]
  uint64_t* s_full = bars + 1 + 2 * NST;  // [2]
  uint64_t* p_full = s_full + 2;          // [2]
  uint64_t* done = p_full + 2;
  uint32_t* tmem_slot = (uint32_t*)(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (T_ + 127) / 128;
  const int qb = nqb - 1 - blockIdx.x;
  const int bh = blockIdx.y, b = bh / h, hh = bh % h;
  const int d = h * DH;
  const int q0 = qb * 128;
  const int nblk = min((q0 + 127) / 64 + 1, (T_ + 63) / 64);
  const int row0 = b * T_;

  if (threadIdx.x == 0) {
    mbar_init(qo_full, C::TSA ? 256 : 1);   // TSA: the elementwise threads store Q, dO rows into TMEM
    for (int s = 0; s < NST; ++s) {
      mbar_init(&st_full[s], 1);
      mbar_init(&st_empty[s], 1);
    }
    for (int u = 0; u < 2; ++u) {
      mbar_init(&s_full[u], 1);
      mbar_init(&p_full[u], 256);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      if (!C::TSA) {
        mbar_expect_tx(qo_full, C::FIX);
        for (int p = 0; p < C::NP; ++p) {
          tma_load(sQ + p * C::P128, &tm_q, qo_full, hh * DH + 64 * p, row0 + q0);
          tma_load(sO + p * C::P128, &tm_do, qo_full, hh * DH + 64 * p, row0 + q0);
        }
      }
      for (int j = 0; j < nblk; ++j) {
        const int s = j % NST;
        mbar_wait(&st_empty[s], ((j / NST) & 1) ^ 1);
        uint8_t* k = sS + s * C::STG;
        uint8_t* v = k + C::NP * C::P64;
        mbar_expect_tx(&st_full[s], C::STG);
        for (int p = 0; p < C::NP; ++p) {
          tma_load(k + p * C::P64, &tm_kv, &st_full[s], d + hh * DH + 64 * p, row0 + j * 64);
          tma_load(v + p * C::P64, &tm_kv, &st_full[s], 2 * d + hh * DH + 64 * p, row0 + j * 64);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16(128, 64, false, false);   // S = Q K^T, dP = dO V^T
    constexpr uint32_t id_q = idesc_bf16(128, DH, false, true);    // dQ += dS K
    mbar_wait(qo_full, 0);
    const bool elected = elect_one();
    const uint64_t dq = desc_sw128(smem_u32(sQ), 16, 1024), dg = desc_sw128(smem_u32(sO), 16, 1024);
    const uint64_t ds_k = desc_sw128(smem_u32(sS), 16, 1024);       // stage tiles, K-major
    const uint64_t ds_mn = desc_sw128(smem_u32(sS), C::P64, 1024);  // stage tiles, MN-major
    auto issue_s = [&](int j) {
      const int s = j % NST, u = j & 1;
      mbar_wait(&st_full[s], (j / NST) & 1);
      fence_after();
      if (elected) {
        const uint64_t k = ds_k + (uint64_t)((s * C::STG) >> 4), v = k + ((C::NP * C::P64) >> 4);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t oa = ((kk >> 2) * C::P128 + (kk & 3) * 32) >> 4;
          const uint32_t ob = ((kk >> 2) * C::P64 + (kk & 3) * 32) >> 4;
          if constexpr (C::TSA) {
            mma_ts(tbase + C::ST_COL + 128 * u, tbase + C::FA_COL + 8 * kk, k + ob, id_s, kk > 0);
            mma_ts(tbase + C::DPT_COL + 128 * u, tbase + C::FB_COL + 8 * kk, v + ob, id_s, kk > 0);
          } else {
            mma(tbase + C::ST_COL + 128 * u, dq + oa, k + ob, id_s, kk > 0);
            mma(tbase + C::DPT_COL + 128 * u, dg + oa, v + ob, id_s, kk > 0);
          }
        }
        commit(&s_full[u]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < nblk; ++j) {
      const int s = j % NST, u = j & 1;
      if (j + 1 < nblk) issue_s(j + 1);
      mbar_wait(&p_full[u], (j >> 1) & 1);
      fence_after();
      if (elected) {
        const uint64_t k = ds_mn + (uint64_t)((s * C::STG) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)   // 64 keys = 4 x 16
          mma_ts(tbase + C::ACC0, tbase + C::ST_COL + 128 * u + 8 * kk, k + kk * 128, id_q,
                 (j > 0 || kk > 0) ? 1u : 0u);
        commit(&st_empty[s]);
        if (j == nblk - 1) commit(done);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int wg = (warp - 4) >> 2, qw = warp & 3;
    const int r = 32 * qw + lane, qi = q0 + r;
    const uint32_t la = tbase + ((uint32_t)(32 * qw) << 16);
    const float sc = rsqrtf((float)DH) * LOG2E;
    const float L = qi < T_ ? lse[((long)b * h + hh) * T_ + qi] * LOG2E : INFINITY;
    const float Dr = qi < T_ ? Dsum[((long)b * h + hh) * T_ + qi] : 0.f;
    if constexpr (C::TSA) {   // Q row (warpgroup 0) / dO row (warpgroup 1) of this thread's query
      row_to_tmem<DH>(la + (wg ? C::FB_COL : C::FA_COL),
                      wg ? dout + ((long)row0 + qi) * d + hh * DH : qkv + ((long)row0 + qi) * 3 * d + hh * DH,
                      qi < T_);
      tmem_wait_st();
      fence_before();
      mbar_arrive(qo_full);
    }
    for (int j = 0; j < nblk; ++j) {
      const int u = j & 1;
      mbar_wait(&s_full[u], (j >> 1) & 1);
      fence_after();
      uint32_t sv[32], dv[32];
      tmem_ld32(la + C::ST_COL + 128 * u + 32 * wg, sv);
      tmem_ld32(la + C::DPT_COL + 128 * u + 32 * wg, dv);
      tmem_wait_ld();
      const int kbase = j * 64 + 32 * wg;
      const bool masked = j * 64 + 63 > q0 || (j + 1) * 64 > T_;   // diagonal or ragged keys
      uint32_t dk[16];
      const uint64_t sc2 = f2pack(sc, sc), nl2 = f2pack(-L, -L), d2 = f2pack(Dr, Dr);
      uint32_t keep = 0xFFFFFFFFu;   // bit c: key kbase + c kept
      if constexpr (DROP) {
        const uint64_t g0 = ((((uint64_t)bh * T_ + qi) * T_) >> 3) + (uint64_t)kbase / 8;
        keep = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) keep |= drop_keep8(drop, (uint32_t)(g0 + q)) << (8 * q);
      }
#pragma unroll
      for (int c2 = 0; c2 < 16; ++c2) {
        const int c = 2 * c2;
        const uint64_t x2 = ffma2(f2pack(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1])), sc2, nl2);
        uint64_t p2;
        if (!masked && poly_pick(c2, ATOM_BWD_POLY_Q)) {
          p2 = exp2_poly2(x2);
        } else {
          float x0, x1;
          f2unpack(x2, x0, x1);
          float p0 = fast_exp2(x0), p1 = fast_exp2(x1);
          if (masked) {
            if (kbase + c > qi || kbase + c >= T_) p0 = 0.f;
            if (kbase + c + 1 > qi || kbase + c + 1 >= T_) p1 = 0.f;
          }
          p2 = f2pack(p0, p1);
        }
        float e0 = __uint_as_float(dv[c]), e1 = __uint_as_float(dv[c + 1]);
        if constexpr (DROP) {
          e0 = (keep >> c) & 1u ? e0 * drop.scale : 0.f;
          e1 = (keep >> (c + 1)) & 1u ? e1 * drop.scale : 0.f;
        }
        const uint64_t ds2 = fmul2(p2, fsub2(f2pack(e0, e1), d2));
        float g0, g1;
        f2unpack(ds2, g0, g1);
        __nv_bfloat162 b2 = __floats2bfloat162_rn(g0, g1);
        dk[c2] = *(uint32_t*)&b2;
      }
      named_sync(1 + qw, 64);
      tmem_st16(la + C::ST_COL + 128 * u + 16 * wg, dk);
      tmem_wait_st();
      fence_before();
      mbar_arrive(&p_full[u]);
    }
    mbar_wait(done, 0);
    fence_after();
    // each warpgroup writes half of the dQ row
    const float isq = rsqrtf((float)DH);
    bf16* row = dqkv + ((long)row0 + qi) * 3 * d + hh * DH;
    constexpr int HALF = ((DH / 16) + 1) / 2 * 16;   // 64 / 48 / 32 columns for warpgroup 0
    auto store_cols = [&](auto lo_c, auto hi_c) {   // columns [lo, hi): loads in flight, one wait
      constexpr int LO = decltype(lo_c)::value, HI = decltype(hi_c)::value;
      uint32_t gq[HI - LO];
#pragma unroll
      for (int c = LO; c < HI; c += 16) tmem_ld16(la + C::ACC0 + c, gq + (c - LO));
      tmem_wait_ld();
      if (qi < T_) {
#pragma unroll
        for (int c = LO; c < HI; c += 16) {
          uint32_t pk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            __nv_bfloat162 q2 = __floats2bfloat162_rn(__uint_as_float(gq[c - LO + 2 * i]) * isq,
                                                      __uint_as_float(gq[c - LO + 2 * i + 1]) * isq);
            pk[i] = *(uint32_t*)&q2;
          }
          *(uint4*)(row + c) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *(uint4*)(row + c + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
    };
    if (wg) store_cols(std::integral_constant<int, HALF>{}, std::integral_constant<int, DH>{});
    else store_cols(std::integral_constant<int, 0>{}, std::integral_constant<int, HALF>{});
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512));
  }
}

// dQ = dS K from the dS^T the dK/dV kernel wrote (no recomputation of S and dP): one CTA per
// (b, h, 128-query block), key blocks of 64 up to the diagonal (entries above it are exact zeros:
// the dK/dV kernel masked P there).  A = dS [M = 128 queries, K = 64 keys] read MN-major from the
// dS^T rows (queries contiguous), B = K_j [N = d_h, K = 64 keys] MN-major, D in TMEM.
//   warp 0 TMA (dS^T box pair + K tile per stage), warp 1 MMA, warp 2 TMEM, warps 4-7 epilogue.
// Two CTAs per SM: the second CTA's stream of tiles covers the first one's prologue / epilogue.
constexpr int DQ_NST = 3;
template <int DH>
struct DqCfg {
  static constexpr int NP = (DH + 63) / 64;
  static constexpr int A_BYTES = 2 * 64 * 128;      // 128 queries x 64 keys, two 64-query panels
  static constexpr int B_BYTES = NP * 64 * 128;     // 64 keys x d_h
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int SMEM = DQ_NST * STAGE + 1024 + 256;
  static constexpr uint32_t TCOLS = DH <= 64 ? 64 : 128;
};

template <int DH>
__global__ void __launch_bounds__(256, 2)
    attn_bwd_dq_ds_kernel(const __grid_constant__ CUtensorMap tm_ds, const __grid_constant__ CUtensorMap tm_kv,
                          bf16* __restrict__ dqkv, int T_, int h) {
  using C = DqCfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = (uint64_t*)(sm + DQ_NST * C::STAGE);
  uint64_t* full = bars;               // [NST]
  uint64_t* empty = bars + DQ_NST;     // [NST]
  uint64_t* done = bars + 2 * DQ_NST;
  uint32_t* tmem_slot = (uint32_t*)(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (T_ + 127) / 128;
  const int qb = nqb - 1 - blockIdx.x;   // heavy (late) query blocks first
  const int bh = blockIdx.y, b = bh / h, hh = bh % h;
  const int d = h * DH;
  const int q0 = qb * 128;
  const int nblk = min((q0 + 127) / 64 + 1, (T_ + 63) / 64);
  const int row0 = b * T_;
  if (threadIdx.x == 0) {
    for (int s = 0; s < DQ_NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      for (int j = 0; j < nblk; ++j) {
        const int s = j % DQ_NST;
        mbar_wait(&empty[s], ((j / DQ_NST) & 1) ^ 1);
        uint8_t* a = sm + s * C::STAGE;
        uint8_t* k = a + C::A_BYTES;
        mbar_expect_tx(&full[s], C::STAGE);
        // dS^T rows j*64 .. +63 (keys) of this (b, h), queries q0 .. q0 + 127 as two 64-wide boxes
        tma_load(a, &tm_ds, &full[s], q0, bh * T_ + j * 64);
        tma_load(a + 64 * 128, &tm_ds, &full[s], q0 + 64, bh * T_ + j * 64);
        for (int p = 0; p < C::NP; ++p) tma_load(k + p * 64 * 128, &tm_kv, &full[s], d + hh * DH + 64 * p, row0 + j * 64);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_q = idesc_bf16(128, DH, true, true);   // dQ += dS K (A and B MN-major)
    const bool elected = elect_one();
    const uint64_t da0 = desc_sw128(smem_u32(sm), 64 * 128, 1024);
    const uint64_t db0 = desc_sw128(smem_u32(sm) + C::A_BYTES, 64 * 128, 1024);
    for (int j = 0; j < nblk; ++j) {
      const int s = j % DQ_NST;
      mbar_wait(&full[s], (j / DQ_NST) & 1);
      fence_after();
      if (elected) {
        const uint64_t so = (uint64_t)((s * C::STAGE) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)   // 64 keys = 4 x 16
          mma(tbase, da0 + so + kk * 128, db0 + so + kk * 128, id_q, (j > 0 || kk > 0) ? 1u : 0u);
        commit(&empty[s]);
        if (j == nblk - 1) commit(done);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int qw = warp & 3;
    const int qi = q0 + 32 * qw + lane;
    const uint32_t la = tbase + ((uint32_t)(32 * qw) << 16);
    mbar_wait(done, 0);
    fence_after();
    uint32_t gq[DH];
#pragma unroll
    for (int c = 0; c < DH; c += 16) tmem_ld16(la + c, gq + c);
    tmem_wait_ld();
    if (qi < T_) {
      const float isq = rsqrtf((float)DH);
      bf16* row = dqkv + ((long)row0 + qi) * 3 * d + hh * DH;
#pragma unroll
      for (int c = 0; c < DH; c += 16) {
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          __nv_bfloat162 q2 = __floats2bfloat162_rn(__uint_as_float(gq[c + 2 * i]) * isq,
                                                    __uint_as_float(gq[c + 2 * i + 1]) * isq);
          pk[i] = *(uint32_t*)&q2;
        }
        *(uint4*)(row + c) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        *(uint4*)(row + c + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(C::TCOLS));
  }
}

// D[b, h, t] = sum_f dO[t, h f] O[t, h f]: one thread per (token, head), 16-byte vectors;
// consecutive threads take consecutive heads of a token (contiguous bytes)
template <int DH>
__global__ void dsum_tc_kernel(const bf16* __restrict__ o, const bf16* __restrict__ dout, float* __restrict__ Dsum,
                               int B, int T_, int h) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= (long)B * T_ * h) return;
  const long row = i / h;
  const int hh = (int)(i - row * h);
  const long off = row * h * DH + hh * DH;
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < DH; c += 8) {
    const uint4 a = *(const uint4*)(o + off + c), g = *(const uint4*)(dout + off + c);
    const bf16* ap = (const bf16*)&a;
    const bf16* gp = (const bf16*)&g;
#pragma unroll
    for (int e = 0; e < 8; ++e) s = fmaf(__bfloat162float(ap[e]), __bfloat162float(gp[e]), s);
  }
  const long b = row / T_, t = row - b * T_;
  Dsum[(b * h + hh) * T_ + t] = s;
}

// Fixed MMA operands in TMEM (TS MMAs, d_h <= 80): bit 2 = the recomputing dQ kernel's Q, dO rows
// in TMEM, on by default (measured: it helps that kernel; the same form slowed the dK/dV kernel,
// and the persistent forward keeps Q in shared memory, where the next item's Q is loaded while it
// runs).  ATOM_ATTN_TSA=<mask> overrides for A/B runs.
static bool tsa_mask(int bit) {
  const char* e = getenv("ATOM_ATTN_TSA");
  const int m = e ? atoi(e) : 4;
  return (m >> bit) & 1;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled encoder() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  }
  return fn;
}

// Heads per item group of the persistent forward: among power-of-two group sizes whose K / V
// (128 padded columns x 2 B x 2 tensors per key) fit in 32 MB of L2, the one whose snake deal
// gives the smallest per-CTA maximum of (key blocks + 2.5 blocks of per-item cost) -- a host-side
// simulation of the kernel's own item order, cached per shape
static int fwd_group(int BH, int npair, int T_, int G) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, int> memo;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(BH, npair, T_, G);
  auto f = memo.find(key);
  if (f != memo.end()) return f->second;
  const int nkb_all = (T_ + BKV - 1) / BKV;
  const long n = (long)BH * npair;
  std::vector<double> load(G);
  int best = 1;
  double best_max = 1e300;
  for (int grp = 1; grp <= BH; grp *= 2) {
    if (grp > 1 && (double)grp * T_ * 512.0 > 32.0 * (1 << 20)) break;
    std::fill(load.begin(), load.end(), 0.0);
    for (long i = 0; i < n; ++i) {
      int bh, qp;
      fwd_item_pos((int)i, BH, npair, grp, &bh, &qp);
      const int nkb0 = std::min(2 * qp + 1, nkb_all);
      const int nkb1 = (2 * qp + 1) * BQ < T_ ? std::min(2 * qp + 2, nkb_all) : 0;
      const long r = i / G, c = i % G;
      load[(r & 1) ? G - 1 - c : c] += nkb0 + nkb1 + 2.5;
    }
    const double mx = *std::max_element(load.begin(), load.end());
    if (mx < best_max * 0.999) {
      best_max = mx;
      best = grp;
    }
  }
  memo[key] = best;
  return best;
}

template <int DH>
bool fwd(const bf16* qkv, bf16* o, float* lse, int B, int T_, int h, cudaStream_t st, const Drop& drop) {
  PFN_encodeTiled enc = encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  CUtensorMap tm;
  const long d = (long)h * DH;
  cuuint64_t dims[2] = {(cuuint64_t)(3 * d), (cuuint64_t)B * T_};
  cuuint64_t strides[1] = {(cuuint64_t)(3 * d) * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(qkv), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    set_error("attention: tensor map encode failed");
    return false;
  }
  if (drop.thr && T_ % 8) {
    set_error("tcgen05 attention dropout needs T %% 8 == 0 (8-key Philox groups), T = %d", T_);
    return false;
  }
  static bool once = false;
  static int sms = 0;
  if (!once) {
    ATOM_CUDA_OK(cudaFuncSetAttribute(attn_fwd3_tc_kernel<DH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cfg2<DH>::SMEM));
    ATOM_CUDA_OK(cudaFuncSetAttribute(attn_fwd3_tc_kernel<DH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cfg2<DH>::SMEM));
    int dev = 0;
    ATOM_CUDA_OK(cudaGetDevice(&dev));
    ATOM_CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    once = true;
  }
  // persistent: one CTA per SM (or per item when there are fewer items)
  const int npair = (T_ + 2 * BQ - 1) / (2 * BQ);
  const long n_items = (long)npair * B * h;
  const int grid = (int)(n_items < sms ? n_items : sms);
  if (grid == 0) return true;
  const int grp = fwd_group(B * h, npair, T_, grid);
  if (drop.thr)
    attn_fwd3_tc_kernel<DH, true><<<grid, 384, Cfg2<DH>::SMEM, st>>>(tm, o, lse, T_, h, B * h, grp, drop);
  else
    attn_fwd3_tc_kernel<DH, false><<<grid, 384, Cfg2<DH>::SMEM, st>>>(tm, o, lse, T_, h, B * h, grp, drop);
  static const std::string name = std::string("attn_fwd3<") + std::to_string(DH) + ">";
  count_launch(name.c_str());
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

static bool make_map2d(CUtensorMap* m, const bf16* base, long cols, long rows, int box_rows) {
  PFN_encodeTiled enc = encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(base), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    set_error("attention: tensor map encode failed");
    return false;
  }
  return true;
}

// st2 != NULL: the dQ kernel runs on st2 concurrently with the dK/dV kernel (independent outputs;
// each fills the SMs the other's causal tail leaves idle), joined back into st
template <int DH>
bool bwd(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, float* Dsum, bf16* dqkv, int B, int T_,
         int h, cudaStream_t st, cudaStream_t st2, const Drop& drop, bf16* dsT) {
  const long d = (long)h * DH, rows = (long)B * T_;
  CUtensorMap qkv64, qkv128, do64, do128;
  if (!make_map2d(&qkv64, qkv, 3 * d, rows, 64) || !make_map2d(&qkv128, qkv, 3 * d, rows, 128) ||
      !make_map2d(&do64, dout, d, rows, 64) || !make_map2d(&do128, dout, d, rows, 128))
    return false;
  if (drop.thr && T_ % 8) {
    set_error("tcgen05 attention dropout needs T %% 8 == 0 (8-key Philox groups), T = %d", T_);
    return false;
  }
  static bool once = false;
  static bool tsa_q = false;
  if (!once) {
#define ATOM_BWD_ATTR(K, TS, DR)                                                                                   \
  ATOM_CUDA_OK(cudaFuncSetAttribute(K<DH, TS, DR>, cudaFuncAttributeMaxDynamicSharedMemorySize, BCfg2<DH>::SMEM));
    ATOM_BWD_ATTR(attn_bwd_dq2_kernel, false, false) ATOM_BWD_ATTR(attn_bwd_dq2_kernel, true, false)
    ATOM_BWD_ATTR(attn_bwd_dq2_kernel, false, true) ATOM_BWD_ATTR(attn_bwd_dq2_kernel, true, true)
#undef ATOM_BWD_ATTR
    ATOM_CUDA_OK(cudaFuncSetAttribute(attn_bwd_dq_ds_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      DqCfg<DH>::SMEM));
    ATOM_CUDA_OK(cudaFuncSetAttribute(attn_bwd_dkv4_kernel<DH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      BCfg4<DH>::SMEM));
    ATOM_CUDA_OK(cudaFuncSetAttribute(attn_bwd_dkv4_kernel<DH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      BCfg4<DH>::SMEM));
    tsa_q = tsa_mask(2);
    once = true;
  }
  const long nthr = rows * h;
  dsum_tc_kernel<DH><<<(nthr + 255) / 256, 256, 0, st>>>(o, dout, Dsum, B, T_, h);
  count_launch("attn_dsum");
  dim3 grid((T_ + 127) / 128, B * h);
  const bool dr = drop.thr != 0;
  if (dsT && T_ % 128 == 0) {
    // dK/dV also writes dS^T; dQ = dS K over it (the dQ kernel no longer recomputes S and dP: five
    // products issued for the five the math needs instead of seven)
    CUtensorMap tm_ds;
    PFN_encodeTiled enc = encoder();
    cuuint64_t dims[2] = {(cuuint64_t)T_, (cuuint64_t)B * h * T_};
    cuuint64_t strides[1] = {(cuuint64_t)T_ * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t es[2] = {1, 1};
    CUtensorMap tm_dsw;   // the dK/dV kernel's stores: one warp's 32 keys x 64 queries per box
    cuuint32_t boxw[2] = {64, 32};
    if (!enc || enc(&tm_ds, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dsT, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        enc(&tm_dsw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dsT, dims, strides, boxw, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("attention: dS tensor map encode failed");
      return false;
    }
    if (dr)
      attn_bwd_dkv4_kernel<DH, true><<<grid, 384, BCfg4<DH>::SMEM, st>>>(qkv128, qkv64, do64, lse, Dsum, dqkv, T_, h,
                                                                       drop, true, tm_dsw);
    else
      attn_bwd_dkv4_kernel<DH, false><<<grid, 384, BCfg4<DH>::SMEM, st>>>(qkv128, qkv64, do64, lse, Dsum, dqkv, T_, h,
                                                                        drop, true, tm_dsw);
    static const std::string nkv = "attn_bwd_dkv4<" + std::to_string(DH) + ">";
    count_launch(nkv.c_str());
    attn_bwd_dq_ds_kernel<DH><<<grid, 256, DqCfg<DH>::SMEM, st>>>(tm_ds, qkv64, dqkv, T_, h);
    static const std::string nq = "attn_bwd_dq_ds<" + std::to_string(DH) + ">";
    count_launch(nq.c_str());
    ATOM_CUDA_OK(cudaGetLastError());
    return true;
  }
  // fork / join events of the dQ stream, one pair per device (peers of one process may sit on
  // different GPUs)
  static cudaEvent_t ev_fork[64] = {}, ev_join[64] = {};
  int dev = 0;
  ATOM_CUDA_OK(cudaGetDevice(&dev));
  if (st2 && dev < 64 && !ev_fork[dev]) {
    ATOM_CUDA_OK(cudaEventCreateWithFlags(&ev_fork[dev], cudaEventDisableTiming));
    ATOM_CUDA_OK(cudaEventCreateWithFlags(&ev_join[dev], cudaEventDisableTiming));
  }
  if (dev >= 64) st2 = nullptr;
  if (st2) {   // dQ's inputs (qkv, dO, LSE, D) are ready once dsum has run on st
    ATOM_CUDA_OK(cudaEventRecord(ev_fork[dev], st));
    ATOM_CUDA_OK(cudaStreamWaitEvent(st2, ev_fork[dev], 0));
  }
  const cudaStream_t sq = st2 ? st2 : st;
#define ATOM_DQ(TS, DR)                                                                                         \
  attn_bwd_dq2_kernel<DH, TS, DR><<<grid, 384, BCfg2<DH>::SMEM, sq>>>(qkv128, do128, qkv64, qkv, dout, lse, Dsum, \
                                                                       dqkv, T_, h, drop)
  if (dr)
    attn_bwd_dkv4_kernel<DH, true><<<grid, 384, BCfg4<DH>::SMEM, st>>>(qkv128, qkv64, do64, lse, Dsum, dqkv, T_, h,
                                                                     drop, false, qkv64);
  else
    attn_bwd_dkv4_kernel<DH, false><<<grid, 384, BCfg4<DH>::SMEM, st>>>(qkv128, qkv64, do64, lse, Dsum, dqkv, T_, h,
                                                                      drop, false, qkv64);
  static const std::string nkv = "attn_bwd_dkv4<" + std::to_string(DH) + ">";
  count_launch(nkv.c_str());
  if (tsa_q) { if (dr) ATOM_DQ(true, true); else ATOM_DQ(true, false); }
  else { if (dr) ATOM_DQ(false, true); else ATOM_DQ(false, false); }
#undef ATOM_DQ
  if (st2) {
    ATOM_CUDA_OK(cudaGetLastError());
    ATOM_CUDA_OK(cudaEventRecord(ev_join[dev], st2));
    ATOM_CUDA_OK(cudaStreamWaitEvent(st, ev_join[dev], 0));
  }
  static const std::string nq = "attn_bwd_dq2<" + std::to_string(DH) + ">";
  count_launch(nq.c_str());
  ATOM_CUDA_OK(cudaGetLastError());
  return true;
}

}  // namespace atc

bool attn_tc_supported(int dh, int d) { return (dh == 64 || dh == 80 || dh == 128) && ((3 * d) % 8 == 0); }

bool attn_bwd_tc(const bf16* qkv, const bf16* o, const bf16* dout, const float* lse, float* Dsum, bf16* dqkv, int B,
                 int T_, int h, int dh, cudaStream_t st, cudaStream_t st2, Drop drop, bf16* dsT) {
  switch (dh) {
    case 64: return atc::bwd<64>(qkv, o, dout, lse, Dsum, dqkv, B, T_, h, st, st2, drop, dsT);
    case 80: return atc::bwd<80>(qkv, o, dout, lse, Dsum, dqkv, B, T_, h, st, st2, drop, dsT);
    case 128: return atc::bwd<128>(qkv, o, dout, lse, Dsum, dqkv, B, T_, h, st, st2, drop, dsT);
  }
  set_error("tcgen05 attention: unsupported head size %d", dh);
  return false;
}

bool attn_fwd_tc(const bf16* qkv, bf16* o, float* lse, int B, int T_, int h, int dh, cudaStream_t st, Drop drop) {
  switch (dh) {
    case 64: return atc::fwd<64>(qkv, o, lse, B, T_, h, st, drop);
    case 80: return atc::fwd<80>(qkv, o, lse, B, T_, h, st, drop);
    case 128: return atc::fwd<128>(qkv, o, lse, B, T_, h, st, drop);
  }
  set_error("tcgen05 attention: unsupported head size %d", dh);
  return false;
}

}  // namespace atom

#ifdef ATOM_DKV_TRACE
extern "C" int atom_k_dkv_trace(void* dst) {
  return cudaMemcpyFromSymbol(dst, atom::atc::g_dkv_trace, sizeof(atom::atc::g_dkv_trace)) == cudaSuccess ? 0 : 1;
}
#endif
