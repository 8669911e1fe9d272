// The per-peer training step: swap engine + step-program interpreter + GPT-3 compute.
//
// PAPER.md §III-C/§IV: sub-models are swapped host -> device "immediately after the current
// sub-model starts" on a prefetch stream, C mini-batches run through each sub-model, the last
// forward sub-model is reused by the backward and sub-model 1 (with the embedding) stays on
// the device.  Every op of the step program (planner.cpp emit_schedule) is
// issued on its lane's CUDA stream with cross-lane waits on CUDA events:
//   compute: CAST FWD BWD FREE ADAM RECAST     h2d: LOAD_F LOAD_B     d2h: STORE     comm: AVG
// GPU AdamW updates each swapped-in segment (north star), NCCL averages masters on sync steps.
#include <string.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <string>

#include "peer.h"

using namespace atom;

namespace atom {
extern unsigned long long g_launch_count;
bool peer_flush_average(atom_peer* p);
bool peers_flush_average(atom_peer* const* ps, int n);
}

#define PEER_CUDA(expr)                                                                                      \
  do {                                                                                                       \
    cudaError_t _e = (expr);                                                                                 \
    if (_e != cudaSuccess) {                                                                                 \
      set_error("CUDA error %s at %s:%d: %s", cudaGetErrorString(_e), __FILE__, __LINE__, #expr);            \
      return false;                                                                                          \
    }                                                                                                        \
  } while (0)
#define PEER_OK(expr) \
  do {                \
    if (!(expr)) return false; \
  } while (0)

namespace {

// ------------------------------------------------------------------ layout helpers
struct SegView {
  uint8_t* W;
  float* grad;
  float* master;
  float* m;
  float* v;
};

SegView seg_view(const atom_peer* p, int k, uint8_t* base) {
  const int64_t P = p->seg_P[k - 1];
  const int64_t wbytes = al256((int64_t)p->dm.wb * P), fbytes = al256(4 * P);
  SegView s;
  s.W = base;
  s.grad = (float*)(base + wbytes);
  s.master = (float*)(base + wbytes + fbytes);
  s.m = (float*)(base + wbytes + 2 * fbytes);
  s.v = (float*)(base + wbytes + 3 * fbytes);
  return s;
}

// element offset of (node, tensor) inside its segment's sub-arrays
int64_t toff(const atom_peer* p, int node, int tensor) {
  const int k = p->seg_of_node[node];
  return p->dm.node_off[node] - p->seg_off[k - 1] + p->dm.tensors[node][tensor].off;
}
// block l's tensor t (BlockTensor) inside the sub-arrays of the segment holding it: the block's
// node, or (operator-granular graph, R40) the node of the half it belongs to
int64_t btoff(const atom_peer* p, int l, int t) {
  return toff(p, blk_tensor_node(p->dm, l, t), blk_tensor_idx(p->dm, t));
}

struct StashView {
  uint8_t *x, *qkv, *o, *x2, *u;
  float *st1, *st2, *lse;
};
StashView stash_view(const atom_peer* p, int l, int mb) {
  const ModelDims& dm = p->dm;
  const int k = p->seg_of_node[blk_node(dm, l, 0)];   // both halves in the last segment: one entry
  const int64_t ab = dm.wb, M = dm.M, d = dm.d;
  StashView s;
  uint8_t* b;
  if (p->blk_full[l]) {
    b = p->stash + p->blk_off[l] + (k == p->S ? 0 : mb) * stash_blk_bytes(dm);
    s.x = b;
  } else {
    // ACT_RECOMPUTE: the block's input checkpoint for this micro-batch; the rest of the entry
    // is the shared one the backward re-forward fills
    s.x = p->stash + p->blk_off[l] + (int64_t)mb * hfin_bytes(dm);
    b = p->stash + p->rc_off;
  }
  // the first block of the last segment reads its input from the C-deep boundary buffer
  if (p->S >= 2 && l == p->l0_last) s.x = p->hfin + (int64_t)mb * hfin_bytes(dm);
  b += al256(ab * M * d);
  s.qkv = b; b += al256(ab * M * 3 * d);
  s.o = b; b += al256(ab * M * d);
  s.x2 = b; b += al256(ab * M * d);
  s.u = b; b += al256(ab * M * 4 * d);
  s.st1 = (float*)b; b += al256(8 * M);
  s.st2 = (float*)b; b += al256(8 * M);
  s.lse = (float*)b;
  return s;
}

// input of the head for micro-batch mb: the single final-hidden buffer, or (head alone in the
// last segment) the C-deep boundary buffer filled by the previous segment
uint8_t* hfin_ptr(const atom_peer* p, int mb) {
  const int64_t hb = hfin_bytes(p->dm);
  if (p->S == 1) return p->hfin;
  if (p->nb_last == 0) return p->hfin + (int64_t)mb * hb;
  return p->hfin + (int64_t)p->C * hb;
}

// scratch sub-buffers (union of block scratch and head scratch; planner work_bytes)
struct Scratch {
  uint8_t *G, *A, *DA, *DX2, *DO;
  float* Dsum;
  uint8_t *G2, *dsT;
  uint8_t *logits, *z, *dz;
  float* hst;
};
Scratch scratch_view(const atom_peer* p) {
  const int64_t ab = p->dm.wb, M = p->dm.M, d = p->dm.d;
  Scratch s;
  uint8_t* b = p->scratch;
  s.G = b; b += al256(ab * M * 4 * d);
  s.A = b; b += al256(ab * M * d);
  s.DA = b; b += al256(ab * M * d);
  s.DX2 = b; b += al256(ab * M * d);
  s.DO = b; b += al256(ab * M * d);
  s.Dsum = (float*)b;
  b += al256(4LL * p->dm.b * p->dm.h * p->dm.T);
  s.G2 = b;                                           // [M, 4d]: dL/du while G holds GELU(u)
  b += al256(ab * M * 4 * d);
  s.dsT = p->dm.dtype == ATOM_BF16 ? b : nullptr;   // [b h][T keys][T queries] bf16
  b = p->scratch;
  s.logits = b; b += al256(ab * M * al(p->dm.V, 8));
  s.z = b; b += al256(ab * M * d);
  s.dz = b; b += al256(ab * M * d);
  s.hst = (float*)b;
  return s;
}

// ------------------------------------------------------------------ per-category kernel timing
// (timing on: CUDA events around each launch group on its stream; atom_get_kernel_log)
enum KCat { KC_GEMM_F, KC_GEMM_D, KC_GEMM_W, KC_ATTN_F, KC_ATTN_B, KC_LN, KC_COLSUM, KC_GELU, KC_CE, KC_EMBED,
            KC_ADAM, KC_CAST, KC_N };
const char* kcat_name(int c) {
  static const char* n[KC_N] = {"gemm_fwd", "gemm_dgrad", "gemm_wgrad", "attn_fwd", "attn_bwd", "layernorm",
                                "colsum", "gelu", "cross_entropy", "embedding", "adamw", "cast"};
  return c >= 0 && c < KC_N ? n[c] : "?";
}
bool kt_mark(atom_peer* p, int cat, cudaStream_t st, bool end) {
  if (p->timing < 2) return true;   // per-category events only at timing level 2 (they cost step time)
  const size_t i = end ? 2 * (p->kt_n - 1) + 1 : 2 * p->kt_n;
  if (!end) {
    while (p->kt_ev.size() < 2 * (p->kt_n + 1)) {
      cudaEvent_t ev;
      PEER_CUDA(cudaEventCreate(&ev));
      p->kt_ev.push_back(ev);
    }
    if (p->kt_cat.size() < p->kt_n + 1) p->kt_cat.resize(p->kt_n + 1);
    p->kt_cat[p->kt_n] = cat;
    p->kt_n++;
  }
  PEER_CUDA(cudaEventRecord(p->kt_ev[i], st ? st : p->s_comp));
  return true;
}
#define KT(cat, st, expr)                  \
  do {                                     \
    PEER_OK(kt_mark(p, cat, st, false));   \
    PEER_OK(expr);                         \
    PEER_OK(kt_mark(p, cat, st, true));    \
  } while (0)

// ------------------------------------------------------------------ compute dispatch
template <typename T>
bool gemm(atom_peer* p, int M, int N, int K, const T* A, long lda, bool a_mn, const T* B, long ldb, bool b_mn,
          const Epi& e, cudaStream_t stream = nullptr) {
  const cudaStream_t st = stream ? stream : p->s_comp;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (p->timing) {
    while (p->gemm_ev.size() < 2 * (p->gemm_n + 1)) {
      cudaEvent_t ev;
      PEER_CUDA(cudaEventCreate(&ev));
      p->gemm_ev.push_back(ev);
    }
    e0 = p->gemm_ev[2 * p->gemm_n];
    e1 = p->gemm_ev[2 * p->gemm_n + 1];
    PEER_CUDA(cudaEventRecord(e0, st));
  }
  bool ok;
  const int cat = a_mn ? KC_GEMM_W : (b_mn ? KC_GEMM_D : KC_GEMM_F);
  PEER_OK(kt_mark(p, cat, st, false));
  if constexpr (std::is_same<T, bf16>::value)
    ok = gemm_tc(M, N, K, A, lda, a_mn, B, ldb, b_mn, e, st);
  else
    ok = gemm_simt<T>(M, N, K, A, lda, a_mn, B, ldb, b_mn, e, st);
  if (!ok) return false;
  PEER_OK(kt_mark(p, cat, st, true));
  p->gemm_launches++;
  if (p->timing) {
    PEER_CUDA(cudaEventRecord(e1, st));
    if (p->gemm_fl.size() < p->gemm_n + 1) p->gemm_fl.resize(p->gemm_n + 1);
    if (p->gemm_key.size() < p->gemm_n + 1) p->gemm_key.resize(p->gemm_n + 1);
    p->gemm_fl[p->gemm_n] = 2.0 * M * N * (double)K;
    char key[96];
    snprintf(key, sizeof key, "%d %d %d %d %d %d", M, N, K, (int)a_mn, (int)b_mn, e.mode);
    p->gemm_key[p->gemm_n] = key;
    p->gemm_n++;
  }
  return true;
}

// attention-probability dropout (site DS_ATTN) runs inside the tcgen05 and SIMT kernels; the
// mma.sync kernels (d_h = 16) have none: peer creation rejects that combination
template <typename T>
bool attn_fwd(atom_peer* p, const T* qkv, T* o, float* lse, const Drop& dr) {
  const ModelDims& dm = p->dm;
  const int dh = dm.d / dm.h;
  if constexpr (std::is_same<T, bf16>::value) {
    if (attn_tc_supported(dh, dm.d)) return attn_fwd_tc(qkv, o, lse, dm.b, dm.T, dm.h, dh, p->s_comp, dr);
    if (attn_fa_supported(dh)) return attn_fwd_fa(qkv, o, lse, dm.b, dm.T, dm.h, dh, p->s_comp);
  }
  return attn_fwd_simt<T>(qkv, o, lse, dm.b, dm.T, dm.h, dh, p->s_comp, dr);
}
template <typename T>
bool attn_bwd(atom_peer* p, const T* qkv, const T* o, const T* dout, const float* lse, float* Dsum, T* dqkv,
              const Drop& dr) {
  const ModelDims& dm = p->dm;
  const int dh = dm.d / dm.h;
  if constexpr (std::is_same<T, bf16>::value) {
    if (attn_tc_supported(dh, dm.d))
      return attn_bwd_tc(qkv, o, dout, lse, Dsum, dqkv, dm.b, dm.T, dm.h, dh, p->s_comp,
                         p->side_wgrad ? p->s_attn : nullptr, dr, (bf16*)scratch_view(p).dsT);
    if (attn_fa_supported(dh)) return attn_bwd_fa(qkv, o, dout, lse, Dsum, dqkv, dm.b, dm.T, dm.h, dh, p->s_comp);
  }
  return attn_bwd_simt<T>(qkv, o, dout, lse, Dsum, dqkv, dm.b, dm.T, dm.h, dh, p->s_comp, dr);
}

// one dropout site of micro-batch mb of this step (R38); thr = 0 when the model has none
Drop mkdrop(const atom_peer* p, uint32_t site, int layer, int mb) {
  Drop d;
  const double pr = p->cfg.dropout_p;
  if (pr <= 0.0) return d;
  d.thr = (uint32_t)floor(pr * 65536.0);
  d.scale = (float)(1.0 / (1.0 - pr));
  d.site = site;
  d.layer = (uint32_t)layer;
  d.step = (uint32_t)(p->rng_step * p->C + mb);
  d.k0 = (uint32_t)p->cfg.dropout_seed;
  d.k1 = (uint32_t)(p->cfg.dropout_seed >> 32);
  return d;
}

Epi epi(int mode, void* out, long ldo) {
  Epi e;
  e.mode = mode;
  e.out = out;
  e.ldo = ldo;
  return e;
}

// forward of block l on micro-batch mb (minGPT Block).  part 0: the whole block; in the
// operator-granular graph (R40) the attention half (part 1: LN1, QKV, attention, output projection
// into the stash's x2) and the MLP half (part 2: LN2 with the residual, fc, GELU, fc2) are separate
// nodes, possibly of different sub-models (the stash entry carries x and x2 between them)
template <typename T>
bool fwd_block(atom_peer* p, int l, int mb, const SegView& sv, int part = 0) {
  const ModelDims& dm = p->dm;
  const long M = dm.M, d = dm.d;
  const T* W = (const T*)sv.W;
  auto w = [&](int t) { return W + btoff(p, l, t); };
  StashView s = stash_view(p, l, mb);
  Scratch sc = scratch_view(p);
  T* x = (T*)s.x;
  Epi e;
  if (part != 2) {
  KT(KC_LN, p->s_comp, ln_fwd<T>(x, w(T_LN1G), w(T_LN1B), (T*)sc.A, s.st1, M, d, p->s_comp));
  e = epi(EPI_BIAS, s.qkv, 3 * d);
  e.bias = w(T_BQKV);
  PEER_OK(gemm<T>(p, M, 3 * d, d, (const T*)sc.A, d, false, w(T_WQKV), d, false, e));
  KT(KC_ATTN_F, p->s_comp, attn_fwd<T>(p, (const T*)s.qkv, (T*)s.o, s.lse, mkdrop(p, DS_ATTN, l, mb)));
  // x2 = x + D(o W_o^T + b_o): the GEMM stores o W_o^T + b_o (plain epilogue), LN2 applies the
  // residual dropout and adds the residual (a per-row residual read in the GEMM epilogue held this
  // K = d GEMM well below the others)
  e = epi(EPI_BIAS, s.x2, d);
  e.bias = w(T_BO);
  PEER_OK(gemm<T>(p, M, d, d, (const T*)s.o, d, false, w(T_WO), d, false, e));
  }
  if (part == 1) return true;
  KT(KC_LN, p->s_comp, ln_fwd<T>((const T*)s.x2, w(T_LN2G), w(T_LN2B), (T*)sc.A, s.st2, M, d, p->s_comp, x,
                                 mkdrop(p, DS_RESID_ATTN, l, mb)));
  e = epi(EPI_BIAS_GELU, s.u, 4 * d);
  e.bias = w(T_BFC);
  e.out2 = sc.G;
  e.ldo2 = 4 * d;
  PEER_OK(gemm<T>(p, M, 4 * d, d, (const T*)sc.A, d, false, w(T_WFC), d, false, e));
  void* out = (l + 1 < dm.L) ? (void*)stash_view(p, l + 1, mb).x : (void*)hfin_ptr(p, mb);
  const Drop d3 = mkdrop(p, DS_RESID_MLP, l, mb);
  e = epi(d3.thr ? EPI_BIAS : EPI_BIAS_RES, out, d);
  e.bias = w(T_BPR);
  e.res = s.x2;
  e.ldr = d;
  PEER_OK(gemm<T>(p, M, d, 4 * d, (const T*)sc.G, 4 * d, false, w(T_WPR), 4 * d, false, e));
  // with dropout: h = x2 + D(fc2 output) in one pass over the block output
  if (d3.thr) KT(KC_COLSUM, p->s_comp, dropout_add<T>((T*)out, (const T*)s.x2, M * d, d3, p->s_comp));
  return true;
}

// backward of block l on micro-batch mb: dh[mb] (grad of the block output) -> dh[mb] (grad of its input).
// part 0: the whole block; operator-granular graph (R40): part 2 = the MLP half (up to LN2's
// backward, which yields DX2 = dL/dx2), then part 1 = the attention half.  When the halves sit in
// different sub-models (their backward ops run at different times) DX2 travels in dh[mb] (LN2's
// backward writes it over dy in place, LN1's backward writes dL/dx over it in place) and each half
// drains the side stream that read its scratch buffers before it returns.
template <typename T>
bool bwd_block(atom_peer* p, int l, int mb, const SegView& sv, int part = 0) {
  const ModelDims& dm = p->dm;
  const long M = dm.M, d = dm.d;
  const T* W = (const T*)sv.W;
  auto w = [&](int t) { return W + btoff(p, l, t); };
  auto g = [&](int t) { return sv.grad + btoff(p, l, t); };
  StashView s = stash_view(p, l, mb);
  Scratch sc = scratch_view(p);
  T* dy = (T*)(p->dh + (int64_t)mb * M * d * dm.wb);
  T* G = (T*)sc.G;
  const bool rc = !p->blk_full[l];   // never in the operator-granular graph (stash only)
  const bool split = part != 0 && p->seg_of_node[blk_node(dm, l, 0)] != p->seg_of_node[blk_node(dm, l, 1)];
  T* dx2 = split ? dy : (T*)sc.DX2;   // dL/dx2 from LN2's backward to the attention half
  // LN outputs the weight gradients read: re-applied from the stash, or (recompute) kept from the
  // re-run forward -- LN1(x) in A, LN2(x2) in DA (free until the fc data-gradient GEMM)
  T* ln1 = (T*)sc.A;
  T* ln2 = rc ? (T*)sc.DA : (T*)sc.A;
  const Drop d3 = mkdrop(p, DS_RESID_MLP, l, mb), d2 = mkdrop(p, DS_RESID_ATTN, l, mb);
  // Weight-gradient GEMMs that nothing later in the block reads run on the side stream (fork after
  // their inputs exist; the main stream waits before overwriting what they read). Buffers: WFC's
  // LN2 output (A under stash) is rewritten by LN1's re-apply after the attention backward, which
  // also rewrites G; WO reads DX2 / o, WQKV reads G / A; the next block rewrites G, A, DX2.
  const bool side = p->side_wgrad;
  // MLP projection: out = x2 + D3(GELU(u) W_pr^T + b_pr).  Its weight gradient reads GELU(u) in G
  // and dy: on the side stream when the fc pre-activation gradient goes to the second buffer G2
  // (so nothing on the main stream rewrites G or dy before the join ahead of the attention
  // backward); on the main stream with dropout (dym lives in DX2), under the re-forward (no
  // join there) and for a split block (dy is rewritten in place by LN2's backward)
  const bool wpr_side = side && !rc && !d3.thr && !split;
  const cudaStream_t sd = side ? p->s_side : p->s_comp;
  auto fork = [&]() -> bool {
    if (side) {
      PEER_CUDA(cudaEventRecord(p->ev_side[0], p->s_comp));
      PEER_CUDA(cudaStreamWaitEvent(p->s_side, p->ev_side[0], 0));
    }
    return true;
  };
  auto mark = [&](int i) -> bool {
    if (side) PEER_CUDA(cudaEventRecord(p->ev_side[i], p->s_side));
    return true;
  };
  auto join = [&](int i) -> bool {
    if (side) PEER_CUDA(cudaStreamWaitEvent(p->s_comp, p->ev_side[i], 0));
    return true;
  };
  if (part != 1) {
  if (rc) {
    // ACT_RECOMPUTE: re-run the block forward from its input checkpoint into the shared entry
    // (same kernels and inputs as the forward: bit-identical tensors); the MLP projection's
    // output is not needed by the backward and is skipped
    KT(KC_LN, p->s_comp, ln_fwd<T>((const T*)s.x, w(T_LN1G), w(T_LN1B), ln1, s.st1, M, d, p->s_comp));
    Epi e = epi(EPI_BIAS, s.qkv, 3 * d);
    e.bias = w(T_BQKV);
    PEER_OK(gemm<T>(p, M, 3 * d, d, (const T*)sc.A, d, false, w(T_WQKV), d, false, e));
    KT(KC_ATTN_F, p->s_comp, attn_fwd<T>(p, (const T*)s.qkv, (T*)s.o, s.lse, mkdrop(p, DS_ATTN, l, mb)));
    e = epi(EPI_BIAS, s.x2, d);
    e.bias = w(T_BO);
    PEER_OK(gemm<T>(p, M, d, d, (const T*)s.o, d, false, w(T_WO), d, false, e));
    KT(KC_LN, p->s_comp, ln_fwd<T>((const T*)s.x2, w(T_LN2G), w(T_LN2B), ln2, s.st2, M, d, p->s_comp, (const T*)s.x,
                                   mkdrop(p, DS_RESID_ATTN, l, mb)));
    e = epi(EPI_BIAS_GELU, s.u, 4 * d);   // u and GELU(u) in one pass, as in the forward
    e.bias = w(T_BFC);
    e.out2 = G;
    e.ldo2 = 4 * d;
    PEER_OK(gemm<T>(p, M, 4 * d, d, (const T*)ln2, d, false, w(T_WFC), d, false, e));
  } else if (!wpr_side) {
    KT(KC_GELU, p->s_comp, gelu_apply<T>((const T*)s.u, G, M * 4 * d, p->s_comp));
  }
  // residual dropout (R38): the projections' branches see the masked gradients
  // D3(dy) (MLP, in DX2 until LN2's backward rewrites it) and D2(DX2) (attention, in DA until the
  // QKV data gradient rewrites it); the residual paths keep the unmasked ones
  const T* dym = dy;
  if (d3.thr) {
    KT(KC_COLSUM, p->s_comp, dropout<T>(dy, (T*)sc.DX2, M * d, d3, p->s_comp));
    dym = (const T*)sc.DX2;
  }
  T* Gx = wpr_side ? (T*)sc.G2 : G;   // dL/du
  if (!wpr_side)
    PEER_OK(gemm<T>(p, d, 4 * d, M, dym, d, true, G, 4 * d, true, epi(EPI_ACC_F32, g(T_WPR), 4 * d), p->s_comp));
  KT(KC_COLSUM, p->s_comp, bias_grad<T>(dym, d, M, d, g(T_BPR), p->red, p->red_ticket, p->s_comp));
  // fc pre-activation gradient: (dy W_pr) with a plain-store epilogue, then the GELU derivative
  // and the fc bias gradient in one pass over it (the GEMM epilogue reading u per row was the
  // slow part of the fused form).  With W_pr's gradient on the side stream the same pass also
  // re-applies GELU(u) into G (one read of u instead of two), and that gradient starts after it
  PEER_OK(gemm<T>(p, M, 4 * d, d, dym, d, false, w(T_WPR), 4 * d, true, epi(EPI_STORE, Gx, 4 * d)));
  KT(KC_COLSUM, p->s_comp, dgelu_bias_grad<T>(Gx, (const T*)s.u, M, 4 * d, g(T_BFC), p->red, p->red_ticket, p->s_comp,
                                              wpr_side ? G : nullptr));
  if (wpr_side) {
    PEER_OK(fork());
    PEER_OK(gemm<T>(p, d, 4 * d, M, dym, d, true, G, 4 * d, true, epi(EPI_ACC_F32, g(T_WPR), 4 * d), sd));
  }
  // MLP fc: u = LN2(x2) W_fc^T + b_fc (under recompute LN2's output is DA, rewritten just below:
  // that gradient stays on the main stream)
  if (!rc) KT(KC_LN, p->s_comp, ln_apply<T>((const T*)s.x2, w(T_LN2G), w(T_LN2B), s.st2, ln2, M, d, p->s_comp));
  if (!rc) PEER_OK(fork());
  PEER_OK(gemm<T>(p, 4 * d, d, M, Gx, 4 * d, true, (const T*)ln2, d, true, epi(EPI_ACC_F32, g(T_WFC), d),
                  rc ? p->s_comp : sd));
  if (!rc) PEER_OK(mark(1));
  PEER_OK(gemm<T>(p, M, d, 4 * d, Gx, 4 * d, false, w(T_WFC), d, true, epi(EPI_STORE, sc.DA, d)));
  KT(KC_LN, p->s_comp, ln_bwd<T>((const T*)sc.DA, (const T*)s.x2, s.st2, w(T_LN2G), dy, dx2, g(T_LN2G), g(T_LN2B), p->red,
                    p->red_ticket, M, d, p->s_comp));
  // the attention half runs in another op: the W_fc gradient has read G / LN2's output by then
  if (split) PEER_OK(join(1));
  }
  if (part == 2) return true;
  // attention projection: x2 = x + D2(o W_o^T + b_o)
  const T* dx2m = dx2;
  if (d2.thr) {
    KT(KC_COLSUM, p->s_comp, dropout<T>((const T*)dx2, (T*)sc.DA, M * d, d2, p->s_comp));
    dx2m = (const T*)sc.DA;
  }
  PEER_OK(fork());
  PEER_OK(gemm<T>(p, d, d, M, dx2m, d, true, (const T*)s.o, d, true, epi(EPI_ACC_F32, g(T_WO), d), sd));
  PEER_OK(mark(2));
  KT(KC_COLSUM, p->s_comp, bias_grad<T>(dx2m, d, M, d, g(T_BO), p->red, p->red_ticket, p->s_comp));
  PEER_OK(gemm<T>(p, M, d, d, dx2m, d, false, w(T_WO), d, true, epi(EPI_STORE, sc.DO, d)));
  // attention (writes G, which the fc weight gradient reads)
  if (!rc) PEER_OK(join(1));
  KT(KC_ATTN_B, p->s_comp, attn_bwd<T>(p, (const T*)s.qkv, (const T*)s.o, (const T*)sc.DO, s.lse, sc.Dsum, G,
                                       mkdrop(p, DS_ATTN, l, mb)));
  // QKV: qkv = LN1(x) W_qkv^T + b_qkv
  if (!rc) KT(KC_LN, p->s_comp, ln_apply<T>((const T*)s.x, w(T_LN1G), w(T_LN1B), s.st1, ln1, M, d, p->s_comp));
  PEER_OK(fork());
  PEER_OK(gemm<T>(p, 3 * d, d, M, G, 3 * d, true, (const T*)ln1, d, true, epi(EPI_ACC_F32, g(T_WQKV), d), sd));
  PEER_OK(mark(3));
  KT(KC_COLSUM, p->s_comp, bias_grad<T>(G, 3 * d, M, 3 * d, g(T_BQKV), p->red, p->red_ticket, p->s_comp));
  if (d2.thr) PEER_OK(join(2));   // the side stream's W_o gradient has read D2(DX2) from DA
  PEER_OK(gemm<T>(p, M, d, 3 * d, G, 3 * d, false, w(T_WQKV), d, true, epi(EPI_STORE, sc.DA, d)));
  if (split && !d2.thr) PEER_OK(join(2));   // W_o's gradient has read DX2 from dh[mb], rewritten next
  KT(KC_LN, p->s_comp, ln_bwd<T>((const T*)sc.DA, (const T*)s.x, s.st1, w(T_LN1G), (const T*)dx2, dy, g(T_LN1G), g(T_LN1B),
                    p->red, p->red_ticket, M, d, p->s_comp));
  // the side stream is in order: its last mark covers WO and WQKV (and WFC)
  PEER_OK(join(3));
  return true;
}

// head on micro-batch mb: ln_f, lm_head, cross-entropy and their backward (interleaved)
template <typename T>
bool head(atom_peer* p, int mb, const SegView& sv) {
  const ModelDims& dm = p->dm;
  const int node = dm.n_nodes - 1;
  const long M = dm.M, d = dm.d, V = dm.V, Vp = al(dm.V, 8);
  const T* W = (const T*)sv.W;
  auto w = [&](int t) { return W + toff(p, node, t); };
  auto g = [&](int t) { return sv.grad + toff(p, node, t); };
  Scratch sc = scratch_view(p);
  const T* h = (const T*)hfin_ptr(p, mb);
  KT(KC_LN, p->s_comp, ln_fwd<T>(h, w(T_LNFG), w(T_LNFB), (T*)sc.z, sc.hst, M, d, p->s_comp));
  PEER_OK(gemm<T>(p, M, V, d, (const T*)sc.z, d, false, w(T_WLM), d, false, epi(EPI_STORE, sc.logits, Vp)));
  const int32_t* tgt = p->tokens + (int64_t)mb * dm.b * (dm.T + 1) + 1;
  KT(KC_CE, p->s_comp, cross_entropy<T>((T*)sc.logits, Vp, V, tgt, dm.T + 1, dm.T, M, 1.f / (float)((double)p->C * M),
                           p->losses + (int64_t)mb * M, p->s_comp));
  PEER_OK(gemm<T>(p, M, d, V, (const T*)sc.logits, Vp, false, w(T_WLM), d, true, epi(EPI_STORE, sc.dz, d)));
  PEER_OK(gemm<T>(p, V, d, M, (const T*)sc.logits, Vp, true, (const T*)sc.z, d, true, epi(EPI_ACC_F32, g(T_WLM), d)));
  T* dout = (T*)(p->dh + (int64_t)mb * M * d * dm.wb);
  KT(KC_LN, p->s_comp, ln_bwd<T>((const T*)sc.dz, h, sc.hst, w(T_LNFG), nullptr, dout, g(T_LNFG), g(T_LNFB), p->red,
                    p->red_ticket, M, d, p->s_comp));
  return true;
}

template <typename T>
bool embed_forward(atom_peer* p, int mb, const SegView& sv) {
  const ModelDims& dm = p->dm;
  const T* W = (const T*)sv.W;
  const int32_t* tok = p->tokens + (int64_t)mb * dm.b * (dm.T + 1);
  T* x0 = (T*)stash_view(p, 0, mb).x;
  PEER_OK(embed_fwd<T>(tok, dm.T + 1, dm.T, dm.M, W + toff(p, 0, T_WTE), W + toff(p, 0, T_WPE), x0, dm.d, p->s_comp));
  const Drop d0 = mkdrop(p, DS_EMBD, 0, mb);   // h0 = D(wte[x] + wpe[t])
  if (d0.thr) PEER_OK(dropout<T>(x0, x0, dm.M * dm.d, d0, p->s_comp));
  return true;
}
template <typename T>
bool embed_backward(atom_peer* p, int mb, const SegView& sv) {
  const ModelDims& dm = p->dm;
  const int32_t* tok = p->tokens + (int64_t)mb * dm.b * (dm.T + 1);
  const T* dh = (const T*)(p->dh + (int64_t)mb * dm.M * dm.d * dm.wb);
  const Drop d0 = mkdrop(p, DS_EMBD, 0, mb);   // the embedding sees D(dh0); dh0 is dead after this
  if (d0.thr) PEER_OK(dropout<T>(dh, (T*)dh, dm.M * dm.d, d0, p->s_comp));
  return embed_bwd<T>(tok, dm.T + 1, dm.T, dm.b, dh, dm.V, dm.d, sv.grad + toff(p, 0, T_WTE),
                      sv.grad + toff(p, 0, T_WPE), p->emb, p->s_comp);
}

// deferred CAST (layer-by-layer loading): wait for node's copy, derive its compute weights
template <typename T>
bool cast_node(atom_peer* p, int k, int node, const SegView& sv) {
  const int64_t off = p->dm.node_off[node] - p->seg_off[k - 1];
  PEER_CUDA(cudaStreamWaitEvent(p->s_comp, p->node_ev[node], 0));
  KT(KC_CAST, p->s_comp, cast_params<T>(sv.master + off, (T*)sv.W + off, p->dm.P[node], p->s_comp));
  return true;
}

template <typename T>
bool run_fwd(atom_peer* p, int k, int mb, const SegView& sv) {
  // the gradient buffer starts each step at zero; under gradient rounds (R37) only the first round
  // of an update starts at zero, later rounds continue the running sum (resident sub-model 1: kept
  // on the device; sub-models 2..S: loaded from the host sum with the master)
  if (k == p->S && mb == 0 && p->round == 0) PEER_CUDA(cudaMemsetAsync(sv.grad, 0, 4 * p->seg_P[k - 1], p->s_comp));
  const bool cast = p->cast_pending[k - 1];
  p->cast_pending[k - 1] = 0;
  for (int node = p->seg_lo[k - 1]; node <= p->seg_hi[k - 1]; ++node) {
    if (cast) PEER_OK(cast_node<T>(p, k, node, sv));
    if (node == 0)
      KT(KC_EMBED, p->s_comp, embed_forward<T>(p, mb, sv));
    else if (is_block_node(p->dm, node))
      PEER_OK(fwd_block<T>(p, node_block(p->dm, node), mb, sv, node_half(p->dm, node)));
    else
      PEER_OK(head<T>(p, mb, sv));
  }
  return true;
}
template <typename T>
bool run_bwd(atom_peer* p, int k, int mb, const SegView& sv) {
  if (k < p->S && mb == 0 && p->round == 0) PEER_CUDA(cudaMemsetAsync(sv.grad, 0, 4 * p->seg_P[k - 1], p->s_comp));
  const bool cast = p->cast_pending[k - 1];
  p->cast_pending[k - 1] = 0;
  for (int node = p->seg_hi[k - 1]; node >= p->seg_lo[k - 1]; --node) {
    if (cast) PEER_OK(cast_node<T>(p, k, node, sv));
    if (node == 0)
      KT(KC_EMBED, p->s_comp, embed_backward<T>(p, mb, sv));
    else if (is_block_node(p->dm, node))
      PEER_OK(bwd_block<T>(p, node_block(p->dm, node), mb, sv, node_half(p->dm, node)));
    // the head's backward ran inside its forward op
  }
  return true;
}

// ------------------------------------------------------------------ op interpreter
cudaStream_t lane_stream(atom_peer* p, int lane) {
  switch (lane) {
    case L_H2D: return p->s_h2d;
    case L_D2H: return p->s_d2h;
    case L_COMM: return p->s_comm;
    default: return p->s_comp;
  }
}

bool copy_seg(atom_peer* p, int k, float* dev, float* host, bool h2d) {
  // one copy per layer (node) of the segment (P:263 layer loading; event per op)
  for (int node = p->seg_lo[k - 1]; node <= p->seg_hi[k - 1]; ++node) {
    const int64_t off = p->dm.node_off[node] - p->seg_off[k - 1];
    const size_t bytes = 4 * (size_t)p->dm.P[node];
    if (h2d) {
      PEER_CUDA(cudaMemcpyAsync(dev + off, host + p->dm.node_off[node], bytes, cudaMemcpyHostToDevice, p->s_h2d));
      p->h2d_bytes += bytes;
    } else {
      PEER_CUDA(cudaMemcpyAsync(host + p->dm.node_off[node], dev + off, bytes, cudaMemcpyDeviceToHost, p->s_d2h));
      p->d2h_bytes += bytes;
    }
  }
  return true;
}

// a sub-model's swap-in, layer by layer: every array's node range, then the node's event (forward:
// nodes in execution order lo..hi; backward: hi..lo, the order the backward consumes them)
bool load_seg_nodes(atom_peer* p, int k, std::initializer_list<std::pair<float*, const float*>> arrays, bool reverse) {
  const int lo = p->seg_lo[k - 1], hi = p->seg_hi[k - 1];
  for (int i = 0; i <= hi - lo; ++i) {
    const int node = reverse ? hi - i : lo + i;
    const int64_t off = p->dm.node_off[node] - p->seg_off[k - 1];
    const size_t bytes = 4 * (size_t)p->dm.P[node];
    for (auto& a : arrays) {
      PEER_CUDA(cudaMemcpyAsync(a.first + off, a.second + p->dm.node_off[node], bytes, cudaMemcpyHostToDevice,
                                p->s_h2d));
      p->h2d_bytes += bytes;
    }
    PEER_CUDA(cudaEventRecord(p->node_ev[node], p->s_h2d));
  }
  return true;
}

// AdamW constants of this step's update: lr warm-up on the update count t; under gradient rounds
// (R37) the summed gradient of R rounds is scaled to their mean
AdamConsts step_consts(const atom_peer* p) {
  const float lr_t = p->cfg.warmup_steps > 0
                         ? p->cfg.lr * (float)std::min(1.0, (double)p->t / (double)p->cfg.warmup_steps)
                         : p->cfg.lr;
  const float gscale = p->cfg.grad_rounds > 0 ? 1.f / (float)p->cfg.grad_rounds : 1.f;
  return adam_consts(lr_t, p->cfg.beta1, p->cfg.beta2, p->cfg.eps, p->cfg.weight_decay, (long)p->t, gscale);
}

// one sub-model's CPU AdamW, run by the CUDA driver in copy-stream order (no CUDA calls inside)
struct HostAdamJob {
  float *p, *g, *m, *v;
  int64_t n;
  AdamConsts k;
  int threads;
};
void CUDART_CB host_adam(void* arg) {
  auto* j = (HostAdamJob*)arg;
  cpu_adamw(j->p, j->g, j->m, j->v, (long)j->n, j->k, j->threads);
  delete j;
}

template <typename T>
bool issue_op(atom_peer* p, const Op& o, bool sync, int idx) {
  cudaStream_t st = lane_stream(p, o.lane);
  const bool hu = p->cfg.grad_rounds > 0;
  for (auto& w : o.waits) {
    // a CAST's load dependency is taken per layer inside the sub-model's first FWD / BWD op
    if (o.kind == K_CAST && (w.kind == K_LOAD_F || w.kind == K_LOAD_B)) continue;
    if (w.kind == -1) {
      auto it = p->rel_of.find(p->slot_phys[w.seg]);
      if (it != p->rel_of.end() && it->second) PEER_CUDA(cudaStreamWaitEvent(st, it->second, 0));
    } else if (w.kind == -2) {
      // host arena of segment w.seg written by the previous step's STORE
      if (p->steps > 0) PEER_CUDA(cudaStreamWaitEvent(st, p->op_ev[{K_STORE, w.seg}], 0));
      // ... and, under gradient rounds, updated by its last CPU AdamW
      if (!p->cpu_ev_set.empty() && p->cpu_ev_set[w.seg - 1])
        PEER_CUDA(cudaStreamWaitEvent(st, p->cpu_ev[w.seg - 1], 0));
    } else {
      PEER_CUDA(cudaStreamWaitEvent(st, p->op_ev[{w.kind, w.seg}], 0));
    }
  }
  PEER_CUDA(cudaEventRecord(p->trace_ev[2 * idx], st));
  const int k = o.seg;
  uint8_t* base = k == 1 ? p->r1 : (o.slot >= 0 ? p->slot_phys[o.slot] : nullptr);
  SegView sv = base ? seg_view(p, k, base) : SegView{};
  const int64_t P = p->seg_P[k - 1];
  switch (o.kind) {
    case K_CAST:   // deferred: layer by layer inside the next FWD / BWD op (cast_node)
      p->cast_pending[k - 1] = 1;
      break;
    case K_FWD:
      PEER_OK(run_fwd<T>(p, k, o.mb, sv));
      break;
    case K_BWD:
      PEER_OK(run_bwd<T>(p, k, o.mb, sv));
      break;
    case K_FREE:
      break;
    case K_ADAM: {
      // host update placement: only the resident sub-model 1 updates on the GPU (at the last round
      // of an update); the others update on the CPU after their gradient sum is stored
      if (hu && (k != 1 || !p->upd_round)) break;
      T* wout = (k == 1 && !sync) ? (T*)sv.W : nullptr;
      KT(KC_ADAM, st, adamw<T>(sv.master, sv.grad, sv.m, sv.v, wout, P, step_consts(p), st));
      break;
    }
    case K_AVG:
      // guarded averaging (R36): the mean of the masters goes out of place into the segment's fp32
      // gradient buffer (free after ADAM); a one-int allreduce (min) of every rank's "arrived" flag
      // follows, and the average replaces the master only if it reads 1.  A peer that dies inside
      // the round never contributes its flag: when the survivors abort the communicator
      // (atom_comm_shrink with abort_ops) the flag stays 0 on every survivor and each keeps its own
      // updated master for that round -- consistent, never a partial reduction.
      if (p->nranks > 1 && !hu) {
        int* flag = p->avg_flags + k;
        PEER_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
        ncclResult_t r = ncclAllReduce(sv.master, sv.grad, (size_t)P, ncclFloat32, ncclAvg, p->comm, st);
        if (r == ncclSuccess) r = ncclAllReduce(p->avg_flags, flag, 1, ncclInt32, ncclMin, p->comm, st);
        if (r != ncclSuccess) {
          set_error("ncclAllReduce failed: %s", ncclGetErrorString(r));
          return false;
        }
        PEER_OK(commit_if(sv.master, sv.grad, P, flag, st));
      }
      break;
    case K_RECAST:
      KT(KC_CAST, st, cast_params<T>(sv.master, (T*)sv.W, P, st));
      break;
    case K_LOAD_F:
      // the interleaved last sub-model accumulates inside its forward op: its running gradient
      // sum comes with the forward load (R37)
      if (hu && k == p->S && p->round > 0)
        PEER_OK(load_seg_nodes(p, k, {{sv.master, p->h_master}, {sv.grad, p->h_gacc}}, false));
      else
        PEER_OK(load_seg_nodes(p, k, {{sv.master, p->h_master}}, false));
      break;
    case K_LOAD_B:
      if (hu) {
        if (k < p->S) {
          if (p->round > 0)
            PEER_OK(load_seg_nodes(p, k, {{sv.master, p->h_master}, {sv.grad, p->h_gacc}}, true));
          else
            PEER_OK(load_seg_nodes(p, k, {{sv.master, p->h_master}}, true));
        }
        break;
      }
      if (k == p->S && p->S >= 2) {   // the last sub-model kept its master: AdamW moments only
        PEER_OK(copy_seg(p, k, sv.m, p->h_m, true));
        PEER_OK(copy_seg(p, k, sv.v, p->h_v, true));
      } else {
        PEER_OK(load_seg_nodes(p, k, {{sv.master, p->h_master}, {sv.m, p->h_m}, {sv.v, p->h_v}}, true));
      }
      break;
    case K_STORE:
      if (hu) {
        // the gradient sum out; at the last round the CPU AdamW of this sub-model runs after it on
        // its own stream (host functions there do not hold up the copies); the next step's forward
        // load of the sub-model waits for it (HOST:k)
        PEER_OK(copy_seg(p, k, sv.grad, p->h_gacc, false));
        if (p->upd_round) {
          cudaEvent_t stored = p->cpu_ev[k - 1];
          PEER_CUDA(cudaEventRecord(stored, st));
          PEER_CUDA(cudaStreamWaitEvent(p->s_cpu, stored, 0));
          auto* job = new HostAdamJob{p->h_master + p->seg_off[k - 1], p->h_gacc + p->seg_off[k - 1],
                                      p->h_m + p->seg_off[k - 1], p->h_v + p->seg_off[k - 1], P, step_consts(p),
                                      p->cfg.cpu_threads};
          PEER_CUDA(cudaLaunchHostFunc(p->s_cpu, host_adam, job));
          PEER_CUDA(cudaEventRecord(p->cpu_ev[k - 1], p->s_cpu));
          p->cpu_ev_set[k - 1] = 1;
        }
        break;
      }
      PEER_OK(copy_seg(p, k, sv.master, p->h_master, false));
      PEER_OK(copy_seg(p, k, sv.m, p->h_m, false));
      PEER_OK(copy_seg(p, k, sv.v, p->h_v, false));
      break;
  }
  PEER_CUDA(cudaEventRecord(p->trace_ev[2 * idx + 1], st));
  cudaEvent_t ev = p->op_ev[{o.kind, o.seg}];
  PEER_CUDA(cudaEventRecord(ev, st));
  if (o.kind == K_FREE || o.kind == K_STORE) p->rel_of[p->slot_phys[o.slot]] = ev;
  // the step's loss is complete after the last micro-batch's head
  if (o.kind == K_FWD && o.seg == p->S && o.mb == p->C - 1) {
    PEER_OK(loss_sum(p->losses, (int64_t)p->C * p->dm.M, 1.f / (float)((double)p->C * p->dm.M), p->loss_dev, st));
    PEER_CUDA(cudaMemcpyAsync(p->h_loss, p->loss_dev, sizeof(float), cudaMemcpyDeviceToHost, st));
    PEER_CUDA(cudaEventRecord(p->ev_loss, st));
  }
  return true;
}

template <typename T>
bool run_step(atom_peer* p, float* loss_out) {
  const auto h0 = std::chrono::steady_clock::now();
  // gradient rounds (R37): step = round; the optimizer step count t advances on update rounds
  const int R = p->cfg.grad_rounds;
  p->round = R > 0 ? (int)(p->steps % R) : 0;
  p->upd_round = R <= 0 || p->round == R - 1;
  if (p->upd_round) p->t += 1;
  bool sync = p->upd_round && ((p->cfg.sync_every > 0 && p->t % p->cfg.sync_every == 0) || p->sync_next);
  if (p->upd_round) p->sync_next = false;
  if (p->nranks <= 1) sync = sync && false;
  // host update placement averages the updated host masters after the step (standalone pass)
  const bool flush_after = sync && R > 0;
  if (flush_after) sync = false;
  const std::vector<Op>& ops = sync ? p->ops_sync : p->ops;
  const std::vector<int>& endq = sync ? p->endq_sync : p->endq;
  if (p->trace_ev.size() < 2 * ops.size()) {
    for (size_t i = p->trace_ev.size(); i < 2 * ops.size(); ++i) {
      cudaEvent_t ev;
      PEER_CUDA(cudaEventCreate(&ev));
      p->trace_ev.push_back(ev);
    }
  }
  for (size_t i = 0; i < ops.size(); ++i) PEER_OK(issue_op<T>(p, ops[i], sync, (int)i));
  // host time spent issuing the step's work (launches, tensor-map encodes, events): if it reaches
  // the device time of a step the GPU waits for the host
  p->host_issue_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
  p->trace_ops = ops;
  p->have_trace = true;
  // relabel logical slots so that the next step starts from the queue [0 .. nslot-1]
  std::vector<uint8_t*> nphys(p->slot_phys.size());
  for (size_t i = 0; i < endq.size(); ++i) nphys[i] = p->slot_phys[endq[i]];
  p->slot_phys = nphys;
  p->steps++;
  p->rng_step++;
  PEER_CUDA(cudaEventSynchronize(p->ev_loss));
  *loss_out = *p->h_loss;
  if (flush_after) PEER_OK(peer_flush_average(p));
  return true;
}

}  // namespace

// ------------------------------------------------------------------ creation
namespace atom {

bool peer_stream_sync(atom_peer* p) {
  PEER_CUDA(cudaSetDevice(p->device));
  for (cudaStream_t s : {p->s_comp, p->s_h2d, p->s_d2h, p->s_comm, p->s_side, p->s_attn, p->s_cpu})
    if (s) PEER_CUDA(cudaStreamSynchronize(s));
  return true;
}

static float init_std(const atom_peer* p, int node, int t, float* fill) {
  const ModelDims& dm = p->dm;
  *fill = 0.f;
  if (node == 0) return 0.02f;
  if (node == dm.n_nodes - 1) {
    if (t == T_LNFG) { *fill = 1.f; return 0.f; }
    if (t == T_LNFB) return 0.f;
    return 0.02f;
  }
  if (node_half(dm, node) == 2) t += T_LN2G;   // operator-granular MLP half: tensors from ln2.g on
  switch (t) {
    case T_LN1G: case T_LN2G: *fill = 1.f; return 0.f;
    case T_WQKV: case T_WFC: return 0.02f;
    case T_WO: case T_WPR: return 0.02f / sqrtf(2.f * dm.L);
    default: return 0.f;
  }
}

bool peer_create(atom_peer* p, const float* init_params, uint64_t seed, const void* nccl_id) {
  const ModelDims& dm = p->dm;
  PEER_CUDA(cudaSetDevice(p->device));
  PEER_CUDA(cudaStreamCreateWithFlags(&p->s_comp, cudaStreamNonBlocking));
  PEER_CUDA(cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking));
  PEER_CUDA(cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking));
  PEER_CUDA(cudaStreamCreateWithFlags(&p->s_comm, cudaStreamNonBlocking));
  PEER_CUDA(cudaStreamCreateWithFlags(&p->s_side, cudaStreamNonBlocking));
  PEER_CUDA(cudaStreamCreateWithFlags(&p->s_attn, cudaStreamNonBlocking));
  if (p->cfg.grad_rounds > 0) {
    PEER_CUDA(cudaStreamCreateWithFlags(&p->s_cpu, cudaStreamNonBlocking));
    p->cpu_ev.assign(p->S, nullptr);
    p->cpu_ev_set.assign(p->S, 0);
    for (auto& ev : p->cpu_ev) PEER_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  for (auto& ev : p->ev_side) PEER_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  p->node_ev.assign(dm.n_nodes, nullptr);
  for (auto& ev : p->node_ev) PEER_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  p->cast_pending.assign(p->S, 0);
  {
    const char* e = getenv("ATOM_SIDE_WGRAD");   // 0: all block-backward kernels on one stream
    p->side_wgrad = !(e && e[0] == '0');
  }
  for (int kind = K_CAST; kind <= K_STORE; ++kind)
    for (int k = 1; k <= p->S; ++k) {
      cudaEvent_t ev;
      PEER_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      p->op_ev[{kind, k}] = ev;
    }
  PEER_CUDA(cudaEventCreateWithFlags(&p->ev_loss, cudaEventDisableTiming | cudaEventBlockingSync));
  // host arenas
  const size_t nb = 4 * (size_t)dm.N_pad;
  if (cudaHostAlloc((void**)&p->h_master, nb, cudaHostAllocPortable) != cudaSuccess ||
      cudaHostAlloc((void**)&p->h_m, nb, cudaHostAllocPortable) != cudaSuccess ||
      cudaHostAlloc((void**)&p->h_v, nb, cudaHostAllocPortable) != cudaSuccess) {
    set_error("pinned host allocation of %zu bytes x3 failed", nb);
    return false;
  }
  memset(p->h_m, 0, nb);
  memset(p->h_v, 0, nb);
  if (p->cfg.grad_rounds > 0) {   // host gradient sums (R37)
    if (cudaHostAlloc((void**)&p->h_gacc, nb, cudaHostAllocPortable) != cudaSuccess) {
      set_error("pinned host allocation of %zu bytes (gradient sums) failed", nb);
      return false;
    }
    memset(p->h_gacc, 0, nb);
  }
  PEER_CUDA(cudaHostAlloc((void**)&p->h_tokens, 4 * (size_t)p->C * dm.b * (dm.T + 1), cudaHostAllocPortable));
  PEER_CUDA(cudaHostAlloc((void**)&p->h_loss, 64, cudaHostAllocPortable));
  // carve the arena: r1 | slots | stash | hfin | work
  uint8_t* a = p->arena;
  p->r1 = a;
  a += p->plan.r1_bytes;
  for (int s = 0; s < p->plan.nslot; ++s) {
    p->slot_phys.push_back(a);
    a += p->plan.slot_bytes;
  }
  // stash: per block either full entries (1 for the interleaved last segment, else C) or, under
  // ACT_RECOMPUTE, C input checkpoints; then the re-forward entry; then the boundary buffers
  p->stash = a;
  int64_t off = 0;
  // blocks 1..n_recompute (never the last segment's) are re-forwarded: input checkpoints only
  bool any_rc = false;
  for (int l = 0; l < dm.L; ++l) {
    const bool last = p->seg_of_node[blk_node(dm, l, 0)] == p->S;   // both halves in the last segment
    const bool rc = !last && l < p->n_recompute;
    any_rc |= rc;
    p->blk_off.push_back(off);
    p->blk_full.push_back(!rc);
    off += !rc ? (last ? 1 : p->C) * stash_blk_bytes(dm) : (int64_t)p->C * hfin_bytes(dm);
  }
  if (any_rc) {
    p->rc_off = off;
    off += stash_blk_bytes(dm);
  }
  p->hfin = p->stash + off;
  a = p->stash + p->plan.stash_bytes;
  const int64_t ab = dm.wb, M = dm.M, d = dm.d;
  p->tokens = (int32_t*)a; a += al256(4LL * p->C * dm.b * (dm.T + 1));
  p->dh = a; a += al256(ab * p->C * M * d);
  p->losses = (float*)a; a += al256(4LL * p->C * M);
  p->scratch = a;
  const int64_t bwd_s = al256(ab * M * 4 * d) + 4 * al256(ab * M * d) + al256(4LL * dm.b * dm.h * dm.T) +
                        al256(ab * M * 4 * d) + (dm.dtype == ATOM_BF16 ? al256(2LL * dm.b * dm.h * dm.T * dm.T) : 0);
  p->scratch_bytes = std::max(bwd_s, al256(ab * M * al(dm.V, 8)) + 2 * al256(ab * M * d) + al256(8 * M));
  a += p->scratch_bytes;
  p->red = (float*)a; a += al256(4 * ceil_div(M, RED_ROWS) * 4 * d);
  p->emb = (int*)a; a += al256(4LL * (3 * dm.V + 1 + M));
  p->loss_dev = (float*)a;                 // 256-byte slot: the step loss at 0,
  p->red_ticket = (int*)(a + 64);          // column-sum tickets at 64 (48 ints, zeroed below)
  a += 256;
  if (a - p->arena != p->plan.device_bytes) {
    set_error("internal: arena carve %lld != plan.device_bytes %lld", (long long)(a - p->arena),
              (long long)p->plan.device_bytes);
    return false;
  }
  PEER_CUDA(cudaMemsetAsync(p->loss_dev, 0, 256, p->s_comp));
  // initial parameters -> host master (padded layout)
  memset(p->h_master, 0, nb);
  if (init_params) {
    for (int node = 0; node < dm.n_nodes; ++node)
      for (auto& ts : dm.tensors[node])
        memcpy(p->h_master + dm.node_off[node] + ts.off, init_params + dm.node_canon[node] + ts.canon, 4 * ts.n);
  } else {
    // draw on the device node by node through R1's master region (R1 holds E, the largest node)
    SegView r = seg_view(p, 1, p->r1);
    for (int node = 0; node < dm.n_nodes; ++node) {
      for (size_t t = 0; t < dm.tensors[node].size(); ++t) {
        float fill;
        const float sd = init_std(p, node, (int)t, &fill);
        const TensorSlot& ts = dm.tensors[node][t];
        PEER_OK(init_normal(r.master + ts.off, ts.n, seed, (uint64_t)(dm.node_canon[node] + ts.canon), sd, fill,
                            p->s_comp));
      }
      PEER_CUDA(cudaMemcpyAsync(p->h_master + dm.node_off[node], r.master, 4 * (size_t)dm.P[node],
                                cudaMemcpyDeviceToHost, p->s_comp));
      PEER_CUDA(cudaStreamSynchronize(p->s_comp));
      // padding stays zero: re-zero the padded gaps (init wrote only tensor ranges)
    }
  }
  // segment 1 becomes resident: master, m, v, compute-dtype weights
  {
    SegView r = seg_view(p, 1, p->r1);
    const int64_t P1 = p->seg_P[0];
    PEER_CUDA(cudaMemcpyAsync(r.master, p->h_master, 4 * (size_t)P1, cudaMemcpyHostToDevice, p->s_comp));
    PEER_CUDA(cudaMemsetAsync(r.m, 0, 4 * (size_t)P1, p->s_comp));
    PEER_CUDA(cudaMemsetAsync(r.v, 0, 4 * (size_t)P1, p->s_comp));
    if (dm.dtype == ATOM_BF16)
      PEER_OK(cast_params<bf16>(r.master, (bf16*)r.W, P1, p->s_comp));
    else
      PEER_OK(cast_params<float>(r.master, (float*)r.W, P1, p->s_comp));
    PEER_CUDA(cudaStreamSynchronize(p->s_comp));
  }
  if (p->nranks > 1) {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&p->comm, p->nranks, id, p->rank);
    if (r != ncclSuccess) {
      set_error("ncclCommInitRank failed: %s", ncclGetErrorString(r));
      return false;
    }
  }
  {   // guarded-averaging flags: [0] = 1 (this rank's contribution), [k] per segment
    PEER_CUDA(cudaMalloc((void**)&p->avg_flags, sizeof(int) * (p->S + 1)));
    std::vector<int> ones(p->S + 1, 1);
    PEER_CUDA(cudaMemcpy(p->avg_flags, ones.data(), sizeof(int) * (p->S + 1), cudaMemcpyHostToDevice));
  }
  p->ops = emit_schedule(p->S, p->C, false, &p->endq);
  p->ops_sync = emit_schedule(p->S, p->C, true, &p->endq_sync);
  PEER_CUDA(cudaEventCreate(&p->step_start));
  p->launch_base = g_launch_count;
  return true;
}

bool peer_step(atom_peer* p, const int32_t* tokens, bool on_device, float* loss) {
  PEER_CUDA(cudaSetDevice(p->device));
  const size_t tb = 4 * (size_t)p->C * p->dm.b * (p->dm.T + 1);
  if (on_device) {
    PEER_CUDA(cudaMemcpyAsync(p->tokens, tokens, tb, cudaMemcpyDeviceToDevice, p->s_comp));
  } else {
    memcpy(p->h_tokens, tokens, tb);
    PEER_CUDA(cudaMemcpyAsync(p->tokens, p->h_tokens, tb, cudaMemcpyHostToDevice, p->s_comp));
  }
  if (p->dm.dtype == ATOM_BF16) return run_step<bf16>(p, loss);
  return run_step<float>(p, loss);
}

// standalone averaging pass (atom_sync flush=1) over the n local peers of this process (each on its
// own device, all members of one communicator): per segment, H2D every peer's master (segments >= 2)
// into its slot 0, ONE NCCL group with every peer's allreduce, then D2H (segments >= 2) or re-derive
// the compute weights (the resident segment 1, averaged in place).  Segments are the outer loop: a
// peer's slot 0 is reused by its next segment only after that segment's allreduce has completed.
bool peers_flush_average(atom_peer* const* ps, int n) {
  for (int i = 0; i < n; ++i) PEER_OK(peer_stream_sync(ps[i]));
  if (ps[0]->nranks <= 1) return true;
  auto view = [](atom_peer* p, int k) {
    uint8_t* slot = p->slot_phys.empty() ? nullptr : p->slot_phys[0];
    return seg_view(p, k, k == 1 ? p->r1 : slot);
  };
  for (int k = 1; k <= ps[0]->S; ++k) {
    const int64_t P = ps[0]->seg_P[k - 1];
    for (int i = 0; i < n; ++i) {
      atom_peer* p = ps[i];
      PEER_CUDA(cudaSetDevice(p->device));
      if (k >= 2) PEER_OK(copy_seg(p, k, view(p, k).master, p->h_master, true));
      PEER_CUDA(cudaStreamSynchronize(p->s_h2d));
    }
    if (n > 1) ncclGroupStart();
    for (int i = 0; i < n; ++i) {
      atom_peer* p = ps[i];
      ncclResult_t r = ncclAllReduce(view(p, k).master, view(p, k).master, (size_t)P, ncclFloat32, ncclAvg, p->comm,
                                     p->s_comm);
      if (r != ncclSuccess) {
        if (n > 1) ncclGroupEnd();
        set_error("ncclAllReduce failed: %s", ncclGetErrorString(r));
        return false;
      }
    }
    if (n > 1) {
      ncclResult_t r = ncclGroupEnd();
      if (r != ncclSuccess) {
        set_error("ncclGroupEnd failed: %s", ncclGetErrorString(r));
        return false;
      }
    }
    for (int i = 0; i < n; ++i) {
      atom_peer* p = ps[i];
      PEER_CUDA(cudaSetDevice(p->device));
      PEER_CUDA(cudaStreamSynchronize(p->s_comm));
      SegView sv = view(p, k);
      if (k >= 2) {
        PEER_OK(copy_seg(p, k, sv.master, p->h_master, false));
        PEER_CUDA(cudaStreamSynchronize(p->s_d2h));
      } else if (p->dm.dtype == ATOM_BF16) {
        PEER_OK(cast_params<bf16>(sv.master, (bf16*)sv.W, P, p->s_comp));
      } else {
        PEER_OK(cast_params<float>(sv.master, (float*)sv.W, P, p->s_comp));
      }
    }
  }
  for (int i = 0; i < n; ++i) PEER_OK(peer_stream_sync(ps[i]));
  return true;
}

bool peer_flush_average(atom_peer* p) { return peers_flush_average(&p, 1); }

// membership change: abort the old communicator, join a new one (P:410 peers join and leave)
bool peer_comm_reset(atom_peer* p, const void* nccl_id, int nranks, int rank) {
  PEER_OK(peer_stream_sync(p));
  if (p->comm) {
    ncclCommAbort(p->comm);
    p->comm = nullptr;
  }
  p->nranks = nranks;
  p->rank = rank;
  if (nranks > 1) {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&p->comm, nranks, id, rank);
    if (r != ncclSuccess) {
      p->comm = nullptr;
      p->nranks = 1;
      p->rank = 0;
      set_error("ncclCommInitRank failed: %s", ncclGetErrorString(r));
      return false;
    }
  }
  return true;
}

// failed / leaving ranks dropped from the communicator without a new bootstrap (ncclCommShrink)
// abort_ops: a peer may have died inside an averaging round, leaving this peer's averaging stuck
// on the comm stream (and the copies / compute that wait for it): the outstanding operations are
// aborted first (NCCL_SHRINK_ABORT, or ncclCommAbort for a sole survivor), which releases the
// streams; the guarded commit (K_AVG) then keeps the local master for the unfinished round
bool peer_comm_shrink(atom_peer* p, const int* exclude, int n_exclude, bool abort_ops) {
  PEER_CUDA(cudaSetDevice(p->device));
  if (!abort_ops) PEER_OK(peer_stream_sync(p));
  if (!p->comm || n_exclude == 0) return peer_stream_sync(p);
  if (p->nranks - n_exclude <= 1) {   // sole survivor: nothing left to shrink to, no NCCL call
    ncclCommAbort(p->comm);
    p->comm = nullptr;
    p->nranks = 1;
    p->rank = 0;
    return peer_stream_sync(p);
  }
  ncclComm_t nc = nullptr;
  std::vector<int> ex(exclude, exclude + n_exclude);
  ncclResult_t r = ncclCommShrink(p->comm, ex.data(), n_exclude, &nc, nullptr,
                                  abort_ops ? NCCL_SHRINK_ABORT : NCCL_SHRINK_DEFAULT);
  if (r != ncclSuccess) {
    set_error("ncclCommShrink failed: %s", ncclGetErrorString(r));
    return false;
  }
  if (abort_ops) PEER_OK(peer_stream_sync(p));   // the aborted operations have released the streams
  ncclCommAbort(p->comm);   // the parent may still reference dead ranks: abort, not destroy
  p->comm = nc;
  int n = 1, rk = 0;
  if (ncclCommCount(nc, &n) != ncclSuccess || ncclCommUserRank(nc, &rk) != ncclSuccess) {
    set_error("nccl: shrunk communicator query failed");
    return false;
  }
  p->nranks = n;
  p->rank = rk;
  if (n == 1) {   // alone: keep no communicator (sync steps are local no-ops)
    ncclCommDestroy(p->comm);
    p->comm = nullptr;
  }
  return true;
}

// a joiner adopts root's model: fp32 master, AdamW m and v and the optimizer step count (AdamW
// bias correction, learning-rate warm-up). Everything travels through the working scratch (idle
// between steps) in chunks; only members with adopt set overwrite their state (the resident
// segment 1 in place, whose compute weights are then re-derived; the others in the host arena).
bool peer_broadcast_state(atom_peer* p, int root, bool adopt) {
  PEER_OK(peer_stream_sync(p));
  if (p->nranks <= 1) return true;
  const bool is_root = p->rank == root;
  float* buf = (float*)p->scratch;
  const int64_t chunk = p->scratch_bytes / 4;
  auto bcast = [&](void* b, size_t n, ncclDataType_t ty) -> bool {
    ncclResult_t r = ncclBroadcast(b, b, n, ty, root, p->comm, p->s_comm);
    if (r != ncclSuccess) {
      set_error("ncclBroadcast failed: %s", ncclGetErrorString(r));
      return false;
    }
    PEER_CUDA(cudaStreamSynchronize(p->s_comm));
    return true;
  };
  SegView r1 = seg_view(p, 1, p->r1);
  const int64_t P1 = p->seg_P[0];
  // [0, P1) lives on the device (segment 1), [P1, N_pad) in the host arena (padded layout)
  auto src = [&](int a, int64_t i) -> float* {
    float* dev[3] = {r1.master, r1.m, r1.v};
    float* host[3] = {p->h_master, p->h_m, p->h_v};
    return i < P1 ? dev[a] + i : host[a] + i;
  };
  for (int a = 0; a < 3; ++a)
    for (int64_t i0 = 0; i0 < p->dm.N_pad;) {
      const int64_t n = std::min(chunk, (i0 < P1 ? P1 : p->dm.N_pad) - i0);
      if (is_root) PEER_CUDA(cudaMemcpy(buf, src(a, i0), 4 * (size_t)n, cudaMemcpyDefault));
      PEER_OK(bcast(buf, (size_t)n, ncclFloat32));
      if (adopt && !is_root) PEER_CUDA(cudaMemcpy(src(a, i0), buf, 4 * (size_t)n, cudaMemcpyDefault));
      i0 += n;
    }
  int64_t* dt = (int64_t*)buf;
  PEER_CUDA(cudaMemcpy(dt, &p->t, sizeof(int64_t), cudaMemcpyHostToDevice));
  PEER_OK(bcast(dt, 1, ncclInt64));
  if (adopt) PEER_CUDA(cudaMemcpy(&p->t, dt, sizeof(int64_t), cudaMemcpyDeviceToHost));
  if (adopt && !is_root) {
    if (p->dm.dtype == ATOM_BF16)
      PEER_OK(cast_params<bf16>(r1.master, (bf16*)r1.W, P1, p->s_comp));
    else
      PEER_OK(cast_params<float>(r1.master, (float*)r1.W, P1, p->s_comp));
  }
  PEER_OK(peer_stream_sync(p));
  return true;
}

bool peer_get_params(atom_peer* p, float* master, float* m, float* v) {
  PEER_OK(peer_stream_sync(p));
  const ModelDims& dm = p->dm;
  // segment 1 lives on the device: refresh its host copy
  SegView r = seg_view(p, 1, p->r1);
  const size_t b1 = 4 * (size_t)p->seg_P[0];
  PEER_CUDA(cudaMemcpy(p->h_master, r.master, b1, cudaMemcpyDeviceToHost));
  PEER_CUDA(cudaMemcpy(p->h_m, r.m, b1, cudaMemcpyDeviceToHost));
  PEER_CUDA(cudaMemcpy(p->h_v, r.v, b1, cudaMemcpyDeviceToHost));
  float* outs[3] = {master, m, v};
  float* srcs[3] = {p->h_master, p->h_m, p->h_v};
  for (int a = 0; a < 3; ++a) {
    if (!outs[a]) continue;
    for (int node = 0; node < dm.n_nodes; ++node)
      for (auto& ts : dm.tensors[node])
        memcpy(outs[a] + dm.node_canon[node] + ts.canon, srcs[a] + dm.node_off[node] + ts.off, 4 * ts.n);
  }
  return true;
}

bool peer_trace(atom_peer* p, std::string* out, atom_stats_t* st) {
  PEER_OK(peer_stream_sync(p));
  out->clear();
  if (!p->have_trace) return true;
  const auto& ops = p->trace_ops;
  std::vector<float> t0(ops.size()), t1(ops.size());
  float base = 0;
  for (size_t i = 0; i < ops.size(); ++i) {
    PEER_CUDA(cudaEventElapsedTime(&t0[i], p->trace_ev[0], p->trace_ev[2 * i]));
    PEER_CUDA(cudaEventElapsedTime(&t1[i], p->trace_ev[0], p->trace_ev[2 * i + 1]));
    base = std::min(base, t0[i]);
  }
  float lo = 1e30f, hi = -1e30f;
  std::vector<std::pair<float, float>> comp, comp_all;
  std::vector<std::pair<float, float>> copies[2];   // h2d, d2h
  char buf[256];
  for (size_t i = 0; i < ops.size(); ++i) {
    const Op& o = ops[i];
    const float a = t0[i] - base, b = t1[i] - base;
    lo = std::min(lo, a);
    hi = std::max(hi, b);
    char mb[16], sl[16];
    if (o.mb < 0) strcpy(mb, "-"); else snprintf(mb, sizeof mb, "%d", o.mb);
    if (o.slot < 0) strcpy(sl, "-"); else snprintf(sl, sizeof sl, "%d", o.slot);
    snprintf(buf, sizeof buf, "%s %s %d %s %s %.1f %.1f\n", lane_name(o.lane), kind_name(o.kind), o.seg, mb, sl,
             a * 1000.0, b * 1000.0);
    *out += buf;
    if (o.lane == L_COMPUTE && (o.kind == K_FWD || o.kind == K_BWD)) comp.push_back({a, b});
    if (o.lane == L_COMPUTE && b > a) comp_all.push_back({a, b});
    if ((o.lane == L_H2D || o.lane == L_D2H) && b > a) copies[o.lane == L_D2H].push_back({a, b});
  }
  if (!st) return true;
  st->step_ms = hi - lo;
  double* tot[2] = {&st->h2d_ms, &st->d2h_ms};
  double* hid[2] = {&st->h2d_hidden_ms, &st->d2h_hidden_ms};
  for (int dir = 0; dir < 2; ++dir) {
    *tot[dir] = *hid[dir] = 0;
    for (auto& c : copies[dir]) {
      *tot[dir] += c.second - c.first;
      for (auto& k : comp) {
        float x = std::max(c.first, k.first), y = std::min(c.second, k.second);
        if (y > x) *hid[dir] += y - x;
      }
    }
  }
  st->copy_ms = st->h2d_ms + st->d2h_ms;
  st->copy_hidden_ms = st->h2d_hidden_ms + st->d2h_hidden_ms;
  // compute lane: union of its op intervals over its span (the rest is the lane waiting on swaps)
  std::sort(comp_all.begin(), comp_all.end());
  double busy = 0;
  float cs = 0, ce = -1e30f, first = 0, last = 0;
  for (size_t i = 0; i < comp_all.size(); ++i) {
    const auto& iv = comp_all[i];
    if (i == 0) first = iv.first;
    last = std::max(last, iv.second);
    if (iv.first > ce) {
      if (i) busy += ce - cs;
      cs = iv.first;
      ce = iv.second;
    } else {
      ce = std::max(ce, iv.second);
    }
  }
  if (!comp_all.empty()) busy += ce - cs;
  st->compute_busy_ms = busy;
  st->compute_span_ms = comp_all.empty() ? 0 : last - first;
  return true;
}

bool peer_stats(atom_peer* p, atom_stats_t* s) {
  PEER_OK(peer_stream_sync(p));
  for (size_t i = 0; i < p->gemm_n; ++i) {
    float ms;
    PEER_CUDA(cudaEventElapsedTime(&ms, p->gemm_ev[2 * i], p->gemm_ev[2 * i + 1]));
    p->gemm_ms_acc += ms;
    p->gemm_fl_acc += p->gemm_fl[i];
    auto& agg = p->gemm_by_shape[p->gemm_key[i]];
    agg.first += 1;
    agg.second += ms;
  }
  p->gemm_n = 0;
  for (size_t i = 0; i < p->kt_n; ++i) {
    float ms;
    PEER_CUDA(cudaEventElapsedTime(&ms, p->kt_ev[2 * i], p->kt_ev[2 * i + 1]));
    p->kt_ms[p->kt_cat[i]] += ms;
    p->kt_count[p->kt_cat[i]] += 1;
  }
  p->kt_n = 0;
  memset(s, 0, sizeof(*s));
  s->steps = p->steps;
  s->host_issue_ms = p->host_issue_ms;
  s->kernel_launches = (int64_t)(g_launch_count - p->launch_base);
  s->gemm_launches = p->gemm_launches;
  s->gemm_ms = p->gemm_ms_acc;
  s->gemm_flops = p->gemm_fl_acc;
  s->h2d_bytes = p->h2d_bytes;
  s->d2h_bytes = p->d2h_bytes;
  std::string tr;
  PEER_OK(peer_trace(p, &tr, s));
  return true;
}

// per-shape GEMM timing since the last reset: "M N K a_mn b_mn epilogue launches ms TFLOP/s" lines
bool peer_gemm_log(atom_peer* p, std::string* out) {
  atom_stats_t s;
  PEER_OK(peer_stats(p, &s));   // folds the pending launch events into gemm_by_shape
  out->clear();
  char buf[192];
  for (auto& kv : p->gemm_by_shape) {
    int M, N, K, a, b, m;
    sscanf(kv.first.c_str(), "%d %d %d %d %d %d", &M, &N, &K, &a, &b, &m);
    const double tf = kv.second.second > 0 ? 2.0 * M * N * (double)K * kv.second.first / (kv.second.second * 1e-3) / 1e12 : 0;
    snprintf(buf, sizeof buf, "%s %lld %.3f %.1f\n", kv.first.c_str(), (long long)kv.second.first, kv.second.second, tf);
    *out += buf;
  }
  return true;
}

// per category since the last reset: "category launch_groups ms" lines
bool peer_kernel_log(atom_peer* p, std::string* out) {
  atom_stats_t s;
  PEER_OK(peer_stats(p, &s));
  out->clear();
  char buf[160];
  for (int c = 0; c < KC_N; ++c) {
    snprintf(buf, sizeof buf, "%s %lld %.3f\n", kcat_name(c), (long long)p->kt_count[c], p->kt_ms[c]);
    *out += buf;
  }
  return true;
}

void peer_reset_stats(atom_peer* p, int timing) {
  p->kt_n = 0;
  for (int c = 0; c < 16; ++c) {
    p->kt_ms[c] = 0;
    p->kt_count[c] = 0;
  }
  p->steps = 0;
  p->gemm_launches = 0;
  p->gemm_ms_acc = p->gemm_fl_acc = 0;
  p->gemm_n = 0;
  p->gemm_by_shape.clear();
  p->h2d_bytes = p->d2h_bytes = 0;
  p->launch_base = g_launch_count;
  p->timing = timing;
}

void peer_free(atom_peer* p) {
  cudaSetDevice(p->device);
  for (cudaStream_t s : {p->s_comp, p->s_h2d, p->s_d2h, p->s_comm, p->s_side, p->s_attn, p->s_cpu})
    if (s) cudaStreamSynchronize(s);
  if (p->comm) ncclCommDestroy(p->comm);
  if (p->avg_flags) cudaFree(p->avg_flags);
  for (auto ev : p->ev_side)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : p->node_ev)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : p->cpu_ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& kv : p->op_ev) cudaEventDestroy(kv.second);
  for (auto ev : p->trace_ev) cudaEventDestroy(ev);
  for (auto ev : p->gemm_ev) cudaEventDestroy(ev);
  for (auto ev : p->kt_ev) cudaEventDestroy(ev);
  if (p->ev_loss) cudaEventDestroy(p->ev_loss);
  if (p->step_start) cudaEventDestroy(p->step_start);
  for (cudaStream_t s : {p->s_comp, p->s_h2d, p->s_d2h, p->s_comm, p->s_side, p->s_attn, p->s_cpu})
    if (s) cudaStreamDestroy(s);
  for (float* h : {p->h_master, p->h_m, p->h_v, p->h_loss, p->h_gacc})
    if (h) cudaFreeHost(h);
  if (p->h_tokens) cudaFreeHost(p->h_tokens);
}

}  // namespace atom
