// Partition planner (§III-D) and swap schedule.
//
// Nodes: 0 = E (wte, wpe), 1..L = transformer blocks, L+1 = H (ln_f, lm_head); sub-models are
// contiguous node runs.  Costs, memory model and constraints follow DESIGN.md §4 and must equal
// oracle/planner.py bit for bit (tests/test_planner_parity.py).
#include "planner.h"

#include <algorithm>
#include <deque>
#include <map>
#include <set>
#include <string.h>

namespace atom {

void set_error(const char* fmt, ...);

typedef __int128 i128;

bool make_dims(const atom_model_cfg& c, ModelDims* o) {
  if (c.n_layer <= 0 || c.d_model <= 0 || c.n_head <= 0 || c.seq_len <= 0 || c.vocab <= 0 || c.micro_batch <= 0) {
    set_error("invalid config: L, d, h, T, V, b must be positive");
    return false;
  }
  if (c.d_model % c.n_head) {
    set_error("invalid config: d_model %% n_head != 0");
    return false;
  }
  if (c.n_layer + 2 > 4096) {
    set_error("invalid config: too many layers");
    return false;
  }
  if (c.dtype != ATOM_FP32 && c.dtype != ATOM_BF16) {
    set_error("invalid config: dtype");
    return false;
  }
  if (c.op_nodes != 0 && c.op_nodes != 1) {
    set_error("invalid config: op_nodes must be 0 or 1");
    return false;
  }
  ModelDims& m = *o;
  m.L = c.n_layer; m.d = c.d_model; m.h = c.n_head; m.T = c.seq_len; m.V = c.vocab; m.b = c.micro_batch;
  m.op = c.op_nodes;
  m.M = (int64_t)m.b * m.T;
  m.dtype = c.dtype;
  m.wb = c.dtype == ATOM_FP32 ? 4 : 2;
  m.n_nodes = (m.op ? 2 : 1) * m.L + 2;
  const int64_t d = m.d, V = m.V, T = m.T;
  auto mk = [](std::initializer_list<int64_t> sizes) {
    std::vector<TensorSlot> v;
    int64_t off = 0, canon = 0;
    for (int64_t n : sizes) {
      v.push_back({n, off, canon});
      off += al64(n);
      canon += n;
    }
    return v;
  };
  m.tensors.clear();
  m.tensors.push_back(mk({V * d, T * d}));
  for (int l = 0; l < m.L; ++l) {
    if (m.op) {   // attention half, MLP half (the canonical block order split in two)
      m.tensors.push_back(mk({d, d, 3 * d * d, 3 * d, d * d, d}));
      m.tensors.push_back(mk({d, d, 4 * d * d, 4 * d, 4 * d * d, d}));
    } else {
      m.tensors.push_back(mk({d, d, 3 * d * d, 3 * d, d * d, d, d, d, 4 * d * d, 4 * d, 4 * d * d, d}));
    }
  }
  m.tensors.push_back(mk({d, d, V * d}));
  m.P.clear(); m.P_canon.clear(); m.node_off.clear(); m.node_canon.clear();
  int64_t off = 0, canon = 0;
  for (auto& ts : m.tensors) {
    int64_t p = 0, pc = 0;
    for (auto& t : ts) { p += al64(t.n); pc += t.n; }
    m.node_off.push_back(off);
    m.node_canon.push_back(canon);
    m.P.push_back(p);
    m.P_canon.push_back(pc);
    off += p;
    canon += pc;
  }
  m.N_pad = off;
  m.N_canon = canon;
  return true;
}

static int64_t ceil_ns(i128 amount, int64_t rate) {  // ceil(amount * 1e9 / rate)
  i128 num = amount * (i128)1000000000;
  return (int64_t)((num + rate - 1) / rate);
}

Costs node_costs(const atom_model_cfg& c, const ModelDims& dm, int64_t link_bw) {
  Costs k;
  const int n = dm.n_nodes;
  const i128 d = dm.d, V = dm.V, T = dm.T, b = dm.b, M = dm.M;
  const int64_t d2h = c.d2h_bw > 0 ? c.d2h_bw : link_bw;
  for (int i = 0; i < n; ++i) {
    // forward FLOPs per micro-batch: block 24 d^2 M + attention; operator-granular halves
    // 8 d^2 M + attention (QKV, attention, projection) and 16 d^2 M (fc, fc2)
    const bool blk = is_block_node(dm, i);
    const int half = blk ? node_half(dm, i) : 0;
    const i128 fattn = 2 * d * T * (T + 1) * b;
    i128 ff = 0;
    if (blk) ff = half == 0 ? 24 * d * d * M + fattn : (half == 1 ? 8 * d * d * M + fattn : 16 * d * d * M);
    if (i == n - 1) ff = 2 * d * V * M;
    k.ff.push_back((int64_t)ff);
    if (c.cost_table) {
      k.tf.push_back(c.cost_table[2 * i]);
      k.tb.push_back(c.cost_table[2 * i + 1]);
      k.tbr.push_back(k.tb.back() + (blk ? k.tf.back() : 0));
    } else {
      // re-forward inside the backward: QKV, proj and fc GEMMs + attention (not the MLP projection)
      const i128 fr = !blk ? 0 : (half == 0 ? 16 * d * d * M + fattn : (half == 1 ? 8 * d * d * M + fattn : 8 * d * d * M));
      k.tf.push_back(ceil_ns(ff, c.peak_flops));
      k.tb.push_back(ceil_ns(2 * ff, c.peak_flops));
      k.tbr.push_back(ceil_ns(2 * ff + fr, c.peak_flops));
    }
    const i128 p = dm.P[i];
    k.P.push_back(dm.P[i]);
    k.tlf.push_back(ceil_ns(4 * p, link_bw));
    // grad_rounds > 0 (host update placement, R37): the backward loads master + gradient sum
    // (the last segment: the sum alone) and stores the sum back
    const bool hu = c.grad_rounds > 0;
    k.tlb.push_back(ceil_ns((hu ? 8 : 12) * p, link_bw));
    k.tmv.push_back(ceil_ns((hu ? 4 : 8) * p, link_bw));
    k.ts.push_back(ceil_ns((hu ? 4 : 12) * p, d2h));
  }
  return k;
}

int64_t seg_need(const ModelDims& dm, int64_t P) { return al256((int64_t)dm.wb * P) + 4 * al256(4 * P); }

int64_t stash_blk_bytes(const ModelDims& dm) {
  const int64_t ab = dm.wb, d = dm.d, M = dm.M;
  return al256(ab * M * d) + al256(ab * M * 3 * d) + al256(ab * M * d) + al256(ab * M * d) + al256(ab * M * 4 * d) +
         al256(8 * M) + al256(8 * M) + al256(4LL * dm.b * dm.h * dm.T);
}
int64_t hfin_bytes(const ModelDims& dm) { return al256((int64_t)dm.wb * dm.M * dm.d); }
int n_rc(const ModelDims& dm, int R, int nb_last) { return std::min(R, dm.L - nb_last); }
// re-forwarded blocks (1..R, none of the last segment) keep C input checkpoints and share one
// entry their backward re-forward fills; the others keep C full entries (1 in the last segment)
int64_t stash_bytes(const ModelDims& dm, int C, int nb_last, int S, int R) {
  const int64_t nh = S == 1 ? 1 : (nb_last == 0 ? C : C + 1);
  const int64_t nb_pre = dm.L - nb_last;
  const int64_t r = n_rc(dm, R, nb_last);
  return stash_blk_bytes(dm) * ((int64_t)C * (nb_pre - r) + nb_last) + hfin_bytes(dm) * C * r + hfin_bytes(dm) * nh +
         (r > 0 ? stash_blk_bytes(dm) : 0);
}
int64_t work_bytes(const ModelDims& dm, int C) {
  const int64_t ab = dm.wb, d = dm.d, V = dm.V, T = dm.T, b = dm.b, h = dm.h, M = dm.M;
  const int64_t Vp = al(V, 8);
  int64_t tokens = al256(4LL * C * b * (T + 1));
  int64_t dh = al256(ab * C * M * d);
  int64_t losses = al256(4LL * C * M);
  // G, A, DA, DX2, DO, D, G2 (dL/du beside GELU(u), so the MLP projection's weight gradient can
  // run on the side stream)
  int64_t bwd_s = al256(ab * M * 4 * d) + 4 * al256(ab * M * d) + al256(4 * b * h * T) + al256(ab * M * 4 * d);
  if (dm.dtype == ATOM_BF16) bwd_s += al256(2 * b * h * T * T);   // attention dS^T between dK/dV and dQ
  int64_t head_s = al256(ab * M * Vp) + 2 * al256(ab * M * d) + al256(8 * M);
  int64_t scratch = std::max(bwd_s, head_s);
  int64_t red = al256(4 * ceil_div(M, RED_ROWS) * 4 * d);
  int64_t emb = al256(4 * (3 * V + 1 + M));
  int64_t small = 256;
  return tokens + dh + losses + scratch + red + emb + small;
}
int nslot_for(int S) { return S == 1 ? 0 : (S == 2 ? 2 : 3); }

// ------------------------------------------------------------------ evaluator
namespace {
struct Eval {
  const atom_model_cfg& c;
  const ModelDims& dm;
  int64_t budget;
  int R;   // blocks 1..R are re-forwarded inside their backward (those before the last segment)
  Costs k;
  int n;
  std::vector<int64_t> pP, ptf, ptb, ptbx, ptlf, ptlb, ptmv, pts;
  Eval(const atom_model_cfg& c_, const ModelDims& dm_, int64_t budget_, int64_t link, int R_)
      : c(c_), dm(dm_), budget(budget_), R(R_), k(node_costs(c_, dm_, link)), n(dm_.n_nodes) {
    auto pre = [&](const std::vector<int64_t>& v, std::vector<int64_t>& p) {
      p.assign(v.size() + 1, 0);
      for (size_t i = 0; i < v.size(); ++i) p[i + 1] = p[i] + v[i];
    };
    std::vector<int64_t> tbx(k.tb);
    if (!dm.op)
      for (int v = 1; v <= std::min(R, dm.L); ++v) tbx[v] = k.tbr[v];
    pre(k.P, pP); pre(k.tf, ptf); pre(k.tb, ptb); pre(tbx, ptbx); pre(k.tlf, ptlf); pre(k.tlb, ptlb);
    pre(k.tmv, ptmv); pre(k.ts, pts);
  }
  static int64_t s(const std::vector<int64_t>& p, int i, int j) { return p[j + 1] - p[i]; }
  // backward time of a segment that is not the last one (its re-forwarded blocks included)
  int64_t tbn(int i, int j) const { return s(ptbx, i, j); }
  int64_t need(int i, int j) const { return seg_need(dm, s(pP, i, j)); }
  // whole blocks inside nodes [i..j] (operator-granular: both halves inside)
  int nblocks(int i, int j) const {
    if (dm.op) {
      int nb = 0;
      for (int l = 0; l < dm.L; ++l) nb += (i <= 2 * l + 1 && 2 * l + 2 <= j) ? 1 : 0;
      return nb;
    }
    int lo = std::max(i, 1), hi = std::min(j, dm.L);
    return std::max(0, hi - lo + 1);
  }
  int64_t r1(int e1) const { return need(0, e1); }
  // pairwise constraints between adjacent segments a=[i..j], b=[j+1..kk]; b_last: b is final
  bool pair_ok(int C, int i, int j, int kk, bool b_last) const {
    if (!c.overlap_check) return true;
    const int j1 = j + 1;
    const bool first = i == 0;
    if (first) {
      if ((i128)C * (s(ptf, i, j) + tbn(i, j)) < (i128)s(pts, j1, kk) + s(ptlf, j1, kk)) return false;
    } else if ((i128)C * s(ptf, i, j) < s(ptlf, j1, kk)) {
      return false;
    }
    if ((i128)C * tbn(i, j) < s(pts, j1, kk)) return false;
    const i128 load_a = first ? 0 : s(ptlb, i, j);
    if (b_last) return (i128)C * (s(ptf, j1, kk) + s(ptb, j1, kk)) >= s(ptmv, j1, kk) + load_a;
    return (i128)C * tbn(j1, kk) >= load_a;
  }
  int64_t slot_need(const std::vector<int>& ends) const {
    int64_t q = 0;
    for (size_t t = 1; t < ends.size(); ++t) q = std::max(q, need(ends[t - 1] + 1, ends[t]));
    return q;
  }
  int64_t device_bytes(int C, const std::vector<int>& ends) const {
    const int S = (int)ends.size();
    const int il = S == 1 ? 0 : ends[S - 2] + 1;
    return r1(ends[0]) + nslot_for(S) * al256(slot_need(ends)) + stash_bytes(dm, C, nblocks(il, n - 1), S, R) +
           work_bytes(dm, C);
  }
  // nullptr if feasible, else the first violated constraint
  const char* violation(int C, const std::vector<int>& ends, int* bad_pair) const {
    if (device_bytes(C, ends) > budget) return "memory";
    if (c.state_budget > 0 && r1(ends[0]) + nslot_for((int)ends.size()) * al256(slot_need(ends)) > c.state_budget)
      return "state memory";
    for (size_t t = 0; t + 1 < ends.size(); ++t) {
      int i = t == 0 ? 0 : ends[t - 1] + 1;
      if (!pair_ok(C, i, ends[t], ends[t + 1], t + 2 == ends.size())) {
        if (bad_pair) *bad_pair = (int)t + 1;
        return "overlap";
      }
    }
    return nullptr;
  }
};

// exact optimum for one C: min S, then lexicographically smallest ends (see oracle/planner.py)
bool dp_for_C(const Eval& ev, int C, std::vector<int>* best_out) {
  const int n = ev.n;
  std::vector<int> e1v = {n - 1};
  if (!ev.violation(C, e1v, nullptr)) { *best_out = e1v; return true; }
  if (n < 2) return false;
  for (int e = 0; e < n - 1; ++e) {
    std::vector<int> v = {e, n - 1};
    if (!ev.violation(C, v, nullptr)) { *best_out = v; return true; }
  }
  if (n < 3) return false;
  std::set<int64_t> needset;
  for (int i = 1; i < n; ++i)
    for (int j = i; j < n; ++j) needset.insert(ev.need(i, j));
  const int64_t wk = work_bytes(ev.dm, C);
  const int64_t sb = ev.c.state_budget;
  const int INF = 1 << 30;
  bool have = false;
  int bestS = INF;
  std::vector<int> best;
  std::vector<int> tab((size_t)n * n, INF);
  auto T = [&](int i, int j) -> int& { return tab[(size_t)i * n + j]; };
  for (int64_t Q : needset) {
    const int64_t base = 3 * al256(Q) + wk;
    if (base > ev.budget) break;
    for (int e1 = 0; e1 < n - 2; ++e1) {
      if (sb > 0 && 3 * al256(Q) + ev.r1(e1) > sb) break;
      const int64_t rem = ev.budget - base - ev.r1(e1);
      if (rem < 0) break;
      std::vector<char> term(n, 0);
      bool any = false;
      for (int il = e1 + 2; il < n; ++il)
        if (ev.need(il, n - 1) <= Q && stash_bytes(ev.dm, C, ev.nblocks(il, n - 1), 3, ev.R) <= rem) {
          term[il] = 1;
          any = true;
        }
      if (!any) continue;
      auto trans = [&](int i, int j) {
        int v = INF;
        if (j + 1 < n && term[j + 1] && ev.pair_ok(C, i, j, n - 1, true)) v = 1;
        for (int kk = j + 1; kk < n - 1; ++kk) {
          int r = T(j + 1, kk);
          if (r + 1 < v && ev.pair_ok(C, i, j, kk, false)) v = r + 1;
        }
        return v;
      };
      for (int j = n - 2; j > e1; --j)
        for (int i = e1 + 1; i <= j; ++i) T(i, j) = ev.need(i, j) > Q ? INF : trans(i, j);
      T(0, e1) = trans(0, e1);
      const int r0 = T(0, e1);
      if (r0 >= INF) continue;
      const int S = r0 + 1;
      std::vector<int> ends = {e1};
      int ci = 0, cj = e1, left = r0;
      while (left > 0) {
        if (left == 1) { ends.push_back(n - 1); break; }
        bool found = false;
        for (int kk = cj + 1; kk < n - 1; ++kk) {
          if (T(cj + 1, kk) == left - 1 && ev.pair_ok(C, ci, cj, kk, false)) {
            ends.push_back(kk);
            ci = cj + 1; cj = kk; --left;
            found = true;
            break;
          }
        }
        if (!found) return false;  // cannot happen (consistent table)
      }
      if (!have || S < bestS || (S == bestS && ends < best)) {
        have = true;
        bestS = S;
        best = ends;
      }
    }
  }
  if (have) *best_out = best;
  return have;
}
}  // namespace

// ------------------------------------------------------------------ schedule
const char* lane_name(int l) {
  static const char* n[] = {"compute", "h2d", "d2h", "comm"};
  return n[l];
}
const char* kind_name(int k) {
  static const char* n[] = {"CAST", "FWD", "BWD", "FREE", "ADAM", "AVG", "RECAST", "LOAD_F", "LOAD_B", "STORE"};
  return n[k];
}

std::vector<Op> emit_schedule(int S, int C, bool sync, std::vector<int>* end_queue) {
  const int nslot = nslot_for(S);
  std::deque<int> q;
  std::vector<Wait> rel(nslot);
  for (int s = 0; s < nslot; ++s) { q.push_back(s); rel[s] = {-1, s}; }
  std::map<int, int> slot;
  std::vector<Op> ops;
  auto op = [&](int lane, int kind, int k, int mb, int s, std::vector<Wait> w) { ops.push_back({lane, kind, k, mb, s, w}); };
  auto alloc = [&](int k, Wait* w) {
    int s = q.front();
    q.pop_front();
    slot[k] = s;
    *w = rel[s];
    return s;
  };
  auto release = [&](int s, Wait ev) { q.push_back(s); rel[s] = ev; };
  auto sl = [&](int k) { auto it = slot.find(k); return it == slot.end() ? -1 : it->second; };

  for (int k = 1; k <= S; ++k) {
    if (k >= 2) op(L_COMPUTE, K_CAST, k, -1, slot[k], {{K_LOAD_F, k}});
    for (int mb = 0; mb < C; ++mb) {
      op(L_COMPUTE, K_FWD, k, mb, k >= 2 ? sl(k) : -1, {});
      if (mb == 0) {
        if (k < S) {
          Wait w;
          int s = alloc(k + 1, &w);
          op(L_H2D, K_LOAD_F, k + 1, -1, s, {w, {-2, k + 1}});
        } else if (S >= 2) {
          op(L_H2D, K_LOAD_B, S, -1, slot[S], {{-2, S}});
          if (S - 1 >= 2) {
            Wait w;
            int s = alloc(S - 1, &w);
            op(L_H2D, K_LOAD_B, S - 1, -1, s, {w, {-2, S - 1}});
          }
        }
      }
      if (k == S) op(L_COMPUTE, K_BWD, S, mb, sl(S), {});
    }
    if (k >= 2 && k < S) {
      op(L_COMPUTE, K_FREE, k, -1, slot[k], {});
      release(slot[k], {K_FREE, k});
    }
  }
  auto finish = [&](int k) {
    int s = sl(k);
    std::vector<Wait> w;
    if (k == S && S >= 2) w.push_back({K_LOAD_B, k});
    op(L_COMPUTE, K_ADAM, k, -1, s, w);
    Wait last = {K_ADAM, k};
    if (sync) {
      op(L_COMM, K_AVG, k, -1, s, {last});
      last = {K_AVG, k};
      if (k == 1) op(L_COMPUTE, K_RECAST, 1, -1, -1, {last});
    }
    if (k >= 2) {
      op(L_D2H, K_STORE, k, -1, s, {last});
      release(s, {K_STORE, k});
    }
  };
  finish(S);
  for (int k = S - 1; k >= 1; --k) {
    if (k >= 2) op(L_COMPUTE, K_CAST, k, -1, slot[k], {{K_LOAD_B, k}});
    for (int mb = 0; mb < C; ++mb) {
      op(L_COMPUTE, K_BWD, k, mb, sl(k), {});
      if (mb == 0 && k - 1 >= 2) {
        Wait w;
        int s = alloc(k - 1, &w);
        op(L_H2D, K_LOAD_B, k - 1, -1, s, {w, {-2, k - 1}});
      }
    }
    finish(k);
  }
  if (end_queue) end_queue->assign(q.begin(), q.end());
  return ops;
}

std::string schedule_text(const std::vector<Op>& ops) {
  std::string out;
  char buf[256];
  for (auto& o : ops) {
    std::string w;
    for (size_t i = 0; i < o.waits.size(); ++i) {
      if (i) w += ",";
      if (o.waits[i].kind == -1)
        snprintf(buf, sizeof buf, "PREV:%d", o.waits[i].seg);
      else if (o.waits[i].kind == -2)
        snprintf(buf, sizeof buf, "HOST:%d", o.waits[i].seg);
      else
        snprintf(buf, sizeof buf, "%s:%d", kind_name(o.waits[i].kind), o.waits[i].seg);
      w += buf;
    }
    char mb[16], sl[16];
    if (o.mb < 0) strcpy(mb, "-"); else snprintf(mb, sizeof mb, "%d", o.mb);
    if (o.slot < 0) strcpy(sl, "-"); else snprintf(sl, sizeof sl, "%d", o.slot);
    snprintf(buf, sizeof buf, "%s %s %d %s %s %s\n", lane_name(o.lane), kind_name(o.kind), o.seg, mb, sl,
             w.empty() ? "-" : w.c_str());
    out += buf;
  }
  return out;
}

// integer-time 4-lane simulation of one step (oracle/schedule.py simulate)
static void simulate(const Eval& ev, const std::vector<int>& ends, const std::vector<Op>& ops, int64_t* makespan,
                     int64_t* hidden_ppm) {
  const int S = (int)ends.size();
  auto seg = [&](const std::vector<int64_t>& p, int k) {
    int i = k == 1 ? 0 : ends[k - 2] + 1, j = ends[k - 1];
    return Eval::s(p, i, j);
  };
  int64_t lane[4] = {0, 0, 0, 0};
  std::map<std::pair<int, int>, int64_t> done;
  std::vector<std::pair<int64_t, int64_t>> comp, copies;
  for (auto& o : ops) {
    int64_t dur = 0;
    switch (o.kind) {
      case K_FWD: dur = seg(ev.ptf, o.seg); break;
      case K_BWD: dur = o.seg == S ? seg(ev.ptb, o.seg) : seg(ev.ptbx, o.seg); break;
      case K_LOAD_F: dur = seg(ev.ptlf, o.seg); break;
      case K_LOAD_B: dur = (o.seg == S && S >= 2) ? seg(ev.ptmv, o.seg) : seg(ev.ptlb, o.seg); break;
      case K_STORE: dur = seg(ev.pts, o.seg); break;
      default: dur = 0;
    }
    int64_t start = lane[o.lane];
    for (auto& w : o.waits)
      if (w.kind >= 0) start = std::max(start, done[{w.kind, w.seg}]);
    int64_t end = start + dur;
    lane[o.lane] = end;
    done[{o.kind, o.seg}] = end;
    if (o.lane == L_COMPUTE && dur > 0) comp.push_back({start, end});
    if ((o.lane == L_H2D || o.lane == L_D2H) && dur > 0) copies.push_back({start, end});
  }
  *makespan = std::max(std::max(lane[0], lane[1]), std::max(lane[2], lane[3]));
  i128 tot = 0, hid = 0;
  for (auto& cp : copies) tot += cp.second - cp.first;
  for (auto& cp : copies)
    for (auto& cm : comp) {
      int64_t lo = std::max(cp.first, cm.first), hi = std::min(cp.second, cm.second);
      if (hi > lo) hid += hi - lo;
    }
  *hidden_ppm = tot ? (int64_t)(hid * 1000000 / tot) : 1000000;
}

static void fill_plan(const Eval& ev, int C, const std::vector<int>& ends, int64_t link, atom_plan_t* p) {
  const ModelDims& dm = ev.dm;
  memset(p, 0, sizeof(*p));
  const int S = (int)ends.size();
  p->n_seg = S;
  for (int i = 0; i < S; ++i) p->seg_end[i] = ends[i];
  p->C = C;
  p->nslot = nslot_for(S);
  const int il = S == 1 ? 0 : ends[S - 2] + 1;
  p->cut_bytes = (int64_t)(S - 1) * dm.wb * dm.M * dm.d;
  p->r1_bytes = ev.r1(ends[0]);
  p->slot_bytes = al256(ev.slot_need(ends));
  p->stash_bytes = stash_bytes(dm, C, ev.nblocks(il, ev.n - 1), S, ev.R);
  const int r = n_rc(dm, ev.R, ev.nblocks(il, ev.n - 1));
  p->n_recompute = r;
  p->act_policy = r == 0 ? ATOM_ACT_STASH : (r == dm.L - ev.nblocks(il, ev.n - 1) ? ATOM_ACT_RECOMPUTE : ATOM_ACT_HYBRID);
  p->work_bytes = work_bytes(dm, C);
  p->device_bytes = p->r1_bytes + p->nslot * p->slot_bytes + p->stash_bytes + p->work_bytes;
  std::vector<int64_t> P;
  for (int t = 0; t < S; ++t) P.push_back(Eval::s(ev.pP, t == 0 ? 0 : ends[t - 1] + 1, ends[t]));
  int64_t h2d = 0, d2h = 0;
  if (S >= 2) {
    const bool hu = ev.c.grad_rounds > 0;
    for (int t = 1; t < S; ++t) h2d += 4 * P[t];
    for (int t = 1; t < S - 1; ++t) h2d += (hu ? 8 : 12) * P[t];
    h2d += (hu ? 4 : 8) * P[S - 1];
    for (int t = 1; t < S; ++t) d2h += (hu ? 4 : 12) * P[t];
  }
  p->pred_h2d_B = h2d;
  p->pred_d2h_B = d2h;
  i128 fl = 0;
  for (int64_t f : ev.k.ff) fl += 3 * (i128)f;
  p->pred_flops = (int64_t)(fl * C);
  p->hbm_budget = ev.budget;
  p->link_bw = link;
  auto ops = emit_schedule(S, C, false, nullptr);
  simulate(ev, ends, ops, &p->pred_step_ns, &p->pred_hidden_ppm);
}

// re-derive the arena sizes of a plan for this cfg (peer creation rejects stale plans)
bool check_plan(const atom_model_cfg& c, const atom_plan_t& p) {
  ModelDims dm;
  if (!make_dims(c, &dm)) return false;
  const int n = dm.n_nodes;
  if (p.n_seg < 1 || p.n_seg > ATOM_MAX_SEG || p.C < 1 || p.seg_end[p.n_seg - 1] != n - 1) {
    set_error("invalid plan: segments / C do not match the model");
    return false;
  }
  std::vector<int> ends(p.seg_end, p.seg_end + p.n_seg);
  for (int i = 0; i < p.n_seg; ++i)
    if (ends[i] < 0 || (i && ends[i] <= ends[i - 1])) {
      set_error("invalid plan: segment ends must ascend");
      return false;
    }
  const int S = p.n_seg;
  const int il = S == 1 ? 0 : ends[S - 2] + 1;
  {
    int nb_last = std::max(0, dm.L - std::max(il, 1) + 1);   // blocks of the last segment
    if (dm.op) {
      nb_last = 0;
      for (int l = 0; l < dm.L; ++l) nb_last += il <= 2 * l + 1 ? 1 : 0;
    }
    const int nb_pre = dm.L - nb_last;
    const int r = p.n_recompute;
    const int want = r == 0 ? ATOM_ACT_STASH : (r == nb_pre ? ATOM_ACT_RECOMPUTE : ATOM_ACT_HYBRID);
    if (r < 0 || r > nb_pre || p.act_policy != want) {
      set_error("invalid plan: act_policy / n_recompute");
      return false;
    }
  }
  Eval ev(c, dm, p.hbm_budget > 0 ? p.hbm_budget : 1, p.link_bw > 0 ? p.link_bw : 1, p.n_recompute);
  if (ev.r1(ends[0]) != p.r1_bytes || al256(ev.slot_need(ends)) != p.slot_bytes || nslot_for(S) != p.nslot ||
      stash_bytes(dm, p.C, ev.nblocks(il, n - 1), S, p.n_recompute) != p.stash_bytes || work_bytes(dm, p.C) != p.work_bytes ||
      p.r1_bytes + p.nslot * p.slot_bytes + p.stash_bytes + p.work_bytes != p.device_bytes) {
    set_error("invalid plan: arena sizes do not match this configuration (plan made for another cfg?)");
    return false;
  }
  return true;
}

bool make_plan(const atom_model_cfg& c, int64_t budget, int64_t link, atom_plan_t* out) {
  ModelDims dm;
  if (!make_dims(c, &dm)) return false;
  if (link <= 0 || (c.peak_flops <= 0 && !c.cost_table) || budget <= 0) {
    set_error("invalid config: link_bw, peak_flops and hbm_budget must be positive");
    return false;
  }
  const int maxC = c.max_C > 0 ? c.max_C : 64;
  if (c.C < 0 || c.C > 4096 || maxC > 4096) {
    set_error("invalid config: C / max_C out of range");
    return false;
  }
  if (c.act_policy < ATOM_ACT_AUTO || c.act_policy > ATOM_ACT_HYBRID ||
      (c.act_policy == ATOM_ACT_HYBRID && (c.n_recompute < 0 || c.n_recompute > dm.L))) {
    set_error("invalid config: act_policy / n_recompute");
    return false;
  }
  std::vector<int> forced;
  if (c.forced_ends) {
    for (int i = 0; i < c.n_forced; ++i) forced.push_back(c.forced_ends[i]);
    bool ok = !forced.empty() && forced.back() == dm.n_nodes - 1 && (int)forced.size() <= ATOM_MAX_SEG;
    for (size_t i = 0; ok && i < forced.size(); ++i)
      ok = forced[i] >= 0 && (i == 0 || forced[i] > forced[i - 1]);
    if (!ok) {
      set_error("invalid config: forced_ends must ascend and end at node %d", dm.n_nodes - 1);
      return false;
    }
  }
  const int c_lo = c.C > 0 ? c.C : 1, c_hi = c.C > 0 ? c.C : maxC;
  const char* first_violation = nullptr;
  int bad_pair = 0;
  // re-forward counts R to try: ACT_AUTO the fewest (0 = full stash, ..., L = every block before
  // the last segment), each over C ascending (R35)
  std::vector<int> pols;
  if (dm.op) {   // operator-granular graph: the full stash only (R40)
    if (c.act_policy != ATOM_ACT_AUTO && c.act_policy != ATOM_ACT_STASH) {
      set_error("invalid config: op_nodes plans use the full activation stash (act_policy AUTO or STASH)");
      return false;
    }
    pols = {0};
  } else if (c.act_policy == ATOM_ACT_AUTO) {
    for (int r = 0; r <= dm.L; ++r) pols.push_back(r);
  } else {
    pols = {c.act_policy == ATOM_ACT_STASH ? 0 : (c.act_policy == ATOM_ACT_RECOMPUTE ? dm.L : c.n_recompute)};
  }
  for (int pol : pols) {
    Eval ev(c, dm, budget, link, pol);
    for (int C = c_lo; C <= c_hi; ++C) {
      std::vector<int> ends;
      if (!forced.empty()) {
        int bp = 0;
        const char* v = ev.violation(C, forced, &bp);
        if (!v) {
          fill_plan(ev, C, forced, link, out);
          return true;
        }
        if (!first_violation) { first_violation = v; bad_pair = bp; }
        continue;
      }
      if (dp_for_C(ev, C, &ends)) {
        if ((int)ends.size() > ATOM_MAX_SEG) {
          set_error("plan needs %d sub-models (> %d)", (int)ends.size(), ATOM_MAX_SEG);
          return false;
        }
        fill_plan(ev, C, ends, link, out);
        return true;
      }
    }
  }
  Eval ev(c, dm, budget, link, pols[0]);
  if (first_violation)
    set_error("no feasible C in [%d, %d] for the forced partition: first violation at C=%d: %s%s", c_lo, c_hi, c_lo,
              first_violation, bad_pair ? " (sub-models around the first failing boundary)" : "");
  else
    set_error("no feasible partition for C in [%d, %d]: the fully resident plan needs %lld bytes of %lld; "
              "swapped plans violate memory or the compute >= load constraints",
              c_lo, c_hi, (long long)ev.device_bytes(c_lo, {dm.n_nodes - 1}), (long long)budget);
  return false;
}

}  // namespace atom
