// Measured profile -> planner inputs ("the model is profiled offline", "We
// empirically determine C offline via profiling for a particular GPU"; SURVEY §8 NEXT-2;
// DESIGN.md R34).  Pure host code over the canonical per-op trace text of one step
// (atom_get_trace: "<lane> <KIND> <seg> <mb|-> <slot|-> <t0_us> <t1_us>" per line):
//
//   * compute rate  = FLOPs the step executes (model FLOPs + the re-forward of the plan's
//                     n_recompute blocks) / busy time of the compute lane (union of its op intervals);
//   * copy rates    = planned bytes per direction / summed op time of that copy lane;
//   * cost table    = per node {t_f, t_b} in ns for one micro-batch (atom_model_cfg.cost_table):
//                     blocks from the blocks-only sub-models (their FWD / BWD op means divided by
//                     their block counts, the backward without the re-forwards), E and H from what
//                     is left of the first / last sub-model; FWD(S) carries the head's forward and
//                     backward, split 1 : 2 as their FLOPs are.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/atom.h"
#include "planner.h"

namespace atom {
void set_error(const char* fmt, ...);

namespace {
struct TraceOp {
  std::string lane, kind;
  int seg = 0;
  double t0 = 0, t1 = 0;   // us
};

bool parse_trace(const char* text, std::vector<TraceOp>* out) {
  std::istringstream in(text ? text : "");
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    TraceOp o;
    std::string mb, slot;
    if (!(ls >> o.lane >> o.kind >> o.seg >> mb >> slot >> o.t0 >> o.t1)) {
      set_error("atom_profile: malformed trace line '%s'", line.c_str());
      return false;
    }
    out->push_back(o);
  }
  return true;
}

// union of the compute lane's op intervals (us)
double compute_busy_us(const std::vector<TraceOp>& ops) {
  std::vector<std::pair<double, double>> iv;
  for (auto& o : ops)
    if (o.lane == "compute") iv.push_back({o.t0, o.t1});
  std::sort(iv.begin(), iv.end());
  double busy = 0, cs = 0, ce = -1e300;
  for (auto& p : iv) {
    if (p.first > ce) {
      if (ce > -1e300) busy += ce - cs;
      cs = p.first;
      ce = p.second;
    } else {
      ce = std::max(ce, p.second);
    }
  }
  if (ce > -1e300) busy += ce - cs;
  return busy;
}

double lane_us(const std::vector<TraceOp>& ops, const char* lane) {
  double t = 0;
  for (auto& o : ops)
    if (o.lane == lane) t += o.t1 - o.t0;
  return t;
}
}  // namespace

// FLOPs one planned step executes: the model FLOPs plus the re-forward of blocks 1..n_recompute
// (QKV, attention-projection and fc GEMMs, 16 d^2 per token, and the attention forward,
// 2 d (T + 1) per token; R28, R35)
double executed_flops(const atom_model_cfg& cfg, const atom_plan_t& plan) {
  const double d = cfg.d_model, T = cfg.seq_len;
  const double tokens = (double)plan.C * cfg.micro_batch * cfg.seq_len;
  return (double)plan.pred_flops + plan.n_recompute * tokens * (16.0 * d * d + 2.0 * d * (T + 1));
}

bool profile_from_trace(const char* trace, const atom_model_cfg& cfg, const atom_plan_t& plan, atom_profile_t* out,
                        int64_t* table, int64_t cap) {
  std::vector<TraceOp> ops;
  if (!parse_trace(trace, &ops)) return false;
  memset(out, 0, sizeof(*out));
  const int L = cfg.n_layer, S = plan.n_seg;
  out->n_nodes = (cfg.op_nodes ? 2 * L : L) + 2;
  const double busy = compute_busy_us(ops);
  out->compute_busy_ms = busy / 1000.0;
  out->executed_flops = executed_flops(cfg, plan);
  out->flops_per_s = busy > 0 ? out->executed_flops / (busy * 1e-6) : 0;
  const double h2d = lane_us(ops, "h2d"), d2h = lane_us(ops, "d2h");
  out->h2d_bytes_per_s = h2d > 0 ? (double)plan.pred_h2d_B / (h2d * 1e-6) : 0;
  out->d2h_bytes_per_s = d2h > 0 ? (double)plan.pred_d2h_B / (d2h * 1e-6) : 0;
  // per (KIND, segment) mean op time of the compute lane over its micro-batches
  std::map<std::pair<std::string, int>, std::pair<int, double>> acc;
  for (auto& o : ops)
    if (o.lane == "compute") {
      auto& a = acc[{o.kind, o.seg}];
      a.first += 1;
      a.second += o.t1 - o.t0;
    }
  auto mean = [&](const char* kind, int k, double* v) {
    auto it = acc.find({kind, k});
    if (it == acc.end()) return false;
    *v = it->second.second / it->second.first;
    return true;
  };
  std::vector<int> lo(S), nblk(S), nrc(S);
  for (int k = 0; k < S; ++k) {
    lo[k] = k == 0 ? 0 : plan.seg_end[k - 1] + 1;
    nblk[k] = nrc[k] = 0;
    for (int v = lo[k]; v <= plan.seg_end[k]; ++v) {
      if (v >= 1 && v <= L) nblk[k]++;
      if (k < S - 1 && v >= 1 && v <= plan.n_recompute) nrc[k]++;
    }
  }
  // blocks-only sub-models (not the interleaved last one) with a traced FWD and BWD
  double sf = 0, sb = 0;
  int nb = 0, nr = 0;
  for (int k = 0; k < S - 1; ++k) {
    bool only = true;
    for (int v = lo[k]; v <= plan.seg_end[k]; ++v) only = only && v >= 1 && v <= L;
    double f, b;
    if (!only || !mean("FWD", k + 1, &f) || !mean("BWD", k + 1, &b)) continue;
    sf += f;
    sb += b;
    nb += nblk[k];
    nr += nrc[k];
  }
  // no table: the plan has no blocks-only sub-model, or the graph is operator-granular (R40: its
  // halves would need per-half op times the per-sub-model trace does not separate); the caller
  // keeps the measured rates
  if (nb == 0 || cfg.op_nodes) return true;
  const double tf_b = sf / nb;
  const double tb_b = (sb - tf_b * nr) / nb;
  double f1 = 0, b1 = 0, fS = 0;
  mean("FWD", 1, &f1);
  mean("BWD", 1, &b1);
  mean("FWD", S, &fS);
  const double tf_e = lo[0] == 0 ? std::max(f1 - nblk[0] * tf_b, 0.0) : 0.0;
  const double tb_e = std::max(b1 - nblk[0] * tb_b - nrc[0] * tf_b, 0.0);
  const double head = std::max(fS - nblk[S - 1] * tf_b, 0.0);
  auto ns = [](double us) { return (int64_t)std::max(llround(us * 1000.0), 1LL); };
  const int64_t need = 2 * (int64_t)(L + 2);
  if (table) {
    if (cap < need) {
      set_error("atom_profile: cost table needs %lld entries", (long long)need);
      return false;
    }
    table[0] = ns(tf_e);
    table[1] = ns(tb_e);
    for (int l = 0; l < L; ++l) {
      table[2 + 2 * l] = ns(tf_b);
      table[3 + 2 * l] = ns(tb_b);
    }
    table[need - 2] = ns(head / 3.0);
    table[need - 1] = ns(2.0 * head / 3.0);
  }
  out->have_table = 1;
  return true;
}

}  // namespace atom

extern "C" atom_status atom_profile_trace(const char* trace, const atom_model_cfg* cfg, const atom_plan_t* plan,
                                          int64_t* cost_table, int64_t cap, atom_profile_t* out) {
  if (!trace || !cfg || !plan || !out || plan->n_seg < 1 || plan->n_seg > ATOM_MAX_SEG) {
    atom::set_error("atom_profile_trace: invalid arguments");
    return ATOM_E_INVALID;
  }
  return atom::profile_from_trace(trace, *cfg, *plan, out, cost_table, cap) ? ATOM_OK : ATOM_E_INVALID;
}
