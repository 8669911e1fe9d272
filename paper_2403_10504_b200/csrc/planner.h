// Partition planner and swap-schedule emitter (host-only, pure, deterministic).
// PAPER.md §III-D (Algorithm 1) and §IV; cost model and readings in
// DESIGN.md §4.  Integer arithmetic only (int64 with __int128 products).
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/atom.h"

namespace atom {

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t al(int64_t x, int64_t a) { return ceil_div(x, a) * a; }
inline int64_t al64(int64_t x) { return al(x, 64); }
inline int64_t al256(int64_t x) { return al(x, 256); }
constexpr int RED_ROWS = 128;   // rows per partial-sum chunk of the deterministic column reductions

// Parameter tensors of one node, in canonical order: element counts and padded offsets.
struct TensorSlot {
  int64_t n;       // elements
  int64_t off;     // padded offset within the node (multiple of 64 elements)
  int64_t canon;   // offset within the node in the unpadded canonical vector
};
enum BlockTensor { T_LN1G, T_LN1B, T_WQKV, T_BQKV, T_WO, T_BO, T_LN2G, T_LN2B, T_WFC, T_BFC, T_WPR, T_BPR, T_NBLOCK };
enum ETensor { T_WTE, T_WPE };
enum HTensor { T_LNFG, T_LNFB, T_WLM };

struct ModelDims {
  int L, d, h, T, V, b;
  int op = 0;  // operator-granular nodes: block l = attention half 2l+1 + MLP half 2l+2 (atom_model_cfg.op_nodes)
  int64_t M;  // b*T
  int dtype;  // ATOM_FP32 / ATOM_BF16
  int wb;     // bytes per compute-dtype element (4 / 2)
  int n_nodes;
  std::vector<std::vector<TensorSlot>> tensors;  // per node
  std::vector<int64_t> P;                        // padded params per node
  std::vector<int64_t> P_canon;                  // unpadded params per node
  std::vector<int64_t> node_off;                 // padded offset of node in the whole model
  std::vector<int64_t> node_canon;               // canonical offset of node
  int64_t N_pad = 0, N_canon = 0;
};
bool make_dims(const atom_model_cfg& c, ModelDims* out);
// node of block l's half (0 = attention: LN1 .. b_o, 1 = MLP: LN2 .. b_pr) and the index of block
// tensor t (BlockTensor) inside that node
inline int blk_node(const ModelDims& m, int l, int half) { return m.op ? 1 + 2 * l + half : 1 + l; }
inline int blk_tensor_node(const ModelDims& m, int l, int t) { return blk_node(m, l, t >= T_LN2G ? 1 : 0); }
inline int blk_tensor_idx(const ModelDims& m, int t) { return m.op && t >= T_LN2G ? t - T_LN2G : t; }
inline bool is_block_node(const ModelDims& m, int i) { return i >= 1 && i <= m.n_nodes - 2; }
inline int node_block(const ModelDims& m, int i) { return m.op ? (i - 1) / 2 : i - 1; }
// 0 = whole block, 1 = attention half, 2 = MLP half (block nodes only)
inline int node_half(const ModelDims& m, int i) { return m.op ? 1 + (i - 1) % 2 : 0; }

struct Costs {
  std::vector<int64_t> P, tf, tb, tlf, tlb, tmv, ts;
  std::vector<int64_t> tbr;  // backward incl. the block re-forward (ATOM_ACT_RECOMPUTE)
  std::vector<int64_t> ff;  // forward FLOPs per micro-batch
};
Costs node_costs(const atom_model_cfg& c, const ModelDims& dm, int64_t link_bw);

// memory model (bytes), DESIGN.md §4
int64_t seg_need(const ModelDims& dm, int64_t P_seg);
int64_t stash_blk_bytes(const ModelDims& dm);
int64_t hfin_bytes(const ModelDims& dm);
int n_rc(const ModelDims& dm, int R, int nb_last);
int64_t stash_bytes(const ModelDims& dm, int C, int nb_last, int S, int R);
int64_t work_bytes(const ModelDims& dm, int C);
int nslot_for(int S);

// planning
bool make_plan(const atom_model_cfg& c, int64_t hbm_budget, int64_t link_bw, atom_plan_t* out);
bool check_plan(const atom_model_cfg& c, const atom_plan_t& p);

// ---- schedule ----
enum Lane { L_COMPUTE = 0, L_H2D = 1, L_D2H = 2, L_COMM = 3 };
enum OpKind { K_CAST, K_FWD, K_BWD, K_FREE, K_ADAM, K_AVG, K_RECAST, K_LOAD_F, K_LOAD_B, K_STORE };
struct Wait {
  int kind;  // OpKind; -1 = release of slot `seg` in the previous step (PREV);
             // -2 = previous step's STORE of segment `seg` (HOST: host arena up to date)
  int seg;
};
struct Op {
  int lane, kind, seg, mb, slot;
  std::vector<Wait> waits;
};
std::vector<Op> emit_schedule(int S, int C, bool sync, std::vector<int>* end_queue);
std::string schedule_text(const std::vector<Op>& ops);
const char* lane_name(int lane);
const char* kind_name(int kind);

}  // namespace atom
