// atom_peer: one whole-model replica on one B200 ("volunteer nodes ...
// independently train a copy of the complete model").
#pragma once
#include <nccl.h>

#include <map>
#include <vector>

#include "../../include/atom.h"
#include "kernels.h"
#include "planner.h"

struct atom_peer {
  atom_model_cfg cfg{};
  atom_plan_t plan{};
  atom::ModelDims dm;
  int device = 0;
  int S = 0, C = 0;
  std::vector<int> seg_lo, seg_hi;      // node range of each segment (1-based index k -> [k-1])
  std::vector<int64_t> seg_P, seg_off;  // padded params and padded offset of each segment
  std::vector<int> seg_of_node;         // node -> segment index (1-based)
  int nb_last = 0;                      // blocks in the last segment
  int l0_last = -1;                     // first block (0-based) of the last segment, -1 if none

  // ---- device arena (caller-owned) ----
  uint8_t* arena = nullptr;
  int64_t arena_bytes = 0;
  uint8_t* r1 = nullptr;                // resident segment 1 state
  std::vector<uint8_t*> slot_phys;      // physical slot base addresses, indexed by LOGICAL slot id
  std::vector<cudaEvent_t> slot_rel;    // per physical slot address: event of its last release (or null)
  std::map<uint8_t*, cudaEvent_t> rel_of;
  uint8_t* stash = nullptr;
  int policy = ATOM_ACT_STASH;          // resolved activation policy of the plan
  int n_recompute = 0;                  // blocks 1..n_recompute re-forward inside their backward
  // host update placement (cfg.grad_rounds = R > 0, R37): this step's gradient round
  // (0..R-1), whether it ends with an update, and the host gradient sums of sub-models 2..S
  int round = 0;
  bool upd_round = true;
  float* h_gacc = nullptr;
  std::vector<int64_t> blk_off;         // per block: byte offset (from stash) of its first stash entry
  std::vector<char> blk_full;           // per block: full entries (1) or input checkpoints only (0)
  int64_t rc_off = -1;                  // byte offset of the entry the backward re-forward fills
  uint8_t* hfin = nullptr;
  // working set
  int32_t* tokens = nullptr;
  uint8_t* dh = nullptr;                // [C][M][d] boundary gradient
  float* losses = nullptr;              // [C*M]
  uint8_t* scratch = nullptr;
  int64_t scratch_bytes = 0;
  float* red = nullptr;
  int* emb = nullptr;
  float* loss_dev = nullptr;
  int* red_ticket = nullptr;            // CS_TICKETS zeroed ints (column-sum kernels)

  // ---- host arenas (library-owned, pinned), padded canonical layout ----
  float* h_master = nullptr;
  float* h_m = nullptr;
  float* h_v = nullptr;
  int32_t* h_tokens = nullptr;          // pinned staging
  float* h_loss = nullptr;

  // ---- streams / events ----
  cudaStream_t s_comp = nullptr, s_h2d = nullptr, s_d2h = nullptr, s_comm = nullptr;
  // block backward: weight-gradient GEMMs that no later kernel of the block waits for run on a
  // side stream, filling the SMs their tile tails (and the main stream's HBM-bound kernels) leave
  // idle; ev_side[0] forks, ev_side[1..3] mark the WFC / WO / WQKV gradients done
  cudaStream_t s_side = nullptr;
  cudaStream_t s_attn = nullptr;        // the attention backward's dQ kernel, beside dK/dV
  cudaStream_t s_cpu = nullptr;         // CPU AdamW host functions (R37), off the copy streams
  std::vector<cudaEvent_t> cpu_ev;      // per segment: its last CPU AdamW finished (index k - 1)
  std::vector<char> cpu_ev_set;
  cudaEvent_t ev_side[4] = {nullptr, nullptr, nullptr, nullptr};
  bool side_wgrad = true;
  std::map<std::pair<int, int>, cudaEvent_t> op_ev;  // (kind, seg) -> completion event
  // layer-by-layer loading: every LOAD_F / LOAD_B records one event per node (layer) on the
  // h2d stream; a sub-model's CAST is deferred into its first FWD / BWD op, which waits for each
  // layer's event and casts that layer right before computing it
  std::vector<cudaEvent_t> node_ev;
  std::vector<char> cast_pending;       // per segment (index k - 1)
  cudaEvent_t ev_loss = nullptr;

  // ---- NCCL ----
  // guarded averaging (R36): per segment an "all arrived" flag (int, min over ranks) reduced after
  // the master's out-of-place average; the commit copies the average over the master only when
  // every rank's allreduce of that segment completed
  int* avg_flags = nullptr;             // device: [0] = 1 (this rank's contribution), [1 + k - 1] per segment
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;

  // ---- schedule ----
  std::vector<atom::Op> ops, ops_sync;
  std::vector<int> endq, endq_sync;
  int64_t t = 0;                        // optimizer step count
  int64_t rng_step = 0;                 // atom_step calls so far (dropout micro_step = rng_step * C + mb)
  bool sync_next = false;
  bool poisoned = false;

  // ---- trace / stats ----
  std::vector<cudaEvent_t> trace_ev;    // 2 per op of the last step
  std::vector<atom::Op> trace_ops;
  cudaEvent_t step_start = nullptr, step_end = nullptr;
  bool have_trace = false;
  int timing = 0;
  std::vector<cudaEvent_t> gemm_ev;
  std::vector<double> gemm_fl;
  std::vector<std::string> gemm_key;    // "M N K a_mn b_mn epilogue" of each timed launch
  std::map<std::string, std::pair<int64_t, double>> gemm_by_shape;   // launches, ms (since reset)
  size_t gemm_n = 0;
  // per kernel category (timing on): CUDA events around every launch group of the compute lane
  std::vector<cudaEvent_t> kt_ev;       // pairs
  std::vector<int> kt_cat;
  size_t kt_n = 0;
  double kt_ms[16] = {0};
  int64_t kt_count[16] = {0};
  int64_t steps = 0, gemm_launches = 0;
  unsigned long long launch_base = 0;
  double h2d_bytes = 0, d2h_bytes = 0;
  double gemm_ms_acc = 0, gemm_fl_acc = 0;
  double host_issue_ms = 0;
};
