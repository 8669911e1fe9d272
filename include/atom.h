/*
 * atom.h -- C-ABI of libatom: the per-peer training step of Atom (arXiv 2403.10504) on B200.
 *
 * The method (PAPER.md = P, SPEC.md = S, line numbers):
 *   - the whole model lives in host memory; contiguous runs of transformer layers
 *     ("sub-models") are swapped into the GPU and executed one after another
 *     ("houses the entire model in a single server's host memory ... memory
 *     swapping technique to transfer model portions to the GPU");
 *   - the partition is chosen offline so that every sub-model fits and the compute of
 *     one sub-model overlaps the loading of the next, with gradient accumulation over
 *     C mini-batches stretching the compute (Algorithm 1);
 *   - one stream executes, another prefetches the next sub-model "immediately after the
 *     current sub-model starts"; the last forward sub-model and the first sub-model are
 *     not swapped out;
 *   - whole-model replicas ("peers") train independently and periodically average their
 *     parameters with an allreduce.
 *
 * Calls: atom_plan (static analysis, pure host), atom_peer_create, atom_step (one swapped
 * forward + backward + update), atom_sync (peer averaging), plus inspection calls.
 *
 * Conventions
 *   - Every function returns atom_status (0 = ATOM_OK).  No C++ exception crosses the ABI.
 *     On failure atom_last_error() returns a thread-local message naming the violated
 *     constraint or the failing CUDA/NCCL call.
 *   - Pointers are plain host or device pointers as stated per argument.  Input buffers are
 *     only read during the call.  The device arena is caller-owned (allocated by PyTorch);
 *     pinned host arenas, streams, events and the NCCL communicator are library-owned and
 *     released by atom_peer_destroy.
 *   - After a CUDA or NCCL failure a peer is poisoned: every later call on it returns
 *     ATOM_E_STATE.
 *   - Canonical parameter order (init_params / atom_get_params): nodes E, B_0..B_{L-1}, H;
 *     E = wte[V,d], wpe[T,d]; block = ln1.g[d], ln1.b[d], W_qkv[3d,d], b_qkv[3d], W_o[d,d],
 *     b_o[d], ln2.g[d], ln2.b[d], W_fc[4d,d], b_fc[4d], W_pr[d,4d], b_pr[d];
 *     H = lnf.g[d], lnf.b[d], W_lm[V,d] (untied, no bias).  Row-major, fp32, unpadded.
 */
#ifndef ATOM_H
#define ATOM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ATOM_OK = 0,
  ATOM_E_INVALID = -1,    /* invalid configuration / argument (S:61 InvalidConfig)             */
  ATOM_E_INFEASIBLE = -2, /* no partition / no C satisfies the constraints        */
  ATOM_E_CAPACITY = -3,   /* device arena smaller than plan.device_bytes (S:230 CapacityViolated) */
  ATOM_E_CUDA = -4,
  ATOM_E_NCCL = -5,
  ATOM_E_OOM = -6,        /* pinned host allocation failed                                        */
  ATOM_E_STATE = -7       /* peer poisoned by an earlier failure                                 */
} atom_status;

enum { ATOM_FP32 = 0, ATOM_BF16 = 1 };        /* compute dtype of weights and activations       */
/* activation policy: STASH keeps every block's forward tensors for all C micro-batches;
 * RECOMPUTE keeps only each block's input and re-runs its forward inside the backward
 * (sub-models before the interleaved last one); HYBRID does that for blocks 1..n_recompute only;
 * AUTO = the fewest re-forwarded blocks R = 0 (STASH), 1, ..., L that make a plan feasible, then
 * the smallest C (R35) */
enum { ATOM_ACT_AUTO = 0, ATOM_ACT_STASH = 1, ATOM_ACT_RECOMPUTE = 2, ATOM_ACT_HYBRID = 3 };
#define ATOM_MAX_SEG 256

/* Model and training configuration.  Caller-owned, read-only during every call. */
typedef struct {
  int32_t n_layer, d_model, n_head, seq_len, vocab, micro_batch; /* L, d, h, T, V, b (b sequences/micro-batch) */
  int32_t dtype;          /* ATOM_FP32 (parity path, SIMT kernels) | ATOM_BF16 (performance path, tcgen05)   */
  int32_t C;              /* micro-batches per step; 0 = planner picks the smallest feasible C       */
  int32_t max_C;          /* upper end of the C search (default 64)                                  */
  int32_t act_policy;     /* ATOM_ACT_AUTO | ATOM_ACT_STASH | ATOM_ACT_RECOMPUTE | ATOM_ACT_HYBRID          */
  int32_t overlap_check;  /* 1 = enforce the compute >= load constraints (Alg. 1 line 4); 0 = memory only    */
  int64_t peak_flops;     /* FLOP/s of the analytic cost model (e.g. measured bf16 GEMM peak)               */
  int64_t d2h_bw;         /* device->host bytes/s; 0 = same as link_bw                                       */
  int64_t state_budget;   /* 0 = none; else cap on device bytes of model state (resident segment 1 + slots):
                             the paper's sub-model "GPU capacity"                         */
  const int64_t* cost_table; /* NULL = analytic; else 2*(L+2) int64 {t_f_ns, t_b_ns} per node (profiled) */
  const int32_t* forced_ends; /* NULL = search; else n_forced ascending segment end-node indices to validate */
  int32_t n_forced;
  float lr, beta1, beta2, eps, weight_decay; /* AdamW (eps/wd: torch defaults, R19)          */
  int32_t warmup_steps;   /* linear warm-up length in steps (3000)                                    */
  int32_t sync_every;     /* average parameters every K steps; 0 = only when atom_sync() asks               */
  int32_t n_recompute;    /* ATOM_ACT_HYBRID: blocks 1..n_recompute (0..L) are re-forwarded in the backward */
  int32_t grad_rounds;    /* 0: fused GPU AdamW on every swapped-in sub-model, every step (north star).
                             R >= 1: the paper's update placement (P:563 CPU AdamW; R37): each
                             atom_step is one gradient round; sub-models 2..S accumulate their fp32
                             gradients in a host arena across R rounds (the backward loads the running sum
                             with the master and stores it back: 8 + 4 B/param per round instead of 12 + 12)
                             and every R-th round a multi-threaded CPU AdamW updates their host master,
                             m and v with the mean gradient; the resident sub-model 1 accumulates on the
                             device and takes the same update on the GPU                                 */
  int32_t cpu_threads;    /* CPU AdamW threads (0 = all online cores)                                       */
  float dropout_p;        /* minGPT dropout (embd / attn / resid sites; R38), 0 <= p < 1;
                             masks from Philox4x32-10 keyed by dropout_seed, counter (i / 8, site, layer,
                             micro_step), micro_step = (atom_step calls so far) * C + micro-batch            */
  int32_t op_nodes;       /* 1 = operator-granular graph ("a node ... is a layer or an operator"):
                             each block is two nodes, its attention half (LN1, QKV, attention, output
                             projection) and its MLP half (LN2, fc, GELU, fc2); nodes E, A_0, M_0, ...,
                             A_{L-1}, M_{L-1}, H, so a sub-model may end in the middle of a block.  The
                             full activation stash only (R40); cost_table then has 2 (2L+2)
                             entries                                                                     */
  uint64_t dropout_seed;
} atom_model_cfg;

/* The plan: plain data, fixed capacity, no pointers.  Produced by atom_plan.  Node indices: 0 = E,
 * blocks 1..L (op_nodes: 2l+1 = attention half of block l, 2l+2 = its MLP half), last = H. */
typedef struct {
  int32_t n_seg;                  /* S: number of sub-models                                            */
  int32_t seg_end[ATOM_MAX_SEG];  /* last node index of each sub-model (nodes 0=E, 1..L blocks, L+1=H)  */
  int32_t C;                      /* micro-batches per step                                             */
  int32_t nslot;                  /* rotating device slots for sub-models 2..S (0, 2 or 3)              */
  int32_t act_policy;             /* resolved activation policy (STASH, RECOMPUTE or HYBRID)            */
  int64_t cut_bytes;              /* activation bytes crossing sub-model boundaries per micro-batch      */
  int64_t r1_bytes;               /* resident sub-model 1 (weights + grad + master + m + v)              */
  int64_t slot_bytes;             /* one slot: the largest swapped sub-model's state                    */
  int64_t stash_bytes;            /* activation stash                                                   */
  int64_t work_bytes;             /* working set                                                        */
  int64_t device_bytes;           /* total device arena = r1 + nslot*slot + stash + work                 */
  int64_t pred_step_ns;           /* integer-time simulation of one step (3 lanes)                      */
  int64_t pred_hidden_ppm;        /* predicted share of copy time overlapped by compute (ppm)           */
  int64_t pred_h2d_B, pred_d2h_B; /* host<->device bytes per step                                       */
  int64_t pred_flops;             /* model FLOPs per step (fwd + bwd)                                   */
  int64_t hbm_budget, link_bw;    /* the inputs the plan was made for                                   */
  int32_t n_recompute;            /* blocks re-forwarded in the backward (1..n_recompute; 0 = STASH)    */
  int32_t reserved;
} atom_plan_t;

/* Static analysis.  Pure, deterministic, no device needed.
 * hbm_budget: max device arena bytes; link_bw: host->device bytes/s.
 * Objective: min total cut bytes, then fewer sub-models, then the
 * lexicographically smallest end vector; C = smallest feasible.
 * Errors: ATOM_E_INVALID (bad cfg), ATOM_E_INFEASIBLE (message names the first violated constraint). */
atom_status atom_plan(const atom_model_cfg* cfg, int64_t hbm_budget, int64_t link_bw, atom_plan_t* out);

/* The step program as canonical text, one op per line:
 *   "<lane> <KIND> <seg> <mb|-> <slot|-> <waits|->"   lanes: compute h2d d2h comm.
 * sync != 0 emits a parameter-averaging step.  Writes at most cap bytes (NUL-terminated when it
 * fits); *len = full length without the NUL.  ATOM_E_INVALID if buf is too small. */
atom_status atom_plan_schedule(const atom_plan_t* plan, int32_t sync, char* buf, int64_t cap, int64_t* len);

/* NCCL unique id for peer averaging (128 bytes written to out).  Call on one rank and
 * broadcast it (e.g. through a torch.distributed group). */
atom_status atom_nccl_unique_id(void* out128);

typedef struct atom_peer atom_peer; /* opaque, library-owned */

/* Create one peer (one whole-model replica) on CUDA device `device`.
 *   device_arena / arena_bytes: caller-owned device memory (>= plan->device_bytes, 256-byte aligned);
 *   init_params: host fp32 [N] in canonical order, or NULL to draw the minGPT init on the device
 *                from `seed` (normal(0, 0.02), residual projections 0.02/sqrt(2L), biases 0, LN 1/0);
 *   nccl_id: 128-byte id from atom_nccl_unique_id (NULL when nranks == 1); rank in [0, nranks).
 * Pins host arenas (12 B/param: fp32 master, m, v) and makes segment 1 resident.
 * Errors: ATOM_E_INVALID, ATOM_E_CAPACITY, ATOM_E_OOM, ATOM_E_CUDA, ATOM_E_NCCL. */
atom_status atom_peer_create(const atom_model_cfg* cfg, const atom_plan_t* plan, int32_t device, void* device_arena,
                             int64_t arena_bytes, const float* init_params, uint64_t seed, const void* nccl_id,
                             int32_t nranks, int32_t rank, atom_peer** out);

/* One training step: swapped forward, backward and AdamW over C micro-batches.
 *   tokens: HOST int32 [C*b, T+1] (inputs = [:, :T], targets = [:, 1:]), copied before return;
 *   loss_out: mean token cross-entropy of the step (fp32).
 * Returns once the loss is on the host; the tail of the backward keeps running on the device
 * and overlaps the next step (P:307 locality).  Steps are ordered on the device. */
atom_status atom_step(atom_peer* peer, const int32_t* tokens, float* loss_out);

/* Same, with the tokens already resident in device memory (int32 [C*b, T+1]). */
atom_status atom_step_device(atom_peer* peer, const int32_t* tokens_dev, float* loss_out);

/* Peer averaging: p <- mean over all ranks' peers of p (fp32 master; m, v stay local).
 * Collective over all ranks (each rank passes its local peers).  flush == 0 marks the next step as a
 * sync step (the allreduce runs per sub-model inside that step's backward swap window, between AdamW
 * and the swap-out, overlapped with the compute of the next sub-model); flush != 0 averages now
 * (standalone pass over all sub-models).  Returns after enqueueing (flush == 0) or completion. */
atom_status atom_sync(atom_peer* const* peers, int32_t n_local, int32_t flush);

/* Membership changes ("peers join and leave"; P:563 GPUs killed mid-training).
 * The host-side registry (paper_2403_10504_b200/elastic.py) decides who is a member; these calls
 * only rebuild the averaging communicator and bring a joiner up to date.  All are collective over
 * the members of the NEW membership and must be called between steps (no sync step in flight).
 *
 * atom_comm_reset: drop the current communicator (aborted: members that died cannot answer) and
 *   join a new one from a fresh 128-byte id (atom_nccl_unique_id on one member, shared through the
 *   registry); nranks == 1 leaves the peer without a communicator (sync steps become local no-ops).
 * atom_comm_shrink: ncclCommShrink of the current communicator without the listed ranks (failed or
 *   leaving peers; abort_ops != 0 first terminates operations of the parent that cannot complete);
 *   the peer's rank / nranks become its position in the shrunk communicator.
 * atom_broadcast_state: root sends its fp32 master, AdamW m, v and optimizer step count; members
 *   with adopt != 0 (joiners: "fetch the current model") overwrite theirs, the others only
 *   take part.  Root's state is unchanged.
 * Errors: ATOM_E_INVALID, ATOM_E_STATE (poisoned peer), ATOM_E_NCCL, ATOM_E_CUDA. */
atom_status atom_comm_reset(atom_peer* peer, const void* nccl_id, int32_t nranks, int32_t rank);
atom_status atom_comm_shrink(atom_peer* peer, const int32_t* exclude_ranks, int32_t n_exclude, int32_t abort_ops);
atom_status atom_broadcast_state(atom_peer* peer, int32_t root, int32_t adopt);
/* The peer's averaging rank / size and optimizer step count. */
atom_status atom_peer_info(atom_peer* peer, int32_t* rank, int32_t* nranks, int64_t* step);

/* Copy the peer's fp32 master parameters and AdamW moments (canonical order, [N] each) to host
 * buffers; NULL skips one.  Waits for all outstanding work of the peer. */
atom_status atom_get_params(atom_peer* peer, float* master_out, float* m_out, float* v_out);

/* Per-op trace of the last completed step: one line per issued op,
 *   "<lane> <KIND> <seg> <mb|-> <slot|-> <t_start_us> <t_end_us>"
 * (device timestamps from CUDA events, relative to the step start).  Same buffer rules as
 * atom_plan_schedule. */
atom_status atom_get_trace(atom_peer* peer, char* buf, int64_t cap, int64_t* len);

/* Counters since creation (or the last reset) for measurement. */
typedef struct {
  int64_t steps;
  int64_t kernel_launches;        /* kernels launched by the library                                   */
  int64_t gemm_launches;          /* GEMM launches (the dominant kernel)                               */
  double gemm_ms;                 /* summed CUDA-event duration of GEMM launches (when timing is on)   */
  double gemm_flops;              /* algorithmic FLOPs of those launches                               */
  double h2d_bytes, d2h_bytes;    /* bytes copied host<->device by the swap engine                     */
  double copy_ms, copy_hidden_ms; /* summed copy time and the part overlapping compute (last step)    */
  double step_ms;                 /* device time of the last step (first op start -> last op end)     */
  double h2d_ms, h2d_hidden_ms;   /* copy_ms / copy_hidden_ms split by direction: host -> device ...   */
  double d2h_ms, d2h_hidden_ms;   /* ... and device -> host (last step, both)   */
  double compute_busy_ms;         /* union of the compute lane's FWD/BWD/ADAM/... op intervals         */
  double compute_span_ms;         /* compute lane: first op start -> last op end (last step)           */
  double host_issue_ms;           /* host wall time atom_step spent issuing the last step's work       */
} atom_stats_t;
atom_status atom_get_stats(atom_peer* peer, atom_stats_t* out);
/* GEMM time per shape since the last reset (timing on): one line per distinct launch shape,
 *   "<M> <N> <K> <a_mn> <b_mn> <epilogue> <launches> <ms> <TFLOP/s>"
 * (ms summed over the launches' CUDA-event durations).  Same buffer rules as atom_plan_schedule. */
atom_status atom_get_gemm_log(atom_peer* peer, char* buf, int64_t cap, int64_t* len);
/* Device time per kernel category since the last reset (timing on): one line per category,
 *   "<category> <launch groups> <ms>"   categories: gemm_fwd gemm_dgrad gemm_wgrad attn_fwd attn_bwd
 *   layernorm colsum gelu cross_entropy embedding adamw cast
 * (timing level 2: CUDA events around each launch group on its own stream; with the side streams
 * on, the categories overlap in time).  Same buffer rules as atom_plan_schedule. */
atom_status atom_get_kernel_log(atom_peer* peer, char* buf, int64_t cap, int64_t* len);
/* Measured profile ("profiled offline", "determine C offline via profiling"; DESIGN.md
 * R34): what the planner needs, derived from the per-op trace of the peer's last step.
 *   flops_per_s      FLOPs the step executes (model + re-forward) / compute-lane busy time
 *   h2d / d2h        planned bytes per direction / summed op time of that copy lane
 *   cost_table       per node {t_f_ns, t_b_ns} for one micro-batch, the atom_model_cfg.cost_table
 *                    layout (nodes E, B_0..B_{L-1}, H): blocks from the blocks-only sub-models,
 *                    E / H from the rest of the first / last sub-model; have_table = 0 when the plan
 *                    has no blocks-only sub-model (then only the rates are measured).
 * cost_table: caller-owned int64 [cap >= 2 (L + 2)] or NULL.  ATOM_E_INVALID on a malformed trace or
 * a short buffer. */
typedef struct {
  double flops_per_s, h2d_bytes_per_s, d2h_bytes_per_s;
  double compute_busy_ms, executed_flops;
  int32_t n_nodes, have_table;
} atom_profile_t;
atom_status atom_profile(atom_peer* peer, int64_t* cost_table, int64_t cap, atom_profile_t* out);
/* The same derivation from trace text in atom_get_trace's format and the plan it ran (pure host). */
atom_status atom_profile_trace(const char* trace, const atom_model_cfg* cfg, const atom_plan_t* plan,
                               int64_t* cost_table, int64_t cap, atom_profile_t* out);
/* Reset counters; timing >= 1 brackets every GEMM launch with CUDA events (GEMM-time roofline),
 * timing >= 2 also every other launch group (atom_get_kernel_log). */
atom_status atom_reset_stats(atom_peer* peer, int32_t timing);

/* Wait for all outstanding device work of the peer, release everything it owns. */
atom_status atom_peer_destroy(atom_peer* peer);

/* Thread-local message of the last failure on this thread. */
const char* atom_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ATOM_H */
