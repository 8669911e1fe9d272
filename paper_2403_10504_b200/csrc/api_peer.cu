// C-ABI: peer lifecycle, training step, peer averaging, inspection (include/atom.h).
#include <string.h>

#include <string>

#include "peer.h"

namespace atom {
bool peer_create(atom_peer* p, const float* init_params, uint64_t seed, const void* nccl_id);
bool peer_step(atom_peer* p, const int32_t* tokens, bool on_device, float* loss);
bool peers_flush_average(atom_peer* const* ps, int n);
bool peer_broadcast_state(atom_peer* p, int root, bool adopt);
bool peer_comm_reset(atom_peer* p, const void* nccl_id, int nranks, int rank);
bool peer_comm_shrink(atom_peer* p, const int* exclude, int n_exclude, bool abort_ops);
bool peer_get_params(atom_peer* p, float* master, float* m, float* v);
bool peer_trace(atom_peer* p, std::string* out, atom_stats_t* st);
bool peer_stats(atom_peer* p, atom_stats_t* s);
bool peer_gemm_log(atom_peer* p, std::string* out);
bool peer_kernel_log(atom_peer* p, std::string* out);
void peer_reset_stats(atom_peer* p, int timing);
void peer_free(atom_peer* p);
bool peer_stream_sync(atom_peer* p);
bool profile_from_trace(const char* trace, const atom_model_cfg& cfg, const atom_plan_t& plan, atom_profile_t* out,
                        int64_t* table, int64_t cap);
}  // namespace atom

using namespace atom;

static atom_status fail(atom_peer* p, atom_status code) {
  if (p && (code == ATOM_E_CUDA || code == ATOM_E_NCCL)) p->poisoned = true;
  return code;
}
static atom_status cuda_or_nccl() {
  return strncmp(last_error(), "nccl", 4) == 0 ? ATOM_E_NCCL : ATOM_E_CUDA;
}

extern "C" {

atom_status atom_nccl_unique_id(void* out128) {
  if (!out128) {
    set_error("atom_nccl_unique_id: NULL");
    return ATOM_E_INVALID;
  }
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    set_error("ncclGetUniqueId failed: %s", ncclGetErrorString(r));
    return ATOM_E_NCCL;
  }
  static_assert(sizeof(id) == 128, "nccl id size");
  memcpy(out128, &id, 128);
  return ATOM_OK;
}

atom_status atom_peer_create(const atom_model_cfg* cfg, const atom_plan_t* plan, int32_t device, void* device_arena,
                             int64_t arena_bytes, const float* init_params, uint64_t seed, const void* nccl_id,
                             int32_t nranks, int32_t rank, atom_peer** out) {
  if (!cfg || !plan || !device_arena || !out) {
    set_error("atom_peer_create: NULL argument");
    return ATOM_E_INVALID;
  }
  *out = nullptr;
  if (!check_plan(*cfg, *plan)) return ATOM_E_INVALID;
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !nccl_id)) {
    set_error("atom_peer_create: invalid nranks/rank/nccl_id");
    return ATOM_E_INVALID;
  }
  if (arena_bytes < plan->device_bytes) {
    set_error("device arena of %lld bytes < plan.device_bytes %lld", (long long)arena_bytes,
              (long long)plan->device_bytes);
    return ATOM_E_CAPACITY;
  }
  if ((uintptr_t)device_arena & 255) {
    set_error("device arena must be 256-byte aligned");
    return ATOM_E_INVALID;
  }
  atom_peer* p = new atom_peer();
  p->cfg = *cfg;
  p->cfg.cost_table = nullptr;
  p->cfg.forced_ends = nullptr;
  p->cfg.n_forced = 0;
  p->plan = *plan;
  make_dims(p->cfg, &p->dm);
  const ModelDims& dm = p->dm;
  if (dm.d / dm.h > 128 || dm.d > 6144 || (dm.dtype == ATOM_BF16 && dm.d % 8)) {
    set_error("unsupported shape: head size <= 128, d_model <= 6144 (and a multiple of 8 for bf16) required");
    delete p;
    return ATOM_E_INVALID;
  }
  if (cfg->dropout_p != 0.f) {
    // DESIGN.md R38: masks are drawn per 8-element Philox group of each site tensor (T % 8 keeps the
    // attention rows whole groups), the group index is one 32-bit counter word, and the bf16
    // attention kernels that apply the attention-site mask are the tcgen05 ones (d_h 64/80/128)
    const int dh = dm.d / dm.h;
    const double n_attn = (double)dm.b * dm.h * dm.T * dm.T;
    if (!(cfg->dropout_p > 0.f && cfg->dropout_p < 1.f) || dm.T % 8 || n_attn > 34359738368.0 ||
        (dm.dtype == ATOM_BF16 && !attn_tc_supported(dh, dm.d))) {
      set_error("invalid config: dropout needs 0 <= p < 1, T %% 8 == 0, b h T^2 <= 2^35 and (bf16) a tcgen05 "
                "attention head size (64, 80, 128)");
      delete p;
      return ATOM_E_INVALID;
    }
  }
  p->device = device;
  p->arena = (uint8_t*)device_arena;
  p->arena_bytes = arena_bytes;
  p->S = plan->n_seg;
  p->C = plan->C;
  p->nranks = nranks;
  p->policy = plan->act_policy;
  p->n_recompute = plan->n_recompute;
  p->rank = rank;
  p->seg_of_node.assign(dm.n_nodes, 0);
  int lo = 0;
  for (int k = 1; k <= p->S; ++k) {
    const int hi = plan->seg_end[k - 1];
    p->seg_lo.push_back(lo);
    p->seg_hi.push_back(hi);
    int64_t P = 0;
    for (int i = lo; i <= hi; ++i) {
      P += dm.P[i];
      p->seg_of_node[i] = k;
    }
    p->seg_P.push_back(P);
    p->seg_off.push_back(dm.node_off[lo]);
    lo = hi + 1;
  }
  // whole blocks of the last segment (operator-granular: both halves in it); the first of them
  // reads its input from the C-deep boundary buffer
  for (int l = 0; l < dm.L; ++l)
    if (blk_node(dm, l, 0) >= p->seg_lo[p->S - 1]) {
      if (p->l0_last < 0) p->l0_last = l;
      p->nb_last++;
    }
  if (!peer_create(p, init_params, seed, nccl_id)) {
    atom_status code = strncmp(last_error(), "pinned", 6) == 0 ? ATOM_E_OOM : cuda_or_nccl();
    std::string msg = last_error();
    peer_free(p);
    delete p;
    set_error("%s", msg.c_str());
    return code;
  }
  *out = p;
  return ATOM_OK;
}

static atom_status do_step(atom_peer* p, const int32_t* tokens, bool dev, float* loss) {
  if (!p || !tokens || !loss) {
    set_error("atom_step: NULL argument");
    return ATOM_E_INVALID;
  }
  if (p->poisoned) {
    set_error("peer poisoned by an earlier CUDA/NCCL failure");
    return ATOM_E_STATE;
  }
  if (!peer_step(p, tokens, dev, loss)) return fail(p, cuda_or_nccl());
  return ATOM_OK;
}

atom_status atom_step(atom_peer* p, const int32_t* tokens, float* loss_out) { return do_step(p, tokens, false, loss_out); }
atom_status atom_step_device(atom_peer* p, const int32_t* tokens_dev, float* loss_out) {
  return do_step(p, tokens_dev, true, loss_out);
}

atom_status atom_sync(atom_peer* const* peers, int32_t n_local, int32_t flush) {
  if (!peers || n_local < 1) {
    set_error("atom_sync: no peers");
    return ATOM_E_INVALID;
  }
  for (int i = 0; i < n_local; ++i) {
    if (!peers[i]) { set_error("atom_sync: NULL peer"); return ATOM_E_INVALID; }
    if (peers[i]->poisoned) { set_error("peer poisoned"); return ATOM_E_STATE; }
  }
  if (!flush) {
    for (int i = 0; i < n_local; ++i) peers[i]->sync_next = true;
    return ATOM_OK;
  }
  for (int i = 1; i < n_local; ++i)
    if (peers[i]->S != peers[0]->S || peers[i]->seg_P != peers[0]->seg_P || (peers[0]->nranks > 1 && peers[i]->comm == peers[0]->comm)) {
      set_error("atom_sync: local peers need the same plan and their own communicator ranks");
      return ATOM_E_INVALID;
    }
  if (!peers_flush_average(peers, n_local)) {
    const atom_status st = cuda_or_nccl();
    for (int i = 0; i < n_local; ++i) fail(peers[i], st);
    return st;
  }
  return ATOM_OK;
}

atom_status atom_comm_reset(atom_peer* p, const void* nccl_id, int32_t nranks, int32_t rank) {
  if (!p || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !nccl_id)) {
    set_error("atom_comm_reset: invalid arguments");
    return ATOM_E_INVALID;
  }
  if (p->poisoned) { set_error("peer poisoned"); return ATOM_E_STATE; }
  if (!peer_comm_reset(p, nccl_id, nranks, rank)) return fail(p, cuda_or_nccl());
  return ATOM_OK;
}

atom_status atom_comm_shrink(atom_peer* p, const int32_t* exclude, int32_t n_exclude, int32_t abort_ops) {
  if (!p || n_exclude < 0 || (n_exclude > 0 && !exclude)) {
    set_error("atom_comm_shrink: invalid arguments");
    return ATOM_E_INVALID;
  }
  if (p->poisoned) { set_error("peer poisoned"); return ATOM_E_STATE; }
  for (int i = 0; i < n_exclude; ++i)
    if (exclude[i] < 0 || exclude[i] >= p->nranks || exclude[i] == p->rank) {
      set_error("atom_comm_shrink: rank %d cannot be excluded (own rank %d of %d)", exclude[i], p->rank, p->nranks);
      return ATOM_E_INVALID;
    }
  if (!peer_comm_shrink(p, exclude, n_exclude, abort_ops != 0)) return fail(p, cuda_or_nccl());
  return ATOM_OK;
}

atom_status atom_broadcast_state(atom_peer* p, int32_t root, int32_t adopt) {
  if (!p || root < 0 || root >= p->nranks) {
    set_error("atom_broadcast_state: invalid root");
    return ATOM_E_INVALID;
  }
  if (p->poisoned) { set_error("peer poisoned"); return ATOM_E_STATE; }
  if (!peer_broadcast_state(p, root, adopt != 0)) return fail(p, cuda_or_nccl());
  return ATOM_OK;
}

atom_status atom_peer_info(atom_peer* p, int32_t* rank, int32_t* nranks, int64_t* step) {
  if (!p) { set_error("atom_peer_info: NULL peer"); return ATOM_E_INVALID; }
  if (rank) *rank = p->rank;
  if (nranks) *nranks = p->nranks;
  if (step) *step = p->t;
  return ATOM_OK;
}

atom_status atom_get_params(atom_peer* p, float* master, float* m, float* v) {
  if (!p) { set_error("atom_get_params: NULL peer"); return ATOM_E_INVALID; }
  if (p->poisoned) { set_error("peer poisoned"); return ATOM_E_STATE; }
  if (!peer_get_params(p, master, m, v)) return fail(p, ATOM_E_CUDA);
  return ATOM_OK;
}

atom_status atom_get_trace(atom_peer* p, char* buf, int64_t cap, int64_t* len) {
  if (!p) { set_error("atom_get_trace: NULL peer"); return ATOM_E_INVALID; }
  std::string s;
  if (!peer_trace(p, &s, nullptr)) return fail(p, ATOM_E_CUDA);
  if (len) *len = (int64_t)s.size();
  if (!buf || cap < (int64_t)s.size() + 1) {
    set_error("buffer too small: need %lld bytes", (long long)s.size() + 1);
    return ATOM_E_INVALID;
  }
  memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  return ATOM_OK;
}

atom_status atom_get_gemm_log(atom_peer* p, char* buf, int64_t cap, int64_t* len) {
  if (!p) { set_error("atom_get_gemm_log: NULL peer"); return ATOM_E_INVALID; }
  std::string s;
  if (!peer_gemm_log(p, &s)) return fail(p, ATOM_E_CUDA);
  if (len) *len = (int64_t)s.size();
  if (!buf || cap < (int64_t)s.size() + 1) {
    set_error("buffer too small: need %lld bytes", (long long)s.size() + 1);
    return ATOM_E_INVALID;
  }
  memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  return ATOM_OK;
}

atom_status atom_get_kernel_log(atom_peer* p, char* buf, int64_t cap, int64_t* len) {
  if (!p) { set_error("atom_get_kernel_log: NULL peer"); return ATOM_E_INVALID; }
  std::string s;
  if (!peer_kernel_log(p, &s)) return fail(p, ATOM_E_CUDA);
  if (len) *len = (int64_t)s.size();
  if (!buf || cap < (int64_t)s.size() + 1) {
    set_error("buffer too small: need %lld bytes", (long long)s.size() + 1);
    return ATOM_E_INVALID;
  }
  memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  return ATOM_OK;
}

atom_status atom_profile(atom_peer* p, int64_t* cost_table, int64_t cap, atom_profile_t* out) {
  if (!p || !out) { set_error("atom_profile: NULL"); return ATOM_E_INVALID; }
  std::string tr;
  if (!peer_trace(p, &tr, nullptr)) return fail(p, ATOM_E_CUDA);
  if (tr.empty()) { set_error("atom_profile: the peer has not run a step"); return ATOM_E_STATE; }
  return profile_from_trace(tr.c_str(), p->cfg, p->plan, out, cost_table, cap) ? ATOM_OK : ATOM_E_INVALID;
}

atom_status atom_get_stats(atom_peer* p, atom_stats_t* out) {
  if (!p || !out) { set_error("atom_get_stats: NULL"); return ATOM_E_INVALID; }
  if (!peer_stats(p, out)) return fail(p, ATOM_E_CUDA);
  return ATOM_OK;
}

atom_status atom_reset_stats(atom_peer* p, int32_t timing) {
  if (!p) { set_error("atom_reset_stats: NULL"); return ATOM_E_INVALID; }
  if (!peer_stream_sync(p)) return fail(p, ATOM_E_CUDA);
  peer_reset_stats(p, timing);
  return ATOM_OK;
}

atom_status atom_peer_destroy(atom_peer* p) {
  if (!p) return ATOM_OK;
  peer_free(p);
  delete p;
  return ATOM_OK;
}

}  // extern "C"
