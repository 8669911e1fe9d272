// C-ABI: atom_plan, atom_plan_schedule, atom_last_error (include/atom.h).  Host only.
#include <string.h>

#include "../../include/atom.h"
#include "planner.h"

namespace atom {
void set_error(const char* fmt, ...);
const char* last_error();
}  // namespace atom

using namespace atom;

static atom_status copy_text(const std::string& s, char* buf, int64_t cap, int64_t* len) {
  if (len) *len = (int64_t)s.size();
  if (!buf || cap < (int64_t)s.size() + 1) {
    set_error("buffer too small: need %lld bytes", (long long)s.size() + 1);
    return ATOM_E_INVALID;
  }
  memcpy(buf, s.data(), s.size());
  buf[s.size()] = 0;
  return ATOM_OK;
}

extern "C" {

atom_status atom_plan(const atom_model_cfg* cfg, int64_t hbm_budget, int64_t link_bw, atom_plan_t* out) {
  if (!cfg || !out) {
    set_error("atom_plan: NULL argument");
    return ATOM_E_INVALID;
  }
  ModelDims dm;
  if (!make_dims(*cfg, &dm)) return ATOM_E_INVALID;
  if (link_bw <= 0 || hbm_budget <= 0 || (cfg->peak_flops <= 0 && !cfg->cost_table)) {
    set_error("atom_plan: hbm_budget, link_bw and peak_flops must be positive");
    return ATOM_E_INVALID;
  }
  if (!make_plan(*cfg, hbm_budget, link_bw, out)) {
    // distinguish invalid input from infeasibility by the message prefix
    return strncmp(last_error(), "invalid", 7) == 0 ? ATOM_E_INVALID : ATOM_E_INFEASIBLE;
  }
  return ATOM_OK;
}

atom_status atom_plan_schedule(const atom_plan_t* plan, int32_t sync, char* buf, int64_t cap, int64_t* len) {
  if (!plan || plan->n_seg < 1 || plan->n_seg > ATOM_MAX_SEG || plan->C < 1) {
    set_error("atom_plan_schedule: invalid plan");
    return ATOM_E_INVALID;
  }
  auto ops = emit_schedule(plan->n_seg, plan->C, sync != 0, nullptr);
  return copy_text(schedule_text(ops), buf, cap, len);
}

const char* atom_last_error(void) { return last_error(); }

}  // extern "C"
