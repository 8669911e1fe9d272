// CPU AdamW for the host update placement ("We used the CPU AdamW optimizer";
// SURVEY NEXT-1; R37).  Sub-models 2..S keep their fp32 master, m, v and gradient sum in
// pinned host memory; every R-th gradient round this runs on the host over one sub-model's range,
// started from the copy stream in stream order (cudaLaunchHostFunc) right after the sub-model's
// gradient sum lands, so the next step's forward load of that sub-model sees the new master.
//
// The arithmetic is the GPU kernel's (elementwise.cu adamw_kernel), operation for operation: every
// product and quotient rounded on its own, the two fused multiply-adds explicit (std::fma), IEEE
// sqrt and division -- so a swapped run with the CPU update is bit-identical to a resident run
// whose update runs on the GPU (tests/test_gpu_host_update.py).
#pragma STDC FP_CONTRACT OFF
#pragma GCC optimize("fp-contract=off")

#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "adam.h"

namespace atom {

AdamConsts adam_consts(float lr_t, float b1, float b2, float eps, float wd, long t, float gscale) {
  const double bc1 = 1.0 - std::pow((double)b1, (double)t), bc2 = 1.0 - std::pow((double)b2, (double)t);
  AdamConsts k;
  k.decay = 1.f - lr_t * wd;
  k.step = lr_t / (float)bc1;
  k.b1 = b1;
  k.b2 = b2;
  k.eps = eps;
  k.sbc2 = (float)std::sqrt(bc2);
  k.gscale = gscale;
  return k;
}

static void adam_range(float* p, const float* g, float* m, float* v, long lo, long hi, const AdamConsts& c) {
  const float omb1 = 1.f - c.b1, omb2 = 1.f - c.b2;
  for (long i = lo; i < hi; ++i) {
    const float gk = g[i] * c.gscale;
    const float pd = p[i] * c.decay;
    const float mk = std::fma(omb1, gk - m[i], m[i]);
    const float t2 = (omb2 * gk) * gk;
    const float vk = std::fma(c.b2, v[i], t2);
    const float den = std::sqrt(vk) / c.sbc2 + c.eps;
    p[i] = pd - (c.step * mk) / den;
    m[i] = mk;
    v[i] = vk;
  }
}

void cpu_adamw(float* p, const float* g, float* m, float* v, long n, const AdamConsts& k, int threads) {
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  const long per = (n + nt - 1) / nt;
  if (nt == 1 || n < (1L << 16)) {
    adam_range(p, g, m, v, 0, n, k);
    return;
  }
  std::vector<std::thread> ws;
  ws.reserve(nt);
  for (int t = 0; t < nt; ++t) {
    const long lo = t * per, hi = std::min(n, lo + per);
    if (lo >= hi) break;
    ws.emplace_back(adam_range, p, g, m, v, lo, hi, std::cref(k));
  }
  for (auto& w : ws) w.join();
}

}  // namespace atom
