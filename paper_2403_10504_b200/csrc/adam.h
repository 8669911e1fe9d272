// AdamW constants shared by the GPU kernel (elementwise.cu) and the CPU AdamW (cpu_adam.cpp).
#pragma once

namespace atom {

// Constants of one update, computed once on the host (float arithmetic, no contraction) so the
// GPU kernel and the CPU AdamW (host update placement, R37) apply bit-identical updates:
//   p <- p * decay;  g' = g * gscale;  m <- m + (1 - b1)(g' - m);  v <- b2 v + (1 - b2) g'^2;
//   p <- p - step * m / (sqrt(v) / sbc2 + eps)      (step = lr_t / (1 - b1^t), sbc2 = sqrt(1 - b2^t))
struct AdamConsts {
  float decay, step, b1, b2, eps, sbc2, gscale;
};
AdamConsts adam_consts(float lr_t, float b1, float b2, float eps, float wd, long t, float gscale);
// the update on host arrays with `threads` workers (0 = all cores); cpu_adam.cpp
void cpu_adamw(float* p, const float* g, float* m, float* v, long n, const AdamConsts& k, int threads);

}  // namespace atom
