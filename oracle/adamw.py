"""AdamW with linear warm-up (TEST INFRASTRUCTURE ONLY).

PAPER.md P:563: "We used the CPU AdamW optimizer (beta1 = 0.9, beta2 = 0.999)
... learning rate 1e-4 ... linear warmup of 3K steps".  The paper leaves eps,
weight decay and the post-warm-up schedule unspecified; reading R19
takes torch's AdamW defaults (eps = 1e-8, weight_decay = 0.01 on all
parameters) and a constant rate after warm-up.  Update at step t (1-based),
decoupled weight decay (Loshchilov & Hutter, cited at P:563):

  lr_t = lr * min(1, t / warmup)            (warmup = 0 -> lr_t = lr)
  p   <- p * (1 - lr_t * wd)
  m   <- b1 m + (1 - b1) g
  v   <- b2 v + (1 - b2) g^2
  p   <- p - lr_t * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass(frozen=True)
class AdamWHyper:
    lr: float = 1e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.01
    warmup_steps: int = 3000


def lr_at(h: AdamWHyper, t: int) -> float:
    if h.warmup_steps <= 0:
        return h.lr
    return h.lr * min(1.0, t / h.warmup_steps)


def adamw_step(h: AdamWHyper, t: int, p, g, m, v, dtype=np.float64):
    """One AdamW update at step t (1-based).  Returns new (p, m, v) (fp64; dtype=np.float32 only
    for timing the oracle as the CPU baseline)."""
    p = np.asarray(p, dtype=dtype)
    g = np.asarray(g, dtype=dtype)
    m = np.asarray(m, dtype=dtype)
    v = np.asarray(v, dtype=dtype)
    lr_t = lr_at(h, t)
    p = p * (1.0 - lr_t * h.weight_decay)
    m = h.beta1 * m + (1.0 - h.beta1) * g
    v = h.beta2 * v + (1.0 - h.beta2) * g * g
    mhat = m / (1.0 - h.beta1 ** t)
    vhat = v / (1.0 - h.beta2 ** t)
    p = p - lr_t * mhat / (np.sqrt(vhat) + h.eps)
    return p, m, v
