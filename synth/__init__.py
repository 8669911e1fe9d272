"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no model math, no planner, no
optimizer).  It only draws the inputs both sides consume:

* ``CONFIGS``     -- the BASELINE.json workload shapes (GPT-3 Table II, PAPER.md
                     P:203-225; layer counts from BASELINE.json).
* ``tokens``      -- int32 token ids, uniform over [0, V) from numpy PCG64
                     (SURVEY §8(d) "Concrete synthetic inputs"); shape [C*b, T+1],
                     inputs = [:, :T], targets = [:, 1:].
* ``structured_tokens`` -- a repeated random 64-gram (learnable stream for the
                     loss-decreases smoke test).
* ``param_layout`` / ``init_params`` -- the canonical flat parameter order
                     (SURVEY §8(b) "Parameter order") and a seeded init drawn
                     from PCG64 (normal(0, 0.02), residual projections
                     0.02/sqrt(2L), biases 0, LN gain 1 -- minGPT).
                     ``perturb=True`` additionally randomises biases and LN
                     parameters so that parity tests see every term.

Random numbers the method itself would draw are not needed (dropout p = 0,
SURVEY §8(c) row 22).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class GPTConfig:
    name: str
    n_layer: int      # L (blocks)
    d_model: int      # d
    n_head: int       # h
    seq_len: int      # T
    vocab: int        # V
    micro_batch: int  # b (sequences per micro-batch)

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_head


# BASELINE.json configs.  XL uses 16 heads x 128 (Table II prints 24 heads at
# d=2048, which gives a non-integer head size).
CONFIGS = {
    "tiny": GPTConfig("tiny", 4, 64, 4, 32, 256, 2),
    "small": GPTConfig("small", 12, 768, 12, 2048, 50257, 8),
    "xl": GPTConfig("xl", 24, 2048, 16, 2048, 50257, 8),
    "2.7b": GPTConfig("2.7b", 32, 2560, 32, 2048, 50257, 8),
    "13b": GPTConfig("13b", 40, 5120, 40, 2048, 50257, 4),
}


def tokens(cfg: GPTConfig, n_seq: int, seed: int) -> np.ndarray:
    """Uniform int32 tokens [n_seq, T+1] from PCG64(seed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, cfg.vocab, size=(n_seq, cfg.seq_len + 1), dtype=np.int64).astype(np.int32)


def step_seed(peer: int, step: int) -> int:
    """PCG64(seed = 1000*peer + step)."""
    return 1000 * peer + step


def structured_tokens(cfg: GPTConfig, n_seq: int, seed: int, ngram: int = 64, pattern_seed: int = 99) -> np.ndarray:
    """One random ``ngram``-long pattern (fixed by ``pattern_seed``) repeated along every
    sequence, each sequence at a random phase drawn from ``seed``."""
    pat = np.random.Generator(np.random.PCG64(pattern_seed)).integers(0, cfg.vocab, size=ngram, dtype=np.int64)
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.empty((n_seq, cfg.seq_len + 1), dtype=np.int32)
    for i in range(n_seq):
        ph = int(rng.integers(0, ngram))
        idx = (np.arange(cfg.seq_len + 1) + ph) % ngram
        out[i] = pat[idx]
    return out


def param_layout(cfg: GPTConfig):
    """Canonical parameter order: list of (node, name, shape, kind).

    node 0 = E (wte, wpe); nodes 1..L = blocks; node L+1 = H (ln_f, lm_head).
    kind in {"w", "wres", "emb", "bias", "gain", "shift"} selects the init law.
    """
    L, d, T, V = cfg.n_layer, cfg.d_model, cfg.seq_len, cfg.vocab
    out = [(0, "wte", (V, d), "emb"), (0, "wpe", (T, d), "emb")]
    for l in range(L):
        n = 1 + l
        out += [
            (n, "ln1_g", (d,), "gain"), (n, "ln1_b", (d,), "shift"),
            (n, "w_qkv", (3 * d, d), "w"), (n, "b_qkv", (3 * d,), "bias"),
            (n, "w_o", (d, d), "wres"), (n, "b_o", (d,), "bias"),
            (n, "ln2_g", (d,), "gain"), (n, "ln2_b", (d,), "shift"),
            (n, "w_fc", (4 * d, d), "w"), (n, "b_fc", (4 * d,), "bias"),
            (n, "w_pr", (d, 4 * d), "wres"), (n, "b_pr", (d,), "bias"),
        ]
    out += [(L + 1, "lnf_g", (d,), "gain"), (L + 1, "lnf_b", (d,), "shift"),
            (L + 1, "w_lm", (V, d), "w")]
    return out


def n_params(cfg: GPTConfig) -> int:
    return sum(int(np.prod(s)) for _, _, s, _ in param_layout(cfg))


def init_params(cfg: GPTConfig, seed: int = 1234, perturb: bool = False,
                dtype=np.float32) -> np.ndarray:
    """Flat canonical-order init vector drawn from PCG64(seed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    std_res = 0.02 / math.sqrt(2 * cfg.n_layer)
    parts = []
    for _, _, shape, kind in param_layout(cfg):
        n = int(np.prod(shape))
        if kind in ("w", "emb"):
            a = rng.standard_normal(n) * 0.02
        elif kind == "wres":
            a = rng.standard_normal(n) * std_res
        elif kind == "gain":
            a = np.ones(n) + (rng.standard_normal(n) * 0.1 if perturb else 0.0)
        else:  # bias / shift
            a = rng.standard_normal(n) * 0.02 if perturb else np.zeros(n)
        parts.append(a.astype(dtype))
    return np.concatenate(parts)
