"""Philox4x32-10 counter-based generator and the dropout keep-mask (TEST INFRASTRUCTURE ONLY).

SURVEY §8 NEXT-4: dropout (minGPT's embd / attn / resid sites, the paper's profiled dropout
layer) drawn from a counter-based generator that the oracle and a GPU kernel
each implement on their own (task ③: "each side implements the same counter-based generator").

Philox4x32-10 (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3"), written
out as its definition:

  round(c, k):  (hi0, lo0) = mulhilo32(0xD2511F53, c0); (hi1, lo1) = mulhilo32(0xCD9E8D57, c2)
                c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
  10 rounds; the key is bumped k <- (k0 + 0x9E3779B9, k1 + 0xBB67AE85) (mod 2^32) between rounds.

Pinned by the published known-answer vectors (tests/test_oracle_dropout.py).

Dropout reading (R38): element i (row-major flat index of the site tensor of one
micro-batch) takes 16-bit half i % 2 (0 = low) of word (i // 2) % 4 of
philox(counter = (i // 8, site, layer, micro_step), key = (seed mod 2^32, seed >> 32)); it is
dropped iff that half < floor(p * 2^16), kept ones are scaled by 1 / (1 - p) (inverted dropout,
minGPT / torch.nn.Dropout).  One Philox call serves 8 elements (p resolution 2^-16).
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = 0xFFFFFFFF

# dropout sites (counter word 1)
SITE_EMBD, SITE_ATTN, SITE_RESID_ATTN, SITE_RESID_MLP = 0, 1, 2, 3


def philox4x32_10(counter, key):
    """counter: 4 uint arrays (broadcastable), key: 2 ints -> 4 uint32 arrays."""
    c = [np.asarray(x, dtype=np.uint64) & MASK32 for x in counter]
    k0, k1 = int(key[0]) & MASK32, int(key[1]) & MASK32
    for r in range(10):
        if r:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = np.uint64(M0) * c[0]
        p1 = np.uint64(M1) * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK32)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK32)
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return [x.astype(np.uint32) for x in c]


def uniform_halves(n, site, layer, micro_step, seed):
    """The n uint16 draws of one site tensor (flat index order)."""
    g = np.arange((n + 7) // 8, dtype=np.uint64)       # counter word 0 = i // 8
    z = np.zeros_like(g)
    words = philox4x32_10((g, z + site, z + layer, z + micro_step), (seed & MASK32, seed >> 32))
    w = np.stack(words, axis=-1).reshape(-1)          # word j of group g -> 4g + j
    halves = np.stack([w & 0xFFFF, w >> 16], axis=-1).reshape(-1)   # half h of word k -> 2k + h
    return halves[:n].astype(np.uint16)


def keep_scale(shape, p, site, layer, micro_step, seed):
    """fp64 multiplier of the site tensor: 0 where dropped, 1/(1-p) where kept."""
    n = int(np.prod(shape))
    thr = np.uint16(int(np.floor(p * 2.0 ** 16)))
    keep = uniform_halves(n, site, layer, micro_step, seed) >= thr
    return (keep.astype(np.float64) / (1.0 - p)).reshape(shape)
