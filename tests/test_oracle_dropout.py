"""Pins for oracle/philox.py and the oracle's dropout sites.

- the generator: Philox4x32-10 known-answer vectors published with the algorithm (Random123
  kat_vectors: counter / key all zero, all ones, and the pi digits);
- the mask: flat index -> (counter, word, half) mapping, the keep rate within a binomial bound, the
  exact 1/(1-p) scale, independence of sites, layers and micro-steps;
- the model: p = 0 reduces bit for bit to the dropout-free oracle; finite differences with a
  fixed mask; torch fp64 autograd of an independently written module fed the same masks.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synth
from oracle import gpt, philox

MICRO = synth.GPTConfig("micro", n_layer=2, d_model=16, n_head=2, seq_len=8, vocab=32, micro_batch=2)

KAT = [  # (counter, key) -> output, Philox4x32-10 (Salmon et al. SC'11, Random123 kat_vectors)
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_known_answers(ctr, key, out):
    assert tuple(int(x) for x in philox.philox4x32_10(ctr, key)) == out


def test_flat_index_mapping():
    seed = (0x1234 << 32) | 0xABCD
    w = philox.uniform_halves(37, philox.SITE_ATTN, 5, 9, seed)
    for i in (0, 1, 3, 4, 7, 8, 17, 36):
        ref = int(philox.philox4x32_10((i // 8, philox.SITE_ATTN, 5, 9), (0xABCD, 0x1234))[(i // 2) % 4])
        assert int(w[i]) == (ref >> 16 if i % 2 else ref & 0xFFFF)


@pytest.mark.parametrize("p", [0.1, 0.5])
def test_keep_rate_and_scale(p):
    n = 1 << 18
    m = philox.keep_scale((n,), p, philox.SITE_RESID_MLP, 3, 0, 42)
    kept = m != 0
    assert np.all(m[kept] == 1.0 / (1.0 - p))
    p_eff = math.floor(p * 2 ** 16) / 2 ** 16                # drop probability of the 16-bit threshold
    sd = math.sqrt(n * p_eff * (1 - p_eff))
    assert abs((~kept).sum() - n * p_eff) <= 6 * sd
    assert abs(m.mean() - (1 - p_eff) / (1 - p)) <= 6 * sd / n / (1 - p)   # E[m] = 1 + 1e-5 at p = 0.1


def test_streams_differ():
    base = philox.keep_scale((4096,), 0.5, 2, 1, 0, 7)
    for args in [(3, 1, 0, 7), (2, 0, 0, 7), (2, 1, 1, 7), (2, 1, 0, 8)]:
        other = philox.keep_scale((4096,), 0.5, *args)
        agree = (base == other).mean()
        assert 0.4 < agree < 0.6, (args, agree)               # independent masks agree ~half


def _setup(cfg, n_seq=3, seed=7):
    p = synth.init_params(cfg, seed=seed, perturb=True, dtype=np.float64) * 5.0
    return p, synth.tokens(cfg, n_seq, seed + 1)


def test_p_zero_is_the_dropout_free_model():
    p, toks = _setup(MICRO)
    l0, g0 = gpt.loss_and_grad(MICRO, p, toks)
    l1, g1 = gpt.loss_and_grad(MICRO, p, toks, drop=gpt.Dropout(0.0, 99, 3))
    assert l0 == l1 and np.array_equal(g0, g1)


def test_dropout_changes_the_loss():
    p, toks = _setup(MICRO)
    l0 = gpt.loss_only(MICRO, p, toks)
    l1 = gpt.loss_only(MICRO, p, toks, drop=gpt.Dropout(0.3, 5, 0))
    l2 = gpt.loss_only(MICRO, p, toks, drop=gpt.Dropout(0.3, 5, 1))
    assert l0 != l1 and l1 != l2


def test_finite_differences_with_a_fixed_mask():
    p, toks = _setup(MICRO)
    drop = gpt.Dropout(0.25, 2024, 1)
    _, g = gpt.loss_and_grad(MICRO, p, toks, drop=drop)
    rng = np.random.default_rng(3)
    h = 1e-6
    for _ in range(6):
        u = rng.standard_normal(p.size)
        u /= np.linalg.norm(u)
        fd = (gpt.loss_only(MICRO, p + h * u, toks, drop=drop)
              - gpt.loss_only(MICRO, p - h * u, toks, drop=drop)) / (2 * h)
        an = float(g @ u)
        assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)) + 1e-9, (fd, an)


def _torch_loss(cfg, flat, toks, drop):
    """Independently written minGPT with dropout as explicit multipliers (masks from philox)."""
    t = torch.tensor(flat, dtype=torch.float64)
    P, off = {}, 0
    leaves = []
    for node, name, shp, _ in synth.param_layout(cfg):
        n = int(np.prod(shp))
        leaf = t[off:off + n].reshape(shp).clone().requires_grad_(True)
        P[(node, name)] = leaf
        leaves.append(leaf)
        off += n
    toks = torch.tensor(toks, dtype=torch.long)
    x, y = toks[:, :-1], toks[:, 1:]
    B, T = x.shape
    d, h = cfg.d_model, cfg.n_head
    M = lambda shape, site, layer: torch.tensor(drop.scale(shape, site, layer))   # noqa: E731
    hcur = (F.embedding(x, P[(0, "wte")]) + P[(0, "wpe")][:T]) * M((B, T, d), 0, 0)
    causal = torch.ones(T, T, dtype=torch.bool).triu(1)
    for l in range(cfg.n_layer):
        n = l + 1
        a = F.layer_norm(hcur, (d,), P[(n, "ln1_g")], P[(n, "ln1_b")], eps=1e-5)
        q, k, v = F.linear(a, P[(n, "w_qkv")], P[(n, "b_qkv")]).split(d, dim=-1)
        q, k, v = (z.view(B, T, h, d // h).transpose(1, 2) for z in (q, k, v))
        s = (q @ k.transpose(-1, -2) / math.sqrt(d // h)).masked_fill(causal, float("-inf"))
        att = F.softmax(s, dim=-1) * M((B, h, T, T), 1, l)
        o = (att @ v).transpose(1, 2).reshape(B, T, d)
        hcur = hcur + F.linear(o, P[(n, "w_o")], P[(n, "b_o")]) * M((B, T, d), 2, l)
        a2 = F.layer_norm(hcur, (d,), P[(n, "ln2_g")], P[(n, "ln2_b")], eps=1e-5)
        g = F.gelu(F.linear(a2, P[(n, "w_fc")], P[(n, "b_fc")]), approximate="tanh")
        hcur = hcur + F.linear(g, P[(n, "w_pr")], P[(n, "b_pr")]) * M((B, T, d), 3, l)
    L1 = cfg.n_layer + 1
    z = F.layer_norm(hcur, (d,), P[(L1, "lnf_g")], P[(L1, "lnf_b")], eps=1e-5)
    loss = F.cross_entropy(F.linear(z, P[(L1, "w_lm")]).reshape(-1, cfg.vocab), y.reshape(-1))
    loss.backward()
    return loss.item(), torch.cat([q.grad.reshape(-1) for q in leaves]).numpy()


@pytest.mark.parametrize("p_drop", [0.1, 0.5])
def test_torch_autograd_crosscheck_with_dropout(p_drop):
    p, toks = _setup(MICRO, n_seq=4)
    drop = gpt.Dropout(p_drop, 77, 2)
    loss, g = gpt.loss_and_grad(MICRO, p, toks, drop=drop)
    tl, tg = _torch_loss(MICRO, p, toks, drop)
    assert abs(loss - tl) <= 1e-12 * abs(loss)
    off = 0
    for node, name, shp in gpt.shapes(MICRO):
        n = int(np.prod(shp))
        a, b = g[off:off + n], tg[off:off + n]
        assert np.linalg.norm(a - b) <= 1e-10 * max(np.linalg.norm(b), 1e-12), name
        off += n
