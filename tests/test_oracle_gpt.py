"""Pins for oracle/gpt.py (fp64 GPT forward + hand-written backward).

Each test pins the oracle to something other than itself:
finite differences, torch-CPU fp64 autograd of an independently written
module, closed forms and invariants.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from torch_gpt import TorchGPT

import synth
from oracle import gpt

MICRO = synth.GPTConfig("micro", n_layer=2, d_model=16, n_head=2, seq_len=8, vocab=32, micro_batch=2)


def _setup(cfg, n_seq=3, seed=7, perturb=True):
    p = synth.init_params(cfg, seed=seed, perturb=perturb, dtype=np.float64)
    # larger weights than the 0.02 init so every nonlinearity is exercised
    p = p * 5.0
    toks = synth.tokens(cfg, n_seq, seed + 1)
    return p, toks


def test_layout_matches_synth():
    for cfg in synth.CONFIGS.values():
        a = [(n, nm, s) for n, nm, s in gpt.shapes(cfg)]
        b = [(n, nm, s) for n, nm, s, _ in synth.param_layout(cfg)]
        assert a == b
    assert synth.n_params(synth.CONFIGS["tiny"]) == 234880      # SURVEY §8 shapes table


def test_finite_differences_directional():
    """Central differences along random directions (h = 1e-6) match g.u (rel <= 1e-6)."""
    p, toks = _setup(MICRO)
    loss, g = gpt.loss_and_grad(MICRO, p, toks)
    rng = np.random.default_rng(0)
    h = 1e-6
    for _ in range(6):
        u = rng.standard_normal(p.size)
        u /= np.linalg.norm(u)
        fd = (gpt.loss_only(MICRO, p + h * u, toks) - gpt.loss_only(MICRO, p - h * u, toks)) / (2 * h)
        an = float(g @ u)
        assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)) + 1e-9, (fd, an)


def test_finite_differences_coordinates():
    """Central differences on sampled coordinates of every tensor."""
    p, toks = _setup(MICRO)
    _, g = gpt.loss_and_grad(MICRO, p, toks)
    rng = np.random.default_rng(1)
    off = 0
    h = 1e-6
    for node, name, shp in gpt.shapes(MICRO):
        n = int(np.prod(shp))
        for idx in rng.choice(n, size=min(3, n), replace=False):
            e = np.zeros(p.size)
            e[off + idx] = h
            fd = (gpt.loss_only(MICRO, p + e, toks) - gpt.loss_only(MICRO, p - e, toks)) / (2 * h)
            an = g[off + idx]
            assert abs(fd - an) <= 1e-6 * abs(an) + 2e-9, (name, idx, fd, an)   # 2e-9 ~ loss*eps/h
        off += n


@pytest.mark.parametrize("cfg", [MICRO, synth.CONFIGS["tiny"]], ids=["micro", "tiny"])
def test_torch_autograd_crosscheck(cfg):
    p, toks = _setup(cfg, n_seq=2 * cfg.micro_batch)
    loss, g = gpt.loss_and_grad(cfg, p, toks)
    m = TorchGPT(cfg, p)
    tl = m(torch.tensor(toks, dtype=torch.long))
    tl.backward()
    tg = torch.cat([q.grad.reshape(-1) for q in m.params]).numpy()
    assert abs(loss - tl.item()) <= 1e-12 * abs(loss)
    rel = np.linalg.norm(g - tg) / np.linalg.norm(tg)
    assert rel <= 1e-10, rel
    # per-tensor too (a wrong term in a small tensor would hide in the global norm)
    off = 0
    for node, name, shp in gpt.shapes(cfg):
        n = int(np.prod(shp))
        a, b = g[off:off + n], tg[off:off + n]
        assert np.linalg.norm(a - b) <= 1e-10 * max(np.linalg.norm(b), 1e-12), name
        off += n


def test_initial_loss_is_ln_vocab():
    """At std-0.02 init the logits are near zero, so loss ~ ln V (5.545 for V = 256)."""
    cfg = synth.CONFIGS["tiny"]
    p = synth.init_params(cfg, seed=1234, dtype=np.float64)
    toks = synth.tokens(cfg, 4, 3)
    loss = gpt.loss_only(cfg, p, toks)
    assert abs(loss - math.log(cfg.vocab)) < 0.05


def test_causality():
    """Perturbing token t+1 leaves the logits at positions <= t unchanged."""
    p, toks = _setup(MICRO, n_seq=1)
    pp = gpt.unflatten(MICRO, p)
    _, lg0, _ = gpt.forward(MICRO, pp, toks, want_cache=False)
    t = 4
    toks2 = toks.copy()
    toks2[0, t + 1] = (toks2[0, t + 1] + 5) % MICRO.vocab
    _, lg1, _ = gpt.forward(MICRO, pp, toks2, want_cache=False)
    assert np.array_equal(lg0[0, :t + 1], lg1[0, :t + 1])
    assert not np.allclose(lg0[0, t + 1:], lg1[0, t + 1:])


def test_attention_single_key_returns_v():
    rng = np.random.default_rng(3)
    q, k, v = (rng.standard_normal((2, 3, 1, 5)) for _ in range(3))
    o, a = gpt.attention(q, k, v)
    assert np.allclose(o, v) and np.allclose(a, 1.0)


def test_attention_matches_torch_sdpa():
    rng = np.random.default_rng(4)
    q, k, v = (rng.standard_normal((2, 3, 7, 5)) for _ in range(3))
    o, _ = gpt.attention(q, k, v)
    to = F.scaled_dot_product_attention(*(torch.tensor(t_) for t_ in (q, k, v)), is_causal=True)
    assert np.allclose(o, to.numpy(), atol=1e-13)


def test_layernorm_and_gelu_against_library():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((4, 9)) * 3 + 1
    g, b = rng.standard_normal(9), rng.standard_normal(9)
    y, _ = gpt.layernorm(x, g, b)
    ty = F.layer_norm(torch.tensor(x), (9,), torch.tensor(g), torch.tensor(b), eps=1e-5)
    assert np.allclose(y, ty.numpy(), atol=1e-13)
    u = np.linspace(-6, 6, 101)
    assert np.allclose(gpt.gelu(u), F.gelu(torch.tensor(u), approximate="tanh").numpy(), atol=1e-14)
    tu = torch.tensor(u, requires_grad=True)
    F.gelu(tu, approximate="tanh").sum().backward()
    assert np.allclose(gpt.gelu_grad(u), tu.grad.numpy(), atol=1e-13)


def test_loss_is_mean_over_all_step_tokens():
    """Reading R31: the step loss over C micro-batches is the mean over all C*b*T tokens,
    i.e. the average of equal-size micro-batch means, and so is its gradient."""
    p, toks = _setup(MICRO, n_seq=4)
    l_all, g_all = gpt.loss_and_grad(MICRO, p, toks)
    l0, g0 = gpt.loss_and_grad(MICRO, p, toks[:2])
    l1, g1 = gpt.loss_and_grad(MICRO, p, toks[2:])
    assert abs(l_all - 0.5 * (l0 + l1)) < 1e-13
    assert np.allclose(g_all, 0.5 * (g0 + g1), atol=1e-15)


def test_key_bias_gradient_is_zero():
    """Adding a constant to every key shifts each softmax row uniformly: d loss / d b_k = 0."""
    p, toks = _setup(MICRO)
    _, g = gpt.loss_and_grad(MICRO, p, toks)
    gp = gpt.unflatten(MICRO, g)
    d = MICRO.d_model
    for blk in gp["B"]:
        assert np.abs(blk["b_qkv"][d:2 * d]).max() < 1e-14
        assert np.abs(blk["b_qkv"][:d]).max() > 1e-6 and np.abs(blk["b_qkv"][2 * d:]).max() > 1e-6


def test_fp32_oracle_is_the_same_arithmetic():
    """bench.py times the oracle in fp32: it must compute the same loss and
    gradient as the fp64 parity oracle up to fp32 rounding (and really run in fp32)."""
    import numpy as np

    import synth
    from oracle import adamw as oadamw
    from oracle import gpt as ogpt
    g = synth.CONFIGS["tiny"]
    p = synth.init_params(g, seed=3, perturb=True)
    toks = synth.tokens(g, 2, 1)
    l64, g64 = ogpt.loss_and_grad(g, p.astype(np.float64), toks)
    l32, g32 = ogpt.loss_and_grad(g, p, toks, dtype=np.float32)
    assert g32.dtype == np.float32
    assert abs(l32 - l64) <= 1e-6 * abs(l64)
    assert np.linalg.norm(g32 - g64) <= 1e-5 * np.linalg.norm(g64)
    h = oadamw.AdamWHyper(warmup_steps=0)
    z = np.zeros_like(p)
    p32 = oadamw.adamw_step(h, 1, p, g32, z, z, dtype=np.float32)[0]
    p64 = oadamw.adamw_step(h, 1, p.astype(np.float64), g64, z, z)[0]
    assert p32.dtype == np.float32 and np.abs(p32 - p64).max() <= 1e-6
