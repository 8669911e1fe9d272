"""Pins for oracle/adamw.py and oracle/peers.py."""
import numpy as np
import torch

import synth
from oracle import adamw, gpt, peers


def test_adamw_step1_closed_form():
    """At t = 1 the bias corrections cancel: dp = -lr_1 g/(|g| + eps) - lr_1 wd p  (up to eps terms)."""
    h = adamw.AdamWHyper(lr=1e-3, warmup_steps=0, eps=1e-8, weight_decay=0.1)
    rng = np.random.default_rng(0)
    p, g = rng.standard_normal(1000), rng.standard_normal(1000)
    p1, m1, v1 = adamw.adamw_step(h, 1, p, g, np.zeros(1000), np.zeros(1000))
    expect = p * (1 - h.lr * h.weight_decay) - h.lr * g / (np.abs(g) + h.eps)
    assert np.allclose(p1, expect, rtol=0, atol=1e-15)
    assert np.allclose(m1, 0.1 * g) and np.allclose(v1, 0.001 * g * g)


def test_adamw_matches_torch_with_warmup():
    """torch.optim.AdamW (fp64) driven with lr_t = lr min(1, t/warmup)."""
    h = adamw.AdamWHyper(lr=1e-2, warmup_steps=3, weight_decay=0.05)
    rng = np.random.default_rng(1)
    p0 = rng.standard_normal(257)
    tp = torch.tensor(p0.copy(), requires_grad=True)
    opt = torch.optim.AdamW([tp], lr=h.lr, betas=(h.beta1, h.beta2), eps=h.eps, weight_decay=h.weight_decay)
    p, m, v = p0.copy(), np.zeros_like(p0), np.zeros_like(p0)
    for t in range(1, 8):
        g = rng.standard_normal(257)
        for grp in opt.param_groups:
            grp["lr"] = adamw.lr_at(h, t)
        tp.grad = torch.tensor(g)
        opt.step()
        p, m, v = adamw.adamw_step(h, t, p, g, m, v)
        assert np.allclose(p, tp.detach().numpy(), rtol=1e-14, atol=1e-15)


def test_lr_warmup_schedule():
    h = adamw.AdamWHyper(lr=1e-4, warmup_steps=3000)
    assert adamw.lr_at(h, 1) == 1e-4 / 3000
    assert adamw.lr_at(h, 3000) == 1e-4 and adamw.lr_at(h, 10 ** 6) == 1e-4


def test_average_identity_and_mean():
    rng = np.random.default_rng(2)
    a = rng.standard_normal(50)
    assert np.array_equal(peers.average([a]), a)                 # n = 1
    assert np.allclose(peers.average([a, a, a]), a)              # identical peers
    b, c = rng.standard_normal(50), rng.standard_normal(50)
    assert np.allclose(peers.average([a, b, c]), (a + b + c) / 3)


def test_two_peer_sync_equals_mean_of_independent_updates():
    """Peers train independently; at a sync step their masters become the mean."""
    cfg = synth.GPTConfig("micro", 1, 16, 2, 8, 32, 2)
    p0 = synth.init_params(cfg, seed=3, perturb=True, dtype=np.float64)
    h = adamw.AdamWHyper(lr=1e-2, warmup_steps=0)
    toks = [[synth.tokens(cfg, 2, synth.step_seed(r, s)) for r in range(2)] for s in range(2)]
    prs, losses = peers.train(cfg, p0, h, toks, sync_steps={2})
    # independent replay
    ind = []
    for r in range(2):
        pr = peers.Peer(cfg, p0, h)
        for s in range(2):
            pr.step(toks[s][r])
        ind.append(pr)
    mean = (ind[0].p + ind[1].p) / 2
    assert np.allclose(prs[0].p, mean, atol=1e-15) and np.allclose(prs[1].p, mean, atol=1e-15)
    assert np.array_equal(prs[0].m, ind[0].m) and np.array_equal(prs[1].v, ind[1].v)   # moments stay local
    assert np.allclose(losses[0][0], gpt.loss_only(cfg, p0, toks[0][0]))


def test_gradient_rounds_equal_one_step_on_the_joined_batch():
    """Host update placement (R37): R = 2 rounds on batches A and B, then AdamW on the mean
    gradient, equals one plain step on the batch A + B (the loss is a mean over equally many
    tokens, so its gradient is the mean of the two); R = 1 is the plain step."""
    cfg = synth.GPTConfig("micro", 1, 16, 2, 8, 32, 2)
    p0 = synth.init_params(cfg, seed=4, perturb=True, dtype=np.float64)
    h = adamw.AdamWHyper(lr=1e-2, warmup_steps=0)
    a, b = synth.tokens(cfg, 2, 11), synth.tokens(cfg, 2, 12)
    two = peers.Peer(cfg, p0, h, grad_rounds=2)
    two.step(a)
    assert np.array_equal(two.p, p0) and two.t == 0          # no update after the first round
    two.step(b)
    one = peers.Peer(cfg, p0, h)
    one.step(np.concatenate([a, b]))
    assert two.t == 1
    for x, y in ((two.p, one.p), (two.m, one.m), (two.v, one.v)):
        assert np.allclose(x, y, rtol=1e-12, atol=1e-15)
    r1, plain = peers.Peer(cfg, p0, h, grad_rounds=1), peers.Peer(cfg, p0, h)
    for s in range(2):
        r1.step(synth.tokens(cfg, 2, 20 + s))
        plain.step(synth.tokens(cfg, 2, 20 + s))
    assert np.array_equal(r1.p, plain.p) and np.array_equal(r1.v, plain.v)
