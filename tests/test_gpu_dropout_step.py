"""Dropout inside the training step (minGPT's embd / attn / resid sites, the
paper's profiled dropout layer; R38) against the fp64 oracle.

The oracle runs each micro-batch with its own Philox stream (micro_step = step * C + mb, the law
of oracle/philox.py) and averages the micro-batch losses and gradients -- the step loss is the
mean over all C b T tokens.  Checked through atom_step:
* fp32 path (SIMT kernels): loss, params, m and sqrt(v) per tensor within 1e-4 over 2 steps;
* bf16 path (tcgen05 attention with the mask regenerated in the forward, dQ and dK/dV kernels):
  loss and the step-1 gradient within the bf16 bounds of tests/grad_check.py;
* swapped == resident, bit-identical, with p > 0 (stash, re-forward and hybrid plans);
* a step with p > 0 differs from the p = 0 step (the masks are really applied).
"""
import numpy as np
import pytest

import synth
from grad_check import check_bf16_gradient
from oracle import adamw as oadamw
from oracle import gpt as ogpt

pytestmark = pytest.mark.gpu

atom = pytest.importorskip("paper_2403_10504_b200.atom")

TINY = synth.CONFIGS["tiny"]
MINI = synth.GPTConfig("mini", n_layer=3, d_model=128, n_head=2, seq_len=128, vocab=1000, micro_batch=2)
HYPER = oadamw.AdamWHyper(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, warmup_steps=0)
P_DROP, SEED = 0.1, 0x1234_5678_9ABC


def make_peer(g, dtype, C, ends=None, init=None, policy=0, n_recompute=0, p=P_DROP):
    cfg = atom.make_cfg(g, dtype=dtype, C_=C, overlap_check=0, forced_ends=ends, lr=HYPER.lr, warmup_steps=0,
                        act_policy=policy, n_recompute=n_recompute, dropout_p=p, dropout_seed=SEED)
    plan = atom.atom_plan(cfg, 10 ** 11, 10 ** 10)
    return atom.Peer(cfg, plan, init_params=init)


def oracle_step(g, p64, toks, C, step, p=P_DROP):
    """(loss, grad) of one step: per micro-batch Philox streams, mean over the micro-batches."""
    b = g.micro_batch
    loss, grad = 0.0, 0.0
    for mb in range(C):
        drop = ogpt.Dropout(p, SEED, micro_step=step * C + mb)
        lo, gr = ogpt.loss_and_grad(g, p64, toks[mb * b:(mb + 1) * b], drop=drop)
        loss, grad = loss + lo / C, grad + gr / C
    return loss, grad


def per_tensor_rel(a, b, g):
    out, off = {}, 0
    for node, name, shp in ogpt.shapes(g):
        n = int(np.prod(shp))
        x, y = a[off:off + n].astype(np.float64), b[off:off + n].astype(np.float64)
        out[(node, name)] = np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-30)
        off += n
    return out


@pytest.mark.parametrize("g,ends,pol,nrc", [(TINY, [2, 5], 0, 0), (TINY, [1, 3, 5], 2, 0), (MINI, [1, 2, 4], 0, 0),
                                             (MINI, [0, 2, 4], 3, 1)],
                         ids=["tiny-2seg", "tiny-3seg-recompute", "mini-3seg", "mini-3seg-hybrid"])
def test_fp32_dropout_step_matches_oracle(g, ends, pol, nrc):
    C = 2
    init = synth.init_params(g, seed=1234, perturb=True)
    peer = make_peer(g, atom.FP32, C, ends, init, policy=pol, n_recompute=nrc)
    p, m, v = init.astype(np.float64), np.zeros(init.size), np.zeros(init.size)
    for s in range(2):
        toks = synth.tokens(g, C * g.micro_batch, synth.step_seed(0, s))
        loss = peer.step(toks)
        rl, grad = oracle_step(g, p, toks, C, s)
        p, m, v = oadamw.adamw_step(HYPER, s + 1, p, grad, m, v)
        assert abs(loss - rl) <= 1e-4 * abs(rl), (s, loss, rl)
        got = peer.params()
        for key, gv, want in (("master", got["master"], p), ("m", got["m"], m),
                              ("sqrt(v)", np.sqrt(got["v"].astype(np.float64)), np.sqrt(v))):
            worst = max(per_tensor_rel(gv, want, g).items(), key=lambda kv: kv[1])
            assert worst[1] <= 1e-4, (s, key, worst)
    peer.destroy()


def test_bf16_dropout_step_gradient_within_bounds():
    g, C = MINI, 2
    init = synth.init_params(g, seed=1234, perturb=True)
    toks = synth.tokens(g, C * g.micro_batch, synth.step_seed(0, 0))
    peer = make_peer(g, atom.BF16, C, [1, 2, 4], init)
    loss = peer.step(toks)
    got = peer.params()
    peer.destroy()
    rl, grad = oracle_step(g, init.astype(np.float64), toks, C, 0)
    assert abs(loss - rl) <= 2e-2 * abs(rl), (loss, rl)
    check_bf16_gradient(got["m"] / (1.0 - HYPER.beta1), grad, g)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_dropout_swapped_equals_resident_bit_exact(dtype):
    g = MINI
    dt = atom.FP32 if dtype == "fp32" else atom.BF16
    C = 3
    init = synth.init_params(g, seed=7, perturb=True)
    toks = [synth.tokens(g, C * g.micro_batch, synth.step_seed(0, s)) for s in range(3)]
    res = make_peer(g, dt, C, None, init)
    base = [res.step(t) for t in toks]
    want = res.params()
    res.destroy()
    for ends, pol, nrc in (([1, 2, 4], atom.ACT_STASH, 0), ([0, 3, 4], atom.ACT_RECOMPUTE, 0),
                           ([2, 4], atom.ACT_HYBRID, 1)):
        pr = make_peer(g, dt, C, ends, init, policy=pol, n_recompute=nrc)
        assert [pr.step(t) for t in toks] == base, (ends, pol)
        got = pr.params()
        for k in ("master", "m", "v"):
            assert np.array_equal(got[k], want[k]), (ends, pol, k)
        pr.destroy()


def test_dropout_changes_the_step():
    g, C = MINI, 2
    init = synth.init_params(g, seed=3)
    toks = synth.tokens(g, C * g.micro_batch, synth.step_seed(0, 0))
    a = make_peer(g, atom.BF16, C, [1, 2, 4], init, p=0.0)
    b = make_peer(g, atom.BF16, C, [1, 2, 4], init, p=P_DROP)
    la, lb = a.step(toks), b.step(toks)
    ga, gb = a.params()["m"], b.params()["m"]
    a.destroy()
    b.destroy()
    assert la != lb and not np.array_equal(ga, gb)
