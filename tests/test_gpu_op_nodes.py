"""Operator-granular sub-models ("a node ... is a layer or an
operator"; R40) executed through atom_step: plans whose sub-models end inside a block
(between a block's attention half and its MLP half) against the fp64 oracle (fp32 path) and
bit-identical to the resident run (bf16 and fp32, with and without dropout).

Nodes of the half-block graph: 0 = E, 2l+1 = attention half of block l, 2l+2 = MLP half, 2L+1 = H.
"""
import numpy as np
import pytest

import synth
from oracle import adamw as oadamw
from oracle import peers as opeers

pytestmark = pytest.mark.gpu

atom = pytest.importorskip("paper_2403_10504_b200.atom")

TINY = synth.CONFIGS["tiny"]   # L = 4: nodes 0..9
MINI = synth.GPTConfig("mini", n_layer=3, d_model=128, n_head=2, seq_len=128, vocab=1000, micro_batch=2)  # 0..7
HYPER = oadamw.AdamWHyper(lr=1e-3, warmup_steps=0)


def make_peer(g, dtype, C, ends, init, op=1, p=0.0):
    cfg = atom.make_cfg(g, dtype=dtype, C_=C, overlap_check=0, forced_ends=ends, lr=HYPER.lr, warmup_steps=0,
                        op_nodes=op, dropout_p=p, dropout_seed=5)
    plan = atom.atom_plan(cfg, 10 ** 11, 10 ** 10)
    if ends is not None:
        assert plan.ends() == list(ends)
    return atom.Peer(cfg, plan, init_params=init)


def rel(a, b):
    return np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("ends", [[1, 4, 7, 9], [3, 5, 9], [0, 2, 3, 6, 8, 9], [7, 9]],
                         ids=["cuts-after-A0-M1-A3", "A1-A2", "mixed", "last-is-M3+H"])
def test_fp32_mid_block_cuts_match_oracle(ends):
    g, C = TINY, 2
    init = synth.init_params(g, seed=1234, perturb=True)
    peer = make_peer(g, atom.FP32, C, ends, init)
    ref = opeers.Peer(g, init.astype(np.float64), HYPER)
    for s in range(2):
        toks = synth.tokens(g, C * g.micro_batch, synth.step_seed(0, s))
        loss = peer.step(toks)
        rl, _ = ref.step(toks)
        assert abs(loss - rl) <= 1e-4 * abs(rl), (s, loss, rl)
        got = peer.params()
        assert rel(got["master"], ref.p) <= 1e-5 and rel(got["m"], ref.m) <= 1e-4, s
    peer.destroy()


@pytest.mark.parametrize("dtype,p", [("bf16", 0.0), ("bf16", 0.1), ("fp32", 0.1)])
def test_mid_block_cuts_equal_resident_bit_exact(dtype, p):
    g, C = MINI, 3
    dt = atom.FP32 if dtype == "fp32" else atom.BF16
    init = synth.init_params(g, seed=7, perturb=True)
    toks = [synth.tokens(g, C * g.micro_batch, synth.step_seed(0, s)) for s in range(3)]
    res = make_peer(g, dt, C, None, init, op=0, p=p)     # the block graph, resident
    assert res.plan.n_seg == 1
    base = [res.step(t) for t in toks]
    want = res.params()
    res.destroy()
    for ends in ([1, 3, 5, 7], [2, 5, 7], [0, 1, 4, 7], [5, 7], [6, 7]):
        pr = make_peer(g, dt, C, ends, init, op=1, p=p)
        assert [pr.step(t) for t in toks] == base, ends
        got = pr.params()
        for k in ("master", "m", "v"):
            assert np.array_equal(got[k], want[k]), (ends, k)
        pr.destroy()
