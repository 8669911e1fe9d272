"""libatom's C++ planner and schedule emitter against the oracle, bit-exact (no GPU needed).

The oracle (oracle/planner.py, oracle/schedule.py) is itself pinned to brute force and to
SPEC/PAPER examples in test_oracle_planner.py / test_oracle_schedule.py.
"""
import random

import pytest

import synth
from oracle import planner as pl
from oracle import schedule as sc
from paper_2403_10504_b200 import atom


def _both(c: pl.PlanCfg, budget, link):
    g = synth.GPTConfig("x", c.n_layer, c.d_model, c.n_head, c.seq_len, c.vocab, c.micro_batch)
    ac = atom.make_cfg(g, dtype=c.dtype, C_=c.C, max_C=c.max_C, overlap_check=c.overlap_check,
                       peak_flops=c.peak_flops, d2h_bw=c.d2h_bw, state_budget=c.state_budget,
                       cost_table=c.cost_table, forced_ends=c.forced_ends, act_policy=c.act_policy,
                       n_recompute=c.n_recompute, grad_rounds=c.grad_rounds, op_nodes=c.op_nodes)
    want = pl.plan(c, budget, link)
    try:
        got = atom.atom_plan(ac, budget, link)
    except atom.AtomError as e:
        assert want is None, (want, str(e))
        assert e.code == atom.ATOM_E_INFEASIBLE
        return None, None
    assert want is not None, got.as_dict()
    return want, got


def _same(want: pl.Plan, got: atom.Plan):
    assert got.ends() == want.seg_end and got.C == want.C and got.n_seg == want.n_seg
    for f in ("nslot", "act_policy", "n_recompute", "cut_bytes", "r1_bytes", "slot_bytes", "stash_bytes", "work_bytes", "device_bytes",
              "pred_h2d_B", "pred_d2h_B", "pred_flops", "pred_step_ns", "pred_hidden_ppm"):
        assert getattr(got, f) == getattr(want, f), f


def test_random_configs_bit_exact():
    rng = random.Random(11)
    found = 0
    for _ in range(400):
        L = rng.randint(1, 9)
        c = pl.PlanCfg(n_layer=L, d_model=64 * rng.randint(1, 4), n_head=rng.choice([1, 2, 4]),
                       seq_len=rng.choice([16, 32, 64]), vocab=rng.choice([64, 300, 1001]),
                       micro_batch=rng.randint(1, 3), dtype=rng.choice([pl.FP32, pl.BF16]),
                       max_C=rng.randint(1, 12), overlap_check=rng.choice([0, 1, 1, 1]))
        if rng.random() < 0.6:
            tf = [0] + [rng.randint(1, 10 ** 6) for _ in range(L + 1)]
            c.cost_table = sum(([t, 2 * t + rng.randint(0, 10 ** 5)] for t in tf), [])
        else:
            c.peak_flops = rng.choice([10 ** 9, 10 ** 10, 10 ** 12])
        if rng.random() < 0.4:
            c.state_budget = rng.randint(10 ** 4, 10 ** 8)
        if rng.random() < 0.1:
            c.C = rng.randint(1, 6)
        c.act_policy = rng.choice([pl.ACT_AUTO, pl.ACT_STASH, pl.ACT_RECOMPUTE, pl.ACT_HYBRID])
        c.n_recompute = rng.randint(0, L)
        c.grad_rounds = rng.choice([0, 0, 1, 3])
        link = rng.choice([10 ** 8, 10 ** 9, 10 ** 10])
        hi = pl.Evaluator(c, 10 ** 18, link).device_bytes(1, [L + 1])
        budget = rng.randint(hi // 4, int(hi * 1.5))
        want, got = _both(c, budget, link)
        if want is not None:
            _same(want, got)
            found += 1
    assert found > 150


def test_random_configs_operator_granular_bit_exact():
    """Operator-granular graphs (a node per block half, cuts may fall inside a block; reading R40)."""
    rng = random.Random(23)
    found = split = 0
    for _ in range(300):
        L = rng.randint(1, 7)
        c = pl.PlanCfg(n_layer=L, d_model=64 * rng.randint(1, 4), n_head=rng.choice([1, 2, 4]),
                       seq_len=rng.choice([16, 32, 64]), vocab=rng.choice([64, 300, 1001]),
                       micro_batch=rng.randint(1, 3), dtype=rng.choice([pl.FP32, pl.BF16]),
                       max_C=rng.randint(1, 12), overlap_check=rng.choice([0, 1, 1, 1]), op_nodes=1,
                       act_policy=rng.choice([pl.ACT_AUTO, pl.ACT_STASH]))
        n = 2 * L + 2
        if rng.random() < 0.6:
            tf = [0] + [rng.randint(1, 10 ** 6) for _ in range(n - 1)]
            c.cost_table = sum(([t, 2 * t + rng.randint(0, 10 ** 5)] for t in tf), [])
        else:
            c.peak_flops = rng.choice([10 ** 9, 10 ** 10, 10 ** 12])
        if rng.random() < 0.4:
            c.state_budget = rng.randint(10 ** 4, 10 ** 8)
        c.grad_rounds = rng.choice([0, 0, 1, 3])
        link = rng.choice([10 ** 8, 10 ** 9, 10 ** 10])
        hi = pl.Evaluator(c, 10 ** 18, link).device_bytes(1, [n - 1])
        budget = rng.randint(hi // 4, int(hi * 1.5))
        want, got = _both(c, budget, link)
        if want is not None:
            _same(want, got)
            found += 1
            split += any(e % 2 == 1 and 1 <= e < n - 1 for e in want.seg_end)   # ends after an attention half
    assert found > 100 and split > 10, (found, split)


def test_operator_granular_rejects_reforward():
    g = synth.CONFIGS["tiny"]
    for pol in (atom.ACT_RECOMPUTE, atom.ACT_HYBRID):
        with pytest.raises(atom.AtomError) as e:
            atom.atom_plan(atom.make_cfg(g, op_nodes=1, act_policy=pol, n_recompute=1), 10 ** 10, 10 ** 9)
        assert e.value.code == atom.ATOM_E_INVALID


@pytest.mark.parametrize("name,frac,link", [("xl", 2, 50 * 10 ** 9), ("xl", 3, 60 * 10 ** 9),
                                            ("2.7b", 0, 60 * 10 ** 9), ("2.7b", 0, 49 * 10 ** 9),
                                            ("13b", 0, 49 * 10 ** 9), ("small", 0, 50 * 10 ** 9)])
def test_real_configs_bit_exact(name, frac, link):
    g = synth.CONFIGS[name]
    sb = 16 * synth.n_params(g) // frac if frac else 24 * 2 ** 30
    c = pl.PlanCfg.from_gpt(g, max_C=16, state_budget=sb)
    want, got = _both(c, 178 * 10 ** 9, link)
    if want is not None:
        _same(want, got)


def test_forced_tiny_plan():
    g = synth.CONFIGS["tiny"]
    c = pl.PlanCfg.from_gpt(g, C=1, overlap_check=0, forced_ends=[2, 5], dtype=pl.FP32)
    want, got = _both(c, 10 ** 10, 10 ** 9)
    _same(want, got)


def test_invalid_config_rejected():
    g = synth.GPTConfig("bad", 2, 65, 4, 8, 16, 1)     # d % h != 0
    with pytest.raises(atom.AtomError) as e:
        atom.atom_plan(atom.make_cfg(g), 10 ** 9, 10 ** 9)
    assert e.value.code == atom.ATOM_E_INVALID
    g = synth.CONFIGS["tiny"]
    with pytest.raises(atom.AtomError) as e:
        atom.atom_plan(atom.make_cfg(g, forced_ends=[3, 2]), 10 ** 9, 10 ** 9)
    assert e.value.code == atom.ATOM_E_INVALID


def test_infeasible_names_constraint():
    g = synth.CONFIGS["tiny"]
    with pytest.raises(atom.AtomError) as e:
        atom.atom_plan(atom.make_cfg(g), 1000, 10 ** 9)
    assert e.value.code == atom.ATOM_E_INFEASIBLE and "resident plan needs" in str(e.value)


@pytest.mark.parametrize("sync", [False, True])
def test_schedule_text_bit_exact(sync):
    for S in range(1, 12):
        for C in range(1, 5):
            p = atom.Plan()
            p.n_seg, p.C = S, C
            assert atom.atom_plan_schedule(p, sync) == sc.to_text(sc.emit(S, C, sync)), (S, C)
