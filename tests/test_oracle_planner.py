"""Pins for oracle/planner.py.

* SPEC worked examples.
* Table II activation payloads from the cut-bytes model.
* Byte counts printed in PAPER.md.
* Algorithm 1 (literal) = brute force on >= 200 random chains.
* The exact DP = brute force over all partitions x all C.
"""
import dataclasses
import os
import random

import pytest

import synth
from oracle import planner as pl

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- SPEC examples
def test_spec_segment_load_sum():
    """t_load = {10,20,30,40} us, segment (1,2) load = 50 us."""
    assert pl.seg_sum([10, 20, 30, 40], 1, 2) == 50
    assert pl.seg_sum([7], 0, 0) == 7


def test_spec_valid_constraints_example():
    """C=4, t_fwd=5 each, t_load=10 each: c=(0,1), d=(2,3) -> 4*10 >= 20 -> true."""
    g = pl.Chain(mem=[1, 1, 1, 1], t_fwd=[5, 5, 5, 5], t_load=[10, 10, 10, 10])
    assert pl.valid_constraints(g, 0, 1, 2, 3, cap=2, C=4)
    assert not pl.valid_constraints(g, 0, 1, 2, 3, cap=1, C=4)       # memory
    z = pl.Chain(mem=[1, 1], t_fwd=[0, 0], t_load=[0, 5])
    assert not pl.valid_constraints(z, 0, 0, 1, 1, cap=9, C=64)      # zero compute vs load


def test_spec_unconstrained_partition_count():
    """constraints disabled on n=4 -> 2^3 = 8 plans."""
    assert len(list(pl.all_partitions(4))) == 8
    g = pl.Chain(mem=[1] * 4, t_fwd=[10] * 4, t_load=[0] * 4)
    assert len(pl.brute_force_chain(g, cap=10 ** 9, C=1, min_segments=1)) == 8


def test_spec_select_best_and_tiebreak():
    """min cut; ties fewer segments, then lexicographic; permutation invariant."""
    cut = {(1, 3): 100, (0, 3): 50, (2, 3): 50, (0, 1, 3): 50}
    plans = list(cut)
    assert pl.select_best(plans, cut.get) == (0, 3)
    random.Random(0).shuffle(plans)
    assert pl.select_best(plans, cut.get) == (0, 3)


def test_spec_determine_C():
    """loads 0 -> 1; fwd 10 vs load 35 -> 4; zero fwd with load > 0 -> infeasible."""
    assert pl.determine_C([10, 10], [0, 0]) == 1
    assert pl.determine_C([10, 10], [0, 35]) == 4
    assert pl.determine_C([0, 10], [0, 5]) is None


# ------------------------------------------------------------ printed numbers
def _cfg(d, h, L=2, V=50257, T=2048, b=1, dtype=pl.FP32):
    return pl.PlanCfg(n_layer=L, d_model=d, n_head=h, seq_len=T, vocab=V, micro_batch=b, dtype=dtype)


def test_table2_activation_payload():
    """Table II: payload MiB = 1 * 2048 * d * 4 B / 2^20 at a block boundary (fp32, b=1)."""
    rows = [l.split() for l in open(os.path.join(GOLD, "table2_payload.txt")) if l.strip() and l[0] != "#"]
    assert len(rows) == 8
    for name, d, h, mib in rows:
        c = _cfg(int(d), int(h))
        ev = pl.Evaluator(c, 10 ** 15, 10 ** 10)
        # a two-segment plan cuts one block boundary
        p = ev.make_plan(1, [1, c.n_layer + 1])
        assert p.cut_bytes == int(mib) * 2 ** 20, name
    # bf16 activations halve it (the B200 path's payload)
    assert pl.Evaluator(_cfg(768, 12, dtype=pl.BF16), 10 ** 15, 10 ** 10).make_plan(1, [1, 3]).cut_bytes == 3 * 2 ** 20


def test_printed_byte_counts():
    gold = {l.split()[0]: float(l.split()[1]) for l in open(os.path.join(GOLD, "printed_bytes.txt"))
            if l.strip() and l[0] != "#"}
    c = _cfg(12288, 96, L=2)
    P = pl.node_params(c)
    d = 12288
    # 16 B/param x (wte + wpe + 2 blocks + ln_f) = 68 GB
    trimmed = 16 * (P[0] + 2 * P[1] + 2 * d)
    assert round(trimmed / 1e9) == gold["trimmed175b_GB"]
    # the 50K x 12288 fp32 embedding ~ 2.4 GB (2.47e9 B)
    assert abs(50257 * 12288 * 4 / 1e9 - gold["embedding175b_GB"]) < 0.1
    # the 16 B/param accounting: 175B params -> 2.8 TB; our segment-1 slot holds
    # grad + master + m + v = 16 B/param next to the compute-dtype copy
    assert 175e9 * 16 / 1e12 == gold["full175b_TB"]
    assert pl.seg_need(c, P[1]) == 16 * P[1] + 4 * P[1]   # fp32 path: + fp32 compute copy
    # a GPT-3 block has 12 d^2 + 13 d parameters (no padding for d % 64 == 0)
    for g in synth.CONFIGS.values():
        cc = pl.PlanCfg.from_gpt(g)
        P = pl.node_params(cc)
        dd = g.d_model
        assert P[1] == 12 * dd * dd + 13 * dd
        assert sum(P) == synth.n_params(g)


# --------------------------------------------------------- Algorithm 1
def _rand_chain(rng, n):
    return pl.Chain(mem=[rng.randint(1, 5) for _ in range(n)],
                    t_fwd=[rng.randint(0, 6) for _ in range(n)],
                    t_load=[rng.randint(0, 12) for _ in range(n)])


def test_alg1_equals_brute_force_random_chains():
    rng = random.Random(42)
    nonempty = 0
    for trial in range(220):
        n = rng.randint(2, 12)
        g = _rand_chain(rng, n)
        cap = rng.randint(3, 14)
        C = rng.randint(1, 4)
        a = pl.alg1_enumerate(g, cap, C)
        b = pl.brute_force_chain(g, cap, C)
        assert a == b, (trial, n)
        nonempty += bool(a)
    assert nonempty > 50


def test_alg1_uniform_six_node_example():
    """6-node uniform chain (t_fwd=10, t_load=10, m=1, capacity=3, C=2)."""
    g = pl.Chain(mem=[1] * 6, t_fwd=[10] * 6, t_load=[10] * 6)
    assert pl.alg1_enumerate(g, 3, 2) == pl.brute_force_chain(g, 3, 2)
    assert (2, 5) in pl.alg1_enumerate(g, 3, 2)


# -------------------------------------------------- DP optimum = brute force
def _rand_plan_cfg(rng):
    L = rng.randint(1, 7)
    h = rng.choice([1, 2, 4])
    d = 64 * rng.randint(1, 3)
    n = L + 2
    c = pl.PlanCfg(n_layer=L, d_model=d, n_head=h, seq_len=rng.choice([16, 32]), vocab=rng.choice([64, 300]),
                   micro_batch=rng.randint(1, 3), dtype=rng.choice([pl.FP32, pl.BF16]),
                   max_C=rng.randint(1, 6), overlap_check=rng.choice([0, 1, 1, 1]))
    if rng.random() < 0.4:
        c.state_budget = rng.randint(10 ** 4, 10 ** 7)
    c.act_policy = rng.choice([pl.ACT_AUTO, pl.ACT_STASH, pl.ACT_RECOMPUTE, pl.ACT_HYBRID])
    c.n_recompute = rng.randint(0, L)
    c.grad_rounds = rng.choice([0, 0, 2])
    if rng.random() < 0.7:
        tf = [0] + [rng.randint(1, 400) for _ in range(n - 1)]
        c.cost_table = sum(([t, 2 * t + rng.randint(0, 50)] for t in tf), [])
    else:
        c.peak_flops = rng.choice([10 ** 9, 10 ** 10, 10 ** 11])
    return c


def test_dp_equals_brute_force():
    rng = random.Random(7)
    found = deep = 0
    for trial in range(1100):
        c = _rand_plan_cfg(rng)
        link = rng.choice([10 ** 9, 10 ** 10, 3 * 10 ** 10])
        ev = pl.Evaluator(c, 0, link)
        lo = pl.work_bytes(c, 1)
        hi = pl.Evaluator(c, 10 ** 18, link).device_bytes(1, [c.n_layer + 1])
        budget = rng.randint(lo, int(hi * 1.3))
        a = pl.brute_force_plan(c, budget, link)
        b = pl.dp_plan(c, budget, link)
        if a is None:
            assert b is None, trial
            continue
        found += 1
        assert b is not None and (a.seg_end, a.C) == (b.seg_end, b.C), (trial, a, b)
        assert a == b
        deep += a.n_seg >= 3
    assert found > 150 and deep > 35, (found, deep)


def test_tiny_forced_two_layer_submodels():
    """BASELINE configs[0]: tiny with '2-layer sub-models' = [E,B0,B1 | B2,B3,H], C=1, overlap off."""
    g = synth.CONFIGS["tiny"]
    c = pl.PlanCfg.from_gpt(g, C=1, overlap_check=0, forced_ends=[2, 5])
    p = pl.plan(c, 10 ** 12, 25 * 10 ** 9)
    assert p.seg_end == [2, 5] and p.n_seg == 2 and p.C == 1
    # searched: the smallest budget for which the optimum is this same 2-segment plan
    c2 = pl.PlanCfg.from_gpt(g, C=1, overlap_check=0)
    full = pl.plan(c2, 10 ** 12, 25 * 10 ** 9)
    assert full.n_seg == 1
    q = pl.plan(c2, full.device_bytes - 1, 25 * 10 ** 9)
    assert q is not None and q.n_seg >= 2


def test_small_per_layer_swapping():
    """BASELINE configs[1]: GPT-3 Small with per-layer sub-models ([E,B0] | B1 | ... | B11 | H).
    The lm_head (38.6M params) must load under one block's forward, so C is large."""
    g = synth.CONFIGS["small"]
    ends = [1] + list(range(2, 13)) + [13]
    c = pl.PlanCfg.from_gpt(g, max_C=32, forced_ends=ends)
    p = pl.plan(c, 178 * 10 ** 9, 50 * 10 ** 9)
    assert p is not None and p.seg_end == ends and p.n_seg == 13
    ev = pl.Evaluator(c, 178 * 10 ** 9, 50 * 10 ** 9)
    assert ev.violation(p.C - 1, ends) is not None       # C is the smallest that overlaps
    assert p.pred_hidden_ppm > 900_000


@pytest.mark.parametrize("name", ["xl"])
def test_real_configs_plan_is_feasible_and_overlapped(name):
    """A model-state cap (R1 + slots, the paper's sub-model 'GPU capacity') below
    16 B/param forces swapping; the plan satisfies every constraint and C > 1."""
    g = synth.CONFIGS[name]
    N = synth.n_params(g)
    c = pl.PlanCfg.from_gpt(g, max_C=16, state_budget=16 * N // 2)
    link = 50 * 10 ** 9
    p = pl.plan(c, 178 * 10 ** 9, link)
    assert p is not None
    ev = pl.Evaluator(c, 178 * 10 ** 9, link)
    assert ev.violation(p.C, p.seg_end) is None
    assert p.C > 1 and p.n_seg >= 3
    assert p.r1_bytes + p.nslot * p.slot_bytes <= c.state_budget
    # the integer-time schedule hides every copy that can be hidden: the
    # compute lane never waits inside the step ("zero steady-state idle")
    assert p.pred_hidden_ppm > 900_000


def test_full_stash_2p7b_needs_more_link_than_pcie():
    """SURVEY §7 hard part 1: hiding 12 B/param each way in the backward phase needs
    ~3*P/W tokens per step; at 50 GB/s the full activation stash of 2.7B does not fit
    next to a 16 GiB model-state cap in 178 GB of HBM (recompute is required)."""
    g = synth.CONFIGS["2.7b"]
    c = pl.PlanCfg.from_gpt(g, max_C=16, state_budget=16 * 2 ** 30, act_policy=pl.ACT_STASH)
    assert pl.dp_plan(c, 178 * 10 ** 9, 50 * 10 ** 9) is None
    # ACT_AUTO falls back to re-forwarding blocks inside the backward (reading R28)
    c.act_policy = pl.ACT_AUTO
    c.act_policy = pl.ACT_RECOMPUTE
    p = pl.dp_plan(c, 178 * 10 ** 9, 50 * 10 ** 9)
    assert p is not None and p.act_policy == pl.ACT_RECOMPUTE and p.n_seg >= 3
    ev = pl.Evaluator(c, 178 * 10 ** 9, 50 * 10 ** 9, c.n_layer)
    assert ev.violation(p.C, p.seg_end) is None
    # the stash keeps block inputs only: far below the full stash at the same C
    assert p.stash_bytes < pl.stash_bytes(c, p.C, 0, p.n_seg, 0) / 4
    # ACT_AUTO re-forwards the fewest blocks that make a plan feasible (reading R35): some, not all
    c.act_policy = pl.ACT_AUTO
    q = pl.dp_plan(c, 178 * 10 ** 9, 50 * 10 ** 9)
    assert q is not None and q.act_policy == pl.ACT_HYBRID and 0 < q.n_recompute < c.n_layer
    assert pl.Evaluator(c, 178 * 10 ** 9, 50 * 10 ** 9, q.n_recompute - 1).violation(q.C, q.seg_end) is not None
    assert pl.dp_plan(dataclasses.replace(c, act_policy=pl.ACT_HYBRID, n_recompute=q.n_recompute - 1),
                      178 * 10 ** 9, 50 * 10 ** 9) is None


# ---------------------------------------------------------------------------------------------
# Operator-granular graph ("a node ... is a layer or an operator"; reading R40): every block
# is an attention-half node and an MLP-half node, so sub-models may end inside a block.
def test_operator_granular_dp_equals_brute_force():
    """The exact DP over half-block nodes equals brute force over all 2^(n-1) partitions x C
    (n = 2L + 2 <= 16 nodes)."""
    rng = random.Random(17)
    found = split = 0
    for trial in range(220):
        c = _rand_plan_cfg(rng)
        c.n_layer = min(c.n_layer, 6)
        c.op_nodes = 1
        c.act_policy = rng.choice([pl.ACT_AUTO, pl.ACT_STASH])
        n = 2 * c.n_layer + 2
        if c.cost_table is not None:
            tf = [0] + [rng.randint(1, 400) for _ in range(n - 1)]
            c.cost_table = sum(([t, 2 * t + rng.randint(0, 50)] for t in tf), [])
        link = rng.choice([10 ** 9, 10 ** 10, 3 * 10 ** 10])
        hi = pl.Evaluator(c, 10 ** 18, link).device_bytes(1, [n - 1])
        budget = rng.randint(pl.work_bytes(c, 1), int(hi * 1.3))
        a = pl.brute_force_plan(c, budget, link)
        b = pl.dp_plan(c, budget, link)
        if a is None:
            assert b is None, trial
            continue
        found += 1
        assert a == b, (trial, a, b)
        split += any(e % 2 == 1 and 1 <= e < n - 1 for e in a.seg_end)
    assert found > 40 and split > 8, (found, split)


def test_operator_granular_halves_partition_the_block():
    """Half nodes split each block's parameters and FLOPs exactly (the canonical tensor order cut
    after b_o); a plan that cuts only between blocks has the block graph's arena, bytes and FLOPs."""
    for g in (synth.CONFIGS["tiny"], synth.CONFIGS["2.7b"]):
        cb = pl.PlanCfg.from_gpt(g)
        co = pl.PlanCfg.from_gpt(g, op_nodes=1)
        pb, po = pl.node_params(cb), pl.node_params(co)
        assert len(po) == 2 * g.n_layer + 2 and pb[0] == po[0] and pb[-1] == po[-1]
        assert all(pb[1 + l] == po[1 + 2 * l] + po[2 + 2 * l] for l in range(g.n_layer))
        fb, fo = pl.node_flops_fwd(cb), pl.node_flops_fwd(co)
        assert all(fb[1 + l] == fo[1 + 2 * l] + fo[2 + 2 * l] for l in range(g.n_layer))
        d, M = g.d_model, g.micro_batch * g.seq_len
        assert fo[2] == 16 * d * d * M                              # fc + fc2
        L = g.n_layer
        for ends_b in ([L + 1], [0, L + 1], [1, L // 2, L + 1], [L, L + 1]):
            ends_o = [0 if e == 0 else (2 * e if e <= L else 2 * L + 1) for e in ends_b]
            ends_o = sorted(set(ends_o))
            evb, evo = pl.Evaluator(cb, 10 ** 18, 10 ** 10), pl.Evaluator(co, 10 ** 18, 10 ** 10)
            assert evb.device_bytes(2, ends_b) == evo.device_bytes(2, ends_o), (g.name, ends_b)
            a, b = evb.make_plan(2, ends_b), evo.make_plan(2, ends_o)
            for f in ("cut_bytes", "r1_bytes", "slot_bytes", "stash_bytes", "work_bytes", "pred_h2d_B",
                      "pred_d2h_B", "pred_flops"):
                assert getattr(a, f) == getattr(b, f), (g.name, ends_b, f)


def test_operator_granular_mid_block_cut_can_be_the_optimum():
    """Under a model-state cap the half-block graph finds plans the block graph cannot: a slot only
    has to hold the largest swapped sub-model, which a mid-block cut makes smaller (the
    objective P:399, S:174 then prefers the fewest sub-models)."""
    g = synth.CONFIGS["tiny"]
    n = 2 * g.n_layer + 2
    feasible_only_split = fewer_with_split = 0
    for k in range(60):
        cap = 2_000_000 + 50_000 * k
        po = pl.plan(pl.PlanCfg.from_gpt(g, op_nodes=1, C=1, overlap_check=0, state_budget=cap), 10 ** 12, 10 ** 10)
        pb = pl.plan(pl.PlanCfg.from_gpt(g, C=1, overlap_check=0, state_budget=cap), 10 ** 12, 10 ** 10)
        if po is None:
            assert pb is None, cap            # the half-block graph contains every block-graph plan
            continue
        assert pb is None or po.n_seg <= pb.n_seg, cap
        mid = any(e % 2 == 1 and 1 <= e < n - 1 for e in po.seg_end)
        feasible_only_split += mid and pb is None
        fewer_with_split += mid and pb is not None and po.n_seg < pb.n_seg
    assert feasible_only_split > 0 and fewer_with_split > 0, (feasible_only_split, fewer_with_split)
