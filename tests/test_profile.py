"""Measured-profile helpers (paper_2403_10504_b200/profile.py): trace interval union and the FLOPs a
planned step executes, checked against hand counts."""
import synth
from paper_2403_10504_b200 import atom
from paper_2403_10504_b200 import profile as aprof


def test_compute_busy_union_and_span():
    tr = "\n".join([
        "compute FWD 1 0 - 100.0 300.0",
        "compute FWD 1 1 - 250.0 400.0",     # overlaps the first: union 100..400
        "h2d LOAD_F 2 - 1 0.0 1000.0",       # other lanes are ignored
        "compute BWD 1 0 - 500.0 600.0",
    ])
    assert abs(aprof.compute_busy_ms(tr) - 0.4) < 1e-12       # (300 + 100) us
    assert abs(aprof.compute_span_ms(tr) - 0.5) < 1e-12       # 100 .. 600 us
    assert abs(aprof.lane_ms(tr, "h2d") - 1.0) < 1e-12


def test_executed_flops_counts_the_reforward():
    g = synth.CONFIGS["2.7b"]
    cfg_r = atom.make_cfg(g, dtype=atom.BF16, max_C=32, peak_flops=int(1.6e15), state_budget=20 * 2 ** 30,
                          act_policy=atom.ACT_RECOMPUTE)
    plan_r = atom.atom_plan(cfg_r, int(178e9), int(49.7e9))
    ends = plan_r.ends()
    nb_last = g.n_layer - ends[-2]
    tok = plan_r.C * g.micro_batch * g.seq_len
    d, T = g.d_model, g.seq_len
    # re-forward of every block outside the last segment: QKV + projection + fc GEMMs, attention fwd
    want = plan_r.pred_flops + (g.n_layer - nb_last) * tok * (2 * (3 + 1 + 4) * d * d + 2 * d * (T + 1))
    assert abs(aprof.executed_flops(cfg_r, plan_r) - want) <= 1e-9 * want
    # without a re-forward the executed FLOPs are the model FLOPs
    cfg_s = atom.make_cfg(g, dtype=atom.BF16, max_C=32, peak_flops=int(1.0e15), state_budget=20 * 2 ** 30,
                          act_policy=atom.ACT_STASH)
    plan_s = atom.atom_plan(cfg_s, int(178e9), int(49.7e9))
    assert aprof.executed_flops(cfg_s, plan_s) == float(plan_s.pred_flops)
