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


class _Plan:
    def __init__(self, ends, policy, n_recompute=0):
        self._ends, self.act_policy, self.n_recompute = ends, policy, n_recompute

    def ends(self):
        return self._ends


def test_cost_table_from_trace_blocks_embed_head():
    # L = 4: nodes E, B0..B3, H; segments [E, B0] [B1, B2] [B3, H]; 2 micro-batches each
    tf, tb, emb_f, emb_b, hf, hb = 100.0, 250.0, 7.0, 11.0, 30.0, 60.0
    lines = []
    for mb in range(2):
        lines.append(f"compute FWD 1 {mb} - 0 {emb_f + tf}")
        lines.append(f"compute BWD 1 {mb} - 0 {emb_b + tb}")
        lines.append(f"compute FWD 2 {mb} - 0 {2 * tf}")
        lines.append(f"compute BWD 2 {mb} - 0 {2 * tb}")
        lines.append(f"compute FWD 3 {mb} - 0 {tf + hf + hb}")   # head fwd + bwd inside FWD(S)
        lines.append(f"compute BWD 3 {mb} - 0 {tb}")
    t = aprof.cost_table_from_trace("\n".join(lines), _Plan([1, 3, 5], atom.ACT_STASH), 4)
    us = [x / 1000.0 for x in t]
    assert us[2:10] == [tf, tb] * 4
    assert abs(us[0] - emb_f) < 1e-6 and abs(us[1] - emb_b) < 1e-6
    assert abs(us[10] - (hf + hb) / 3) < 1e-3 and abs(us[11] - 2 * (hf + hb) / 3) < 1e-3
    # under the re-forward policy the traced backward includes one forward per block: removed
    lines_rc = [l.replace(f"BWD 2 ", "BWD 2 ") for l in lines]
    lines_rc = [(f"compute BWD 2 {l.split()[3]} - 0 {2 * (tb + tf)}" if l.split()[1:3] == ["BWD", "2"] else l)
                for l in lines_rc]
    t_rc = aprof.cost_table_from_trace("\n".join(lines_rc), _Plan([1, 3, 5], atom.ACT_HYBRID, 3), 4)
    assert abs(t_rc[3] / 1000.0 - tb) < 1e-6
    # hybrid: only blocks 1..2 re-forwarded -> segment 2 holds one of them (B1), segment 1 one (B0)
    lines_h = [(f"compute BWD 2 {l.split()[3]} - 0 {2 * tb + tf}" if l.split()[1:3] == ["BWD", "2"] else
                (f"compute BWD 1 {l.split()[3]} - 0 {emb_b + tb + tf}" if l.split()[1:3] == ["BWD", "1"] else l))
               for l in lines]
    t_h = aprof.cost_table_from_trace("\n".join(lines_h), _Plan([1, 3, 5], atom.ACT_HYBRID, 2), 4)
    assert abs(t_h[3] / 1000.0 - tb) < 1e-6 and abs(t_h[1] / 1000.0 - emb_b) < 1e-6
