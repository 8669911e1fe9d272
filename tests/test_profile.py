"""Measured profile (csrc/profile.cpp through atom_profile_trace, pure host): the compute-lane busy
union, the executed FLOPs of a plan (with its re-forward) and the per-node cost table, checked
against hand counts on synthetic traces (P:329 per-layer profiling; R34)."""
import synth
from paper_2403_10504_b200 import atom


def _plan(ends, C=2, n_recompute=0, h2d=0, d2h=0, flops=0):
    p = atom.Plan()
    p.n_seg = len(ends)
    for i, e in enumerate(ends):
        p.seg_end[i] = e
    p.C, p.n_recompute, p.pred_h2d_B, p.pred_d2h_B, p.pred_flops = C, n_recompute, h2d, d2h, flops
    return p


def _cfg(L=4, d=64, T=32, b=2):
    g = synth.GPTConfig("t", n_layer=L, d_model=d, n_head=4, seq_len=T, vocab=256, micro_batch=b)
    return atom.make_cfg(g, dtype=atom.BF16)


def test_busy_union_copy_rates_and_flops():
    tr = "\n".join([
        "compute FWD 1 0 - 100.0 300.0",
        "compute FWD 1 1 - 250.0 400.0",     # overlaps the first: union 100..400
        "h2d LOAD_F 2 - 1 0.0 1000.0",       # 1 ms of h2d
        "d2h STORE 2 - 1 0.0 500.0",         # 0.5 ms of d2h
        "compute BWD 1 0 - 500.0 600.0",
    ])
    pr = atom.atom_profile_trace(tr, _cfg(), _plan([1, 5], h2d=10 ** 9, d2h=10 ** 9, flops=4 * 10 ** 12))
    assert abs(pr["compute_busy_ms"] - 0.4) < 1e-12          # (300 + 100) us
    assert abs(pr["flops"] - 4e12 / 0.4e-3) <= 1e-6 * 1e16
    assert abs(pr["h2d"] - 1e12) <= 1e3 and abs(pr["d2h"] - 2e12) <= 1e3
    assert pr["cost_table"] == []                            # no blocks-only sub-model


def test_executed_flops_counts_the_reforward():
    cfg = _cfg(L=4, d=64, T=32, b=2)
    C, nrc, base = 3, 2, 10 ** 9
    pr = atom.atom_profile_trace("compute FWD 1 0 - 0 1000\n", cfg, _plan([1, 5], C=C, n_recompute=nrc, flops=base))
    tok = C * 2 * 32
    want = base + nrc * tok * (2 * (3 + 1 + 4) * 64 * 64 + 2 * 64 * 33)   # QKV + proj + fc GEMMs, attention fwd
    assert abs(pr["executed_flops"] - want) <= 1e-9 * want


def test_cost_table_blocks_embed_head():
    # L = 4: nodes E, B0..B3, H; segments [E, B0] [B1, B2] [B3, H]; 2 micro-batches each
    tf, tb, emb_f, emb_b, hf, hb = 100.0, 250.0, 7.0, 11.0, 30.0, 60.0
    cfg = _cfg()

    def trace(b2=2 * tb, b1=emb_b + tb):
        lines = []
        for mb in range(2):
            lines += [f"compute FWD 1 {mb} - 0 {emb_f + tf}", f"compute BWD 1 {mb} - 0 {b1}",
                      f"compute FWD 2 {mb} - 0 {2 * tf}", f"compute BWD 2 {mb} - 0 {b2}",
                      f"compute FWD 3 {mb} - 0 {tf + hf + hb}",   # head fwd + bwd inside FWD(S)
                      f"compute BWD 3 {mb} - 0 {tb}"]
        return "\n".join(lines)

    us = [x / 1000.0 for x in atom.atom_profile_trace(trace(), cfg, _plan([1, 3, 5]))["cost_table"]]
    assert us[2:10] == [tf, tb] * 4
    assert abs(us[0] - emb_f) < 1e-6 and abs(us[1] - emb_b) < 1e-6
    assert abs(us[10] - (hf + hb) / 3) < 1e-3 and abs(us[11] - 2 * (hf + hb) / 3) < 1e-3
    # re-forward of blocks 1..3 (B0 in segment 1, B1 B2 in segment 2): their traced backward holds
    # one forward per block, removed again
    t = atom.atom_profile_trace(trace(b2=2 * (tb + tf), b1=emb_b + tb + tf), cfg, _plan([1, 3, 5], n_recompute=3))
    assert abs(t["cost_table"][3] / 1000.0 - tb) < 1e-6 and abs(t["cost_table"][1] / 1000.0 - emb_b) < 1e-6
    # hybrid: blocks 1..2 only -> segment 2 holds one of them (B1), segment 1 one (B0)
    t = atom.atom_profile_trace(trace(b2=2 * tb + tf, b1=emb_b + tb + tf), cfg, _plan([1, 3, 5], n_recompute=2))
    assert abs(t["cost_table"][3] / 1000.0 - tb) < 1e-6 and abs(t["cost_table"][1] / 1000.0 - emb_b) < 1e-6


def test_malformed_trace_is_rejected():
    import pytest
    with pytest.raises(atom.AtomError):
        atom.atom_profile_trace("compute FWD one\n", _cfg(), _plan([1, 5]))
