"""Pins for oracle/schedule.py: the invariants of SPEC S:229-259 and P:459 locality."""
import pytest

import synth
from oracle import planner as pl
from oracle import schedule as sc


def _check_program(S, C, sync):
    ops = sc.emit(S, C, sync)
    nslot = 0 if S == 1 else (2 if S == 2 else 3)
    held = {}
    loads_f, loads_b, stores = {}, {}, {}
    seen_bwd = []
    for lane, kind, k, mb, s, waits in ops:
        if kind in ("LOAD_F",) or (kind == "LOAD_B" and (k != S or S == 1)):
            assert s is not None and 0 <= s < nslot
            assert s not in held.values() or held.get(k) == s, ("slot reused while held", S, C)
            held[k] = s
        if kind == "LOAD_F":
            loads_f[k] = loads_f.get(k, 0) + 1
        if kind == "LOAD_B":
            loads_b[k] = loads_b.get(k, 0) + 1
        if kind == "STORE":
            stores[k] = stores.get(k, 0) + 1
            held.pop(k)
        if kind == "FREE":
            held.pop(k)
        if kind == "BWD":
            seen_bwd.append((k, mb))
        if kind in ("FWD", "BWD", "CAST", "ADAM") and k >= 2:
            assert held.get(k) == s, (kind, k)           # compute only on a resident segment
    # locality: segment 1 never moves; the last forward segment is not evicted
    assert 1 not in loads_f and 1 not in loads_b and 1 not in stores
    assert all(not (kind == "FREE" and k == S) for _, kind, k, *_ in ops)
    assert all(loads_f.get(k) == 1 and stores.get(k) == 1 and loads_b.get(k) == 1 for k in range(2, S + 1))
    # backward order: S..1, micro-batches ascending (canonical accumulation order)
    order = [k for k, _ in seen_bwd]
    assert order == sorted(order, reverse=True)
    for k in range(1, S + 1):
        assert [mb for kk, mb in seen_bwd if kk == k] == list(range(C))
    return ops


@pytest.mark.parametrize("sync", [False, True])
def test_program_invariants(sync):
    for S in range(1, 9):
        for C in range(1, 5):
            _check_program(S, C, sync)


def test_text_is_deterministic_and_relabelling_is_a_permutation():
    for S in range(1, 7):
        a, b = sc.to_text(sc.emit(S, 3)), sc.to_text(sc.emit(S, 3))
        assert a == b
        q = sc.end_queue(S, 3)
        assert sorted(q) == list(range(0 if S == 1 else (2 if S == 2 else 3)))


# tiny's fully resident state is 4.23 MB (bf16 path R1 = 18 B/param); cap the model state below it
STATE_CAP = 4 * 10 ** 6


def _tiny_eval(C, ends, overlap=1):
    g = synth.CONFIGS["tiny"]
    c = pl.PlanCfg.from_gpt(g, C=C, overlap_check=overlap,
                           cost_table=[0, 0] + [10, 20] * g.n_layer + [10, 20])
    return pl.Evaluator(c, 10 ** 12, 10 ** 9), c


def test_no_exec_before_load_and_zero_idle_when_constraints_hold():
    g = synth.CONFIGS["tiny"]
    checked = 0
    for link in (10 ** 8, 3 * 10 ** 8, 10 ** 9):
        c = pl.PlanCfg.from_gpt(g, max_C=64, cost_table=[0, 0] + [400_000, 800_000] * g.n_layer + [300_000, 600_000],
                               state_budget=STATE_CAP)
        p = pl.plan(c, 10 ** 12, link)
        assert p.n_seg >= 2
        checked += 1
        ev = pl.Evaluator(c, 10 ** 12, link)
        ops = sc.emit(p.n_seg, p.C)
        sim = sc.simulate(ops, ev, p)
        assert sim["hidden_ppm"] > 0
        # compute lane never waits: it finishes at exactly the sum of its durations
        busy = p.C * (sum(ev.k.tf) + sum(ev.k.tb))
        assert _compute_end(ops, ev, p) == busy, link
    assert checked == 3


def _compute_end(ops, ev, p):
    segs = ev.segments(p.seg_end)
    S = len(segs)
    lane = {"compute": 0, "h2d": 0, "d2h": 0, "comm": 0}
    done = {}
    for ln, kind, k, mb, s, waits in ops:
        i, j = segs[k - 1]
        dur = {"FWD": ev.s("tf", i, j), "BWD": ev.s("tb", i, j), "LOAD_F": ev.s("tlf", i, j),
               "LOAD_B": ev.s("tmv", i, j) if (k == S and S >= 2) else ev.s("tlb", i, j),
               "STORE": ev.s("ts", i, j)}.get(kind, 0)
        t0 = max([lane[ln]] + [done[w] for w in waits if not w.startswith(("PREV", "HOST"))])
        lane[ln] = t0 + dur
        done[f"{kind}:{k}"] = t0 + dur
    return lane["compute"]


def test_positive_idle_with_one_less_micro_batch():
    """the same plan run with C-1 micro-batches stalls the compute lane."""
    g = synth.CONFIGS["tiny"]
    # the forward prefetch binds (t_f small next to the load), the backward is slack
    c = pl.PlanCfg.from_gpt(g, max_C=64, cost_table=[0, 0] + [100_000, 2_000_000] * g.n_layer + [100_000, 2_000_000],
                           state_budget=STATE_CAP)
    link = 10 ** 9
    p = pl.plan(c, 10 ** 12, link)
    assert p.n_seg >= 3 and p.C >= 2
    ev = pl.Evaluator(c, 10 ** 12, link)
    q = pl.Evaluator(c, 10 ** 12, link).make_plan(p.C - 1, p.seg_end)
    end = _compute_end(sc.emit(p.n_seg, p.C - 1), ev, q)
    assert end > (p.C - 1) * (sum(ev.k.tf) + sum(ev.k.tb))


# ---------------------------------------------------------------------------------------------
# Hand-computed pins for simulate() (SPEC S:233-234 build_schedule examples, "hand-built
# 3-segment instance evaluated against an event-by-event trace").  The durations are given per
# segment directly (no planner cost model involved), so a wrong duration lookup, a dropped wait
# or a wrong lane in simulate() changes the exact makespan / hidden numbers below.
class _HandEv:
    """Segment k is node k (seg_end = [1, 2, ..., S]); s(name, k, k) = the table's value for k."""

    def __init__(self, **tables):
        self.t = tables

    def segments(self, ends):
        return [(k, k) for k in ends]

    def s(self, name, i, j):
        assert i == j
        return self.t[name].get(i, 0)

    def tbn(self, i, j):
        return self.t["tbx"].get(i, 0)


class _HandPlan:
    def __init__(self, S):
        self.seg_end = list(range(1, S + 1))


def _busy(ev, S, C):
    return sum(C * ev.s("tf", k, k) for k in range(1, S + 1)) + C * ev.s("tb", S, S) + \
        sum(C * ev.tbn(k, k) for k in range(1, S))


def test_simulate_two_segments_overlap_with_equality_has_zero_idle():
    """C t_fwd(seg 1) = t_load(seg 2) -> idle 0, the transfer lane busy during the exec."""
    ev = _HandEv(tf={1: 10, 2: 5}, tbx={1: 20}, tb={2: 10}, tlf={2: 20}, tmv={2: 8}, ts={2: 12})
    sim = sc.simulate(sc.emit(2, 2), ev, _HandPlan(2))
    # trace: FWD1 [0,10] [10,20] | LOAD_F2 [0,20] | CAST2 20 | FWD2 [20,25] | LOAD_B2 (m,v) [20,28]
    # BWD2 [25,35] | FWD2 [35,40] | BWD2 [40,50] | ADAM2 50 | STORE2 [50,62] | BWD1 [50,70] [70,90]
    assert sim["makespan"] == 90 == _busy(ev, 2, 2)
    assert sim["copy_ns"] == 20 + 8 + 12
    assert sim["hidden_ns"] == 40 and sim["hidden_ppm"] == 1_000_000


def test_simulate_one_less_micro_batch_idles_by_the_shortfall():
    """the same instance with C - 1 = 1: idle = sum of (load - compute) shortfalls = 20 - 10."""
    ev = _HandEv(tf={1: 10, 2: 5}, tbx={1: 20}, tb={2: 10}, tlf={2: 20}, tmv={2: 8}, ts={2: 12})
    sim = sc.simulate(sc.emit(2, 1), ev, _HandPlan(2))
    # FWD1 [0,10] | LOAD_F2 [0,20] | CAST2 waits -> 20 | FWD2 [20,25] | LOAD_B2 [20,28] | BWD2 [25,35]
    # ADAM2 35 | STORE2 [35,47] | BWD1 [35,55]
    assert _busy(ev, 2, 1) == 45
    assert sim["makespan"] == 55 == 45 + (20 - 10)
    # hidden: LOAD_F2 10 (FWD1), LOAD_B2 5 + 3 (FWD2, BWD2), STORE2 12 (BWD1) of 40 copied
    assert sim["copy_ns"] == 40 and sim["hidden_ns"] == 30
    assert sim["hidden_ppm"] == 750_000


def test_simulate_three_segment_event_by_event_trace():
    """hand-built 3-segment instance (C = 2) against the trace written out below."""
    ev = _HandEv(tf={1: 10, 2: 6, 3: 4}, tbx={1: 20, 2: 12}, tb={3: 8}, tlf={2: 14, 3: 9},
                 tlb={2: 30}, tmv={3: 5}, ts={2: 16, 3: 11})
    ops = sc.emit(3, 2)
    kinds = [(ln, kind, k, mb) for ln, kind, k, mb, _, _ in ops]
    assert kinds == [
        ("compute", "FWD", 1, 0), ("h2d", "LOAD_F", 2, None), ("compute", "FWD", 1, 1),
        ("compute", "CAST", 2, None), ("compute", "FWD", 2, 0), ("h2d", "LOAD_F", 3, None),
        ("compute", "FWD", 2, 1), ("compute", "FREE", 2, None), ("compute", "CAST", 3, None),
        ("compute", "FWD", 3, 0), ("h2d", "LOAD_B", 3, None), ("h2d", "LOAD_B", 2, None),
        ("compute", "BWD", 3, 0), ("compute", "FWD", 3, 1), ("compute", "BWD", 3, 1),
        ("compute", "ADAM", 3, None), ("d2h", "STORE", 3, None), ("compute", "CAST", 2, None),
        ("compute", "BWD", 2, 0), ("compute", "BWD", 2, 1), ("compute", "ADAM", 2, None),
        ("d2h", "STORE", 2, None), ("compute", "BWD", 1, 0), ("compute", "BWD", 1, 1),
        ("compute", "ADAM", 1, None)]
    sim = sc.simulate(ops, ev, _HandPlan(3))
    # compute: FWD1 [0,10] [10,20]; FWD2 [20,26] [26,32]; FWD3 [32,36]; BWD3 [36,44]; FWD3 [44,48];
    #          BWD3 [48,56]; CAST2 waits LOAD_B2 (58): idle 2; BWD2 [58,70] [70,82]; BWD1 [82,102] [102,122]
    # h2d:     LOAD_F2 [0,14]; LOAD_F3 [14,23]; LOAD_B3 (m,v) [23,28]; LOAD_B2 [28,58]
    # d2h:     STORE3 [56,67]; STORE2 [82,98]
    assert _busy(ev, 3, 2) == 120
    assert sim["makespan"] == 122
    assert sim["copy_ns"] == 14 + 9 + 5 + 30 + 11 + 16
    # hidden: 14 + (6 + 3) + (3 + 2) + (4 + 4 + 8 + 4 + 8) + 9 + 16
    assert sim["hidden_ns"] == 81
    assert sim["hidden_ppm"] == 81_000_000 // 85
