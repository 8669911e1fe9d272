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
