"""Sub-model swap schedule and its integer-time simulation (TEST INFRASTRUCTURE ONLY).

PAPER.md Fig. 12 / P:305-317 and §IV P:459:
  "One [stream] is responsible for executing the current sub-model and the
   other one asynchronously prefetches the next sub-model immediately after
   the current sub-models starts. ... does not swap out the last sub-model at
   the end of the forward pass or the first sub-model at the end of the
   backward pass to exploit locality".

Readings (R10-R13): four lanes -- compute, h2d (prefetch), d2h
(evict; its own copy engine) and comm (peer averaging).  Segment 1 (which
holds the embedding) is never swapped: its weights, gradients and AdamW state
stay resident (R11), so a step neither loads nor stores it.  The last segment S runs its C
forward micro-batches interleaved with their backward (FWD S mb; BWD S mb)
and keeps its fp32 master from the forward load, so its backward load is the
AdamW moments only.  Slots come from a FIFO free list (the slot released
longest ago is reused first); logical slot ids are relabelled at the end of
every step so that each step starts from the queue [0 .. NSLOT-1] and emits
the identical program.

Canonical text: one op per line,
  ``<lane> <KIND> <seg> <mb|-> <slot|-> <waits|->``
with waits a comma-separated list of cross-lane dependencies ``KIND:seg``
(``PREV:s`` = the release of logical slot s in the previous step; ``HOST:k`` = the previous
step's STORE of segment k, after which segment k's host arena holds the updated state).
"""
from __future__ import annotations

from collections import deque


def emit(S: int, C: int, sync: bool = False):
    """The op list of one training step for S segments and C micro-batches."""
    return _emit(S, C, sync)[0]


def _emit(S: int, C: int, sync: bool):
    nslot = 0 if S == 1 else (2 if S == 2 else 3)
    q = deque(range(nslot))
    rel = {s: f"PREV:{s}" for s in range(nslot)}
    slot = {}
    ops = []

    def op(lane, kind, k, mb=None, s=None, waits=()):
        ops.append((lane, kind, k, mb, s, tuple(waits)))

    def alloc(k):
        s = q.popleft()
        slot[k] = s
        return s, rel[s]

    def release(s, ev):
        q.append(s)
        rel[s] = ev

    # ---- forward: segments 1..S (segment S interleaves its backward) ----
    for k in range(1, S + 1):
        if k >= 2:
            op("compute", "CAST", k, None, slot[k], [f"LOAD_F:{k}"])
        for mb in range(C):
            op("compute", "FWD", k, mb, slot.get(k) if k >= 2 else None)
            if mb == 0:
                if k < S:
                    s, w = alloc(k + 1)
                    op("h2d", "LOAD_F", k + 1, None, s, [w, f"HOST:{k + 1}"])
                elif S >= 2:
                    op("h2d", "LOAD_B", S, None, slot[S], [f"HOST:{S}"])   # AdamW moments of S only
                    if S - 1 >= 2:
                        s, w = alloc(S - 1)
                        op("h2d", "LOAD_B", S - 1, None, s, [w, f"HOST:{S - 1}"])
            if k == S:
                op("compute", "BWD", S, mb, slot.get(S))
        if 2 <= k < S:
            op("compute", "FREE", k, None, slot[k])
            release(slot[k], f"FREE:{k}")

    def finish(k):
        s = slot.get(k)
        op("compute", "ADAM", k, None, s, [f"LOAD_B:{k}"] if (k == S and S >= 2) else [])
        last = f"ADAM:{k}"
        if sync:
            op("comm", "AVG", k, None, s, [last])
            last = f"AVG:{k}"
            if k == 1:
                op("compute", "RECAST", 1, None, None, [last])
        if k >= 2:
            op("d2h", "STORE", k, None, s, [last])
            release(s, f"STORE:{k}")

    finish(S)
    # ---- backward: segments S-1..1 ----
    for k in range(S - 1, 0, -1):
        if k >= 2:
            op("compute", "CAST", k, None, slot[k], [f"LOAD_B:{k}"])
        for mb in range(C):
            op("compute", "BWD", k, mb, slot.get(k))
            if mb == 0 and k - 1 >= 2:
                s, w = alloc(k - 1)
                op("h2d", "LOAD_B", k - 1, None, s, [w, f"HOST:{k - 1}"])
        finish(k)
    return ops, list(q)


def to_text(ops) -> str:
    lines = []
    for lane, kind, k, mb, s, waits in ops:
        lines.append(f"{lane} {kind} {k} {'-' if mb is None else mb} {'-' if s is None else s} "
                     f"{','.join(waits) if waits else '-'}")
    return "\n".join(lines) + "\n"


def end_queue(S: int, C: int, sync: bool = False):
    """Logical FIFO order at the end of the step (before relabelling)."""
    return _emit(S, C, sync)[1]


def simulate(ops, ev, plan):
    """Integer-time list schedule of one step over 4 lanes.

    Durations (ns, from the planner's cost model ``ev``): FWD(k) = t_f(seg k),
    BWD(k) = t_b(seg k), LOAD_F = t_loadF, LOAD_B = t_loadB (t_mv for the last
    segment when S >= 2), STORE = t_store; CAST/FREE/ADAM/AVG/RECAST = 0.
    Each op starts when its lane is free and its waits are complete (PREV = 0).
    Returns makespan, and the share of copy time that overlaps compute (ppm)."""
    segs = ev.segments(plan.seg_end)
    S = len(segs)

    def seg(name, k):
        i, j = segs[k - 1]
        return ev.s(name, i, j)

    lane_t = {"compute": 0, "h2d": 0, "d2h": 0, "comm": 0}
    done = {}
    comp, copies = [], []
    for lane, kind, k, mb, s, waits in ops:
        if kind == "FWD":
            dur = seg("tf", k)
        elif kind == "BWD":
            i, j = segs[k - 1]
            dur = seg("tb", k) if k == S else ev.tbn(i, j)
        elif kind == "LOAD_F":
            dur = seg("tlf", k)
        elif kind == "LOAD_B":
            dur = seg("tmv", k) if (k == S and S >= 2) else seg("tlb", k)
        elif kind == "STORE":
            dur = seg("ts", k)
        else:
            dur = 0
        start = lane_t[lane]
        for w in waits:
            if not w.startswith(("PREV", "HOST")):
                start = max(start, done[w])
        end = start + dur
        lane_t[lane] = end
        done[f"{kind}:{k}"] = end
        if lane == "compute" and dur > 0:
            comp.append((start, end))
        if lane in ("h2d", "d2h") and dur > 0:
            copies.append((start, end))
    makespan = max(lane_t.values())
    tot = sum(e - s for s, e in copies)
    hid = 0
    for s0, e0 in copies:
        for s1, e1 in comp:
            lo, hi = max(s0, s1), min(e0, e1)
            if hi > lo:
                hid += hi - lo
    ppm = (hid * 1_000_000) // tot if tot else 1_000_000
    return {"makespan": makespan, "hidden_ppm": ppm, "copy_ns": tot, "hidden_ns": hid}
