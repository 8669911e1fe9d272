"""Elastic peers, host logic (SPEC S:363-405 test ideas):
DHT-style heartbeats with TTL, the global-batch averaging trigger, a peer failing mid-run and a
peer joining.  Five CPU processes share a TCPStore on 127.0.0.1; the "peers" are recorders of the
membership calls (the device side is tests/test_gpu_elastic.py)."""
import json
import multiprocessing as mp
import os
import socket
import time

import pytest

STEPS, PER_STEP, GLOBAL_BATCH, TTL = 14, 2, 12, 1.0
KILL_AT, JOINER = 4, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class Recorder:
    """Stands in for atom.Peer: records the collective membership calls."""

    def __init__(self):
        self.calls = []

    def comm_reset(self, nid, n, r):
        self.calls.append(("reset", n, r))

    def comm_shrink(self, ex, abort_ops=False):
        self.calls.append(("shrink", list(ex)))

    def broadcast_state(self, root, adopt):
        self.calls.append(("bcast", root, bool(adopt)))


def _peer(pid, port, q, VICTIM):
    import torch.distributed as dist
    from paper_2403_10504_b200 import elastic
    store = dist.TCPStore("127.0.0.1", port, is_master=False, timeout=__import__("datetime").timedelta(seconds=60))
    co = elastic.Coordinator(store, pid, GLOBAL_BATCH, ttl=TTL, make_id=lambda: os.urandom(128))
    rec, decs, processed = Recorder(), [], 0
    if pid == JOINER:
        while not store.check([f"dec/{KILL_AT + 3}"]):   # arrives after the failure was handled
            time.sleep(0.01)
        d = co.join()
        co.apply(d, rec)
        decs.append(d.to_json())
    else:
        co.start([0, 1, 2, 3])
    while co.s < STEPS - 1:
        time.sleep(0.05)                       # one "training step"
        processed += PER_STEP
        d = co.after_step(PER_STEP)
        co.apply(d, rec)
        decs.append(d.to_json())
        if pid == VICTIM and d.s >= KILL_AT and not d.sync:
            q.put((pid, decs, processed, rec.calls, co.count))
            q.close()
            q.join_thread()
            os._exit(0)                        # abrupt failure: no leave, no further heartbeat
    q.put((pid, decs, processed, rec.calls, co.count))


@pytest.mark.parametrize("VICTIM", [3, 0], ids=["member-fails", "leader-fails"])
def test_heartbeat_trigger_failure_and_join(VICTIM):
    import datetime

    import torch.distributed as dist
    port = _free_port()
    server = dist.TCPStore("127.0.0.1", port, is_master=True, wait_for_workers=False,
                           timeout=datetime.timedelta(seconds=60))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer, args=(pid, port, q, VICTIM)) for pid in range(5)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        pid, decs, processed, calls, count = q.get(timeout=120)
        out[pid] = {"decs": [json.loads(d) for d in decs], "processed": processed, "calls": calls, "count": count}
    for p in procs:
        p.join(timeout=30)
    del server

    # 1. every member applies the same decision at every boundary it reached
    by_s = {}
    for pid, o in out.items():
        for d in o["decs"]:
            by_s.setdefault(d["s"], []).append((pid, json.dumps(d, sort_keys=True)))
    for s, lst in by_s.items():
        assert len({j for _, j in lst}) == 1, (s, lst)
    dec = {s: json.loads(lst[0][1]) for s, lst in by_s.items()}
    steps = sorted(dec)
    assert steps == list(range(STEPS)), steps

    # 2. the victim is dropped at the first boundary after its failure, with a shrink of its rank
    s_kill = out[VICTIM]["decs"][-1]["s"]
    d_drop = dec[s_kill + 1]
    assert d_drop["dead"] == [VICTIM] and VICTIM not in d_drop["members"]
    for pid in (p for p in range(4) if p != VICTIM):
        assert ("shrink", [d_drop["prev"].index(VICTIM)]) in out[pid]["calls"]

    # 3. the joiner is admitted once, with a fresh communicator and the leader's state
    adm = [dec[s] for s in steps if dec[s]["joiners"]]
    assert len(adm) == 1 and adm[0]["joiners"] == [JOINER] and JOINER in adm[0]["members"]
    a = adm[0]
    for pid in a["members"]:
        calls = out[pid]["calls"]
        assert ("reset", len(a["members"]), a["members"].index(pid)) in calls
        assert ("bcast", a["members"].index(a["leader"]), pid == JOINER) in calls
    assert all(JOINER in dec[s]["members"] for s in steps if s > a["s"])

    # 4. trigger correctness: sync exactly when the live members' count reaches the
    #    global batch; the count restarts after each sync step
    for s in steps:
        assert dec[s]["sync"] == (dec[s]["total"] >= GLOBAL_BATCH), dec[s]
        assert dec[s]["total"] == sum(dec[s]["counts"].values())
    assert sum(dec[s]["sync"] for s in steps) >= 3

    # 5. conservation ledger: every processed sequence is either in an averaged
    #    round (a trigger's total or a sync step's own samples), lost with the failed peer, or
    #    still outstanding at the end
    processed = sum(o["processed"] for o in out.values())
    averaged = sum(dec[s]["total"] for s in steps if dec[s]["sync"])
    sync_steps = sum(PER_STEP * len(dec[s]["members"]) for s in steps if dec[s]["sync"] and s + 1 in dec)
    lost = dec[s_kill]["counts"][str(VICTIM)] if str(VICTIM) in dec[s_kill]["counts"] else dec[s_kill]["counts"][VICTIM]
    last = dec[steps[-1]]
    outstanding = 0 if last["sync"] else last["total"]
    assert processed == averaged + sync_steps + lost + outstanding, (processed, averaged, sync_steps, lost, outstanding)


def _slow_peer(pid, port, q, ttl, slow):
    import torch.distributed as dist
    from paper_2403_10504_b200 import elastic
    store = dist.TCPStore("127.0.0.1", port, is_master=False, timeout=__import__("datetime").timedelta(seconds=60))
    co = elastic.Coordinator(store, pid, 10 ** 9, ttl=ttl, boot_grace=5.0)
    co.start([0, 1, 2])
    decs = []
    for s in range(3):
        time.sleep(slow if pid == 2 else 0.01)   # peer 2's steps take 4 TTLs
        decs.append(co.after_step(1).to_json())
    co.stop()
    q.put((pid, decs))


def test_step_longer_than_ttl_keeps_the_member_alive():
    """heartbeats were only written between steps, so a step longer than ~ttl made a
    live member stale and the group collapsed.  The heartbeat thread keeps it fresh."""
    import datetime

    import torch.distributed as dist
    port = _free_port()
    server = dist.TCPStore("127.0.0.1", port, is_master=True, wait_for_workers=False,
                           timeout=datetime.timedelta(seconds=60))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ttl = 0.5
    procs = [ctx.Process(target=_slow_peer, args=(pid, port, q, ttl, 4 * ttl)) for pid in range(3)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=30)
    del server
    for pid, decs in out.items():
        for d in map(json.loads, decs):
            assert d["dead"] == [] and d["members"] == [0, 1, 2], (pid, d)
