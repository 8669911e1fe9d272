"""Elastic peers on B200s (PAPER P:410 peers join and leave, P:563 GPUs killed
mid-training): real atom peers average over NCCL on sync steps chosen by the global-batch
trigger (paper_2403_10504_b200/elastic.py); one peer dies abruptly, the survivors drop it with
ncclCommShrink (atom_comm_shrink) and train on; a joiner takes the dead peer's GPU, gets a fresh
communicator (atom_comm_reset) and adopts the leader's state (atom_broadcast_state).

Checked through the C-ABI: every sync step leaves all members with bit-identical fp32 masters;
right after admission the joiner's master, m, v and step count equal the leader's; training
completes every step on every survivor.  Needs >= 2 GPUs (gpurun --gpus 2 or 4).
"""
import datetime
import hashlib
import json
import multiprocessing as mp
import os
import socket
import sys
import time

import pytest

pytestmark = pytest.mark.gpu

STEPS, GLOBAL_BATCH, TTL, KILL_AT, JOINER = 10, 12, 4.0, 2, 10


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _digest(peer):
    p = peer.params()
    return {k: hashlib.sha256(v.tobytes()).hexdigest() for k, v in p.items()}


def _peer(pid, n0, port, q):
    import torch
    import torch.distributed as dist
    store = dist.TCPStore("127.0.0.1", port, is_master=False, timeout=datetime.timedelta(seconds=300))
    victim = n0 - 1
    gpu = pid if pid != JOINER else victim
    if pid == JOINER:   # wait until the victim's failure has been handled (its GPU is free)
        while not store.check([f"dec/{KILL_AT + 2}"]):
            time.sleep(0.01)
    torch.cuda.set_device(gpu)
    import synth
    from paper_2403_10504_b200 import atom, elastic
    g = synth.CONFIGS["tiny"]
    C = 2
    cfg = atom.make_cfg(g, dtype=atom.BF16, C_=C, overlap_check=0, forced_ends=[2, 5], lr=1e-3, warmup_steps=0)
    plan = atom.atom_plan(cfg, 10 ** 11, 10 ** 10)
    init = synth.init_params(g, seed=1234, perturb=True)
    co = elastic.Coordinator(store, pid, GLOBAL_BATCH, ttl=TTL, make_id=atom.atom_nccl_unique_id)
    log = {"pid": pid, "decs": [], "hash": {}, "info": {}}
    if pid == JOINER:
        peer = atom.Peer(cfg, plan, device=gpu, init_params=synth.init_params(g, seed=99), seed=0)
        print(f"[elastic peer {pid}] registering as joiner", file=sys.stderr, flush=True)
        d = co.join()
        co.apply(d, peer, atom.atom_sync)
        log["decs"].append(d.to_json())
        log["hash"][f"admit{d.s}"] = _digest(peer)
        log["info"][f"admit{d.s}"] = peer.info()
    else:
        if pid == 0:
            store.set("nccl0", atom.atom_nccl_unique_id().hex())
        nid = bytes.fromhex(store.get("nccl0").decode())
        peer = atom.Peer(cfg, plan, device=gpu, init_params=init, seed=0, nccl_id=nid, nranks=n0, rank=pid)
        co.start(list(range(n0)))
    while co.s < STEPS - 1:
        if pid != JOINER and co.s == STEPS - 4:
            # the joiner starts a fresh process after dec/{KILL_AT + 2}; on a fast box the members
            # could finish every step before it registers, so hold until its ticket exists
            while not store.check(["join/0"]):
                time.sleep(0.01)
        print(f"[elastic peer {pid}] s={co.s} members={co.members}", file=sys.stderr, flush=True)
        toks = synth.tokens(g, C * g.micro_batch, synth.step_seed(pid, co.s + 1))
        peer.step(toks)
        torch.cuda.synchronize()
        was_sync = co.sync_step
        d = co.after_step(C * g.micro_batch)
        if was_sync:
            log["hash"][f"sync{d.s}"] = _digest(peer)
        co.apply(d, peer, atom.atom_sync)
        if d.joiners:
            log["hash"][f"admit{d.s}"] = _digest(peer)
            log["info"][f"admit{d.s}"] = peer.info()
        log["decs"].append(d.to_json())
        if pid == victim and d.s >= KILL_AT and not d.sync:
            q.put(json.dumps(log))
            q.close()
            q.join_thread()
            os._exit(0)    # abrupt failure between steps: no leave, no destroy
    log["info"]["end"] = peer.info()
    q.put(json.dumps(log))
    peer.destroy()


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_failure_shrink_join_and_averaging():
    import torch.distributed as dist
    n0 = min(_ngpu(), 3)
    victim = n0 - 1
    port = _free_port()
    server = dist.TCPStore("127.0.0.1", port, is_master=True, wait_for_workers=False,
                           timeout=datetime.timedelta(seconds=300))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pids = list(range(n0)) + [JOINER]
    procs = [ctx.Process(target=_peer, args=(pid, n0, port, q)) for pid in pids]
    for p in procs:
        p.start()
    logs = {}
    for _ in procs:
        lg = json.loads(q.get(timeout=600))
        logs[lg["pid"]] = lg
    for p in procs:
        p.join(timeout=60)
    del server
    decs = {}
    for lg in logs.values():
        for d in lg["decs"]:
            d = json.loads(d)
            assert decs.setdefault(d["s"], d) == d
    assert sorted(decs) == list(range(STEPS))
    s_kill = json.loads(logs[victim]["decs"][-1])["s"]
    assert decs[s_kill + 1]["dead"] == [victim]
    adm = [d for d in decs.values() if d["joiners"]]
    assert len(adm) == 1 and adm[0]["joiners"] == [JOINER]
    a = adm[0]
    leader = a["leader"]
    # the joiner adopted the leader's master, m, v and step count, bit for bit
    key = f"admit{a['s']}"
    assert logs[JOINER]["hash"][key] == logs[leader]["hash"][key]
    assert logs[JOINER]["info"][key]["step"] == logs[leader]["info"][key]["step"]
    assert logs[JOINER]["info"][key]["nranks"] == len(a["members"])
    # every sync step left the members with identical masters (m, v stay local, R16)
    syncs = [s for s in decs if decs[s]["sync"] and s + 1 in decs and len(decs[s]["members"]) > 1]
    assert syncs, decs
    for s in syncs:
        hs = [logs[m]["hash"][f"sync{s + 1}"]["master"] for m in decs[s]["members"]]
        assert len(set(hs)) == 1, (s, decs[s]["members"])
    # survivors and the joiner finished every step
    for pid in [p for p in pids if p != victim]:
        assert json.loads(logs[pid]["decs"][-1])["s"] == STEPS - 1


# ---------------------------------------------------------------------------------------------
# A peer dies INSIDE an averaging round (PAPER P:563 kills GPUs mid-training):
# with every step a sync step, peer 1 issues a step and exits while that step's backward -- whose
# fused per-sub-model averaging waits for it -- is still running.  The survivor's averaging is
# stuck on its comm stream; the coordinator declares peer 1 dead after its TTL and the survivor
# shrinks with abort_ops (atom_comm_shrink): the outstanding NCCL operations are aborted, the
# streams drain, and the guarded commit (R36) leaves each sub-model's master either
# averaged (its round completed on both ranks before the failure) or the survivor's own update --
# never a partial reduction.  Checked against the fp64 oracle replaying each of those outcomes.
A_STEPS, A_KILL, A_TTL = 6, 3, 3.0


def _avg_peer(pid, port, q):
    import torch
    import torch.distributed as dist
    store = dist.TCPStore("127.0.0.1", port, is_master=False, timeout=datetime.timedelta(seconds=300))
    torch.cuda.set_device(pid)
    import synth
    from paper_2403_10504_b200 import atom, elastic
    g = synth.CONFIGS["tiny"]
    C = 2
    cfg = atom.make_cfg(g, dtype=atom.FP32, C_=C, overlap_check=0, forced_ends=[2, 5], lr=1e-3, warmup_steps=0,
                        sync_every=1)
    plan = atom.atom_plan(cfg, 10 ** 11, 10 ** 10)
    init = synth.init_params(g, seed=1234, perturb=True)
    if pid == 0:
        store.set("nccl_avg", atom.atom_nccl_unique_id().hex())
    nid = bytes.fromhex(store.get("nccl_avg").decode())
    peer = atom.Peer(cfg, plan, device=pid, init_params=init, seed=0, nccl_id=nid, nranks=2, rank=pid)
    co = elastic.Coordinator(store, pid, 10 ** 9, ttl=A_TTL, make_id=atom.atom_nccl_unique_id)
    co.start([0, 1])
    decs = []
    for s in range(A_STEPS):
        peer.step(synth.tokens(g, C * g.micro_batch, synth.step_seed(pid, s)))
        if pid == 1 and s == A_KILL:
            os._exit(0)    # the step's backward (with its averaging rounds) is still in flight
        d = co.after_step(C * g.micro_batch)
        co.apply(d, peer, atom.atom_sync)
        decs.append(d.to_json())
    master = peer.params()["master"]
    peer.destroy()
    q.put((pid, decs, master.tobytes()))


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_failure_inside_averaging_round_is_recovered():
    import itertools

    import numpy as np
    import torch.distributed as dist

    import synth
    from oracle import adamw, gpt, peers
    port = _free_port()
    server = dist.TCPStore("127.0.0.1", port, is_master=True, wait_for_workers=False,
                           timeout=datetime.timedelta(seconds=300))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_avg_peer, args=(pid, port, q)) for pid in range(2)]
    for p in procs:
        p.start()
    pid, decs, mbytes = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
    del server
    assert pid == 0
    decs = [json.loads(d) for d in decs]
    assert [d["s"] for d in decs] == list(range(A_STEPS))
    assert decs[A_KILL]["dead"] == [1] and decs[-1]["members"] == [0]
    got = np.frombuffer(mbytes, dtype=np.float32)
    # oracle: both peers average after every update up to step A_KILL - 1; at step A_KILL each of
    # the two sub-models is either averaged or keeps peer 0's update; then peer 0 trains alone
    g = synth.CONFIGS["tiny"]
    C = 2
    h = adamw.AdamWHyper(lr=1e-3, warmup_steps=0)
    init = synth.init_params(g, seed=1234, perturb=True).astype(np.float64)
    prs = [peers.Peer(g, init, h) for _ in range(2)]
    for s in range(A_KILL + 1):
        for r in range(2):
            prs[r].step(synth.tokens(g, C * g.micro_batch, synth.step_seed(r, s)))
        if s < A_KILL:
            mean = peers.average([pr.p for pr in prs])
            for pr in prs:
                pr.p = mean.copy()
    nodes = gpt.node_ranges(g)
    segs = [(nodes[0][0], nodes[2][1]), (nodes[3][0], nodes[5][1])]     # sub-models [E B0 B1 | B2 B3 H]
    mean = peers.average([pr.p for pr in prs])
    matched = []
    for choice in itertools.product([0, 1], repeat=2):   # 1 = that sub-model's round committed
        pr = peers.Peer(g, prs[0].p, h)
        pr.p, pr.m, pr.v, pr.t = prs[0].p.copy(), prs[0].m.copy(), prs[0].v.copy(), prs[0].t
        for (a, b), c in zip(segs, choice):
            if c:
                pr.p[a:b] = mean[a:b]
        for s in range(A_KILL + 1, A_STEPS):
            pr.step(synth.tokens(g, C * g.micro_batch, synth.step_seed(0, s)))
        err = np.linalg.norm(got - pr.p) / np.linalg.norm(pr.p)
        if err <= 1e-5:
            matched.append(choice)
    assert len(matched) == 1, matched
