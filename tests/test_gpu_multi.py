"""Two B200 peers averaging parameters over NCCL (atom_sync / sync_every) against the oracle.

PAPER.md P:410 / P:563: every peer trains a full replica on its own tokens; on a sync step the
fp32 masters become the mean over peers (m, v stay local).  Needs >= 2 GPUs (gpurun --gpus 2).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


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


def _worker(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2403_10504_b200 import atom
        from paper_2403_10504_b200 import dist as adist
        g = synth.CONFIGS["tiny"]
        C = 2
        cfg = atom.make_cfg(g, dtype=atom.FP32, C_=C, overlap_check=0, forced_ends=[2, 5], lr=1e-3,
                            warmup_steps=0, sync_every=2 if mode == "fused" else 0)
        plan = atom.atom_plan(cfg, 10 ** 11, 10 ** 10)
        nid = adist.bootstrap_nccl_id(atom.atom_nccl_unique_id)
        init = synth.init_params(g, seed=1234, perturb=True)
        peer = atom.Peer(cfg, plan, device=rank, init_params=init, nccl_id=nid, nranks=world, rank=rank)
        losses = []
        for s in range(2):
            toks = synth.tokens(g, C * g.micro_batch, synth.step_seed(rank, s))
            losses.append(peer.step(toks))
        if mode == "flush":
            atom.atom_sync([peer], flush=True)
        q.put((rank, losses, peer.params()))
        peer.destroy()
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("mode", ["fused", "flush"])
def test_two_peer_averaging_matches_oracle(mode):
    import torch.multiprocessing as mp

    import synth
    from oracle import adamw, peers
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = synth.CONFIGS["tiny"]
    C = 2
    toks = [[synth.tokens(g, C * g.micro_batch, synth.step_seed(r, s)) for r in range(2)] for s in range(2)]
    init = synth.init_params(g, seed=1234, perturb=True).astype(np.float64)
    prs, losses = peers.train(g, init, adamw.AdamWHyper(lr=1e-3, warmup_steps=0), toks, sync_steps={2})
    for r in range(2):
        got = out[r][2]
        assert np.linalg.norm(got["master"] - prs[r].p) <= 1e-4 * np.linalg.norm(prs[r].p)
        assert np.linalg.norm(got["m"] - prs[r].m) <= 1e-4 * np.linalg.norm(prs[r].m)   # moments stay local
        for s in range(2):
            assert abs(out[r][1][s] - losses[s][r]) <= 1e-4 * abs(losses[s][r])
    assert np.array_equal(out[0][2]["master"], out[1][2]["master"])     # replicas identical after averaging
    assert not np.array_equal(out[0][2]["m"], out[1][2]["m"])


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_two_local_peers_one_process_flush_matches_oracle():
    """atom_sync with n_local = 2 (both ranks' peers in one process, one NCCL group per segment):
    the masters of EVERY sub-model become the oracle's mean (sub-models 2..S used to
    keep their un-averaged values)."""
    import threading

    import synth
    from oracle import adamw, peers
    from paper_2403_10504_b200 import atom
    g = synth.CONFIGS["tiny"]
    C = 2
    cfg = atom.make_cfg(g, dtype=atom.FP32, C_=C, overlap_check=0, forced_ends=[2, 3, 5], lr=1e-3,
                        warmup_steps=0, sync_every=0)
    plan = atom.atom_plan(cfg, 10 ** 11, 10 ** 10)
    assert plan.n_seg == 3
    nid = atom.atom_nccl_unique_id()
    init = synth.init_params(g, seed=1234, perturb=True)
    out = [None, None]

    def make(r):   # ncclCommInitRank blocks until both ranks joined: one thread per local peer
        out[r] = atom.Peer(cfg, plan, device=r, init_params=init, nccl_id=nid, nranks=2, rank=r)

    th = [threading.Thread(target=make, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert all(p is not None for p in out)
    toks = [[synth.tokens(g, C * g.micro_batch, synth.step_seed(r, s)) for r in range(2)] for s in range(2)]
    for s in range(2):
        for r in range(2):
            out[r].step(toks[s][r])
    atom.atom_sync(out, flush=True)
    got = [p.params() for p in out]
    for p in out:
        p.destroy()
    ref = peers.train(g, init.astype(np.float64), adamw.AdamWHyper(lr=1e-3, warmup_steps=0), toks,
                      sync_steps={2})[0]
    for r in range(2):
        assert np.linalg.norm(got[r]["master"] - ref[r].p) <= 1e-4 * np.linalg.norm(ref[r].p)
    assert np.array_equal(got[0]["master"], got[1]["master"])
