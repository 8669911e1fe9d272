"""Multi-peer host logic on CPU: world_size-2 gloo process group over 127.0.0.1.

Covers the N > 1 path without GPUs: libatom's NCCL id reaches every rank intact, the averaging
cadence follows the global batch, the timing reduction is the max over ranks, and the
n-peer averaging semantics the GPU peers implement (oracle.peers) hold rank by rank.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_10504_b200 import atom
        from paper_2403_10504_b200 import dist as adist
        nid = adist.bootstrap_nccl_id(atom.atom_nccl_unique_id)
        t = adist.max_over_ranks(float(10 + rank))
        # every rank trains its own replica on its own tokens; averaging = mean of the masters
        import synth
        from oracle import adamw, peers
        g = synth.GPTConfig("micro", 1, 16, 2, 8, 32, 2)
        p0 = synth.init_params(g, seed=3, dtype=np.float64)
        pr = peers.Peer(g, p0, adamw.AdamWHyper(lr=1e-2, warmup_steps=0))
        pr.step(synth.tokens(g, 2, synth.step_seed(rank, 0)))
        mine = torch.tensor(pr.p)
        tot = mine.clone()
        dist.all_reduce(tot)
        mean = (tot / world).numpy()
        q.put((rank, nid, t, mean, pr.p))
    finally:
        dist.destroy_process_group()


def test_two_rank_bootstrap_cadence_and_average():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    assert out[0][1] == out[1][1] and len(out[0][1]) == 128       # same NCCL id on both ranks
    assert out[0][2] == out[1][2] == 11.0                         # max over ranks
    from oracle import peers
    want = peers.average([out[0][4], out[1][4]])
    assert np.allclose(out[0][3], want) and np.allclose(out[1][3], want)
    assert not np.allclose(out[0][4], out[1][4])                   # replicas really diverged


def test_sync_cadence_from_global_batch():
    from paper_2403_10504_b200 import dist as adist
    assert adist.sync_every(1, 7, 8) == 0
    assert adist.sync_every(2, 7, 8) == 5          # ceil(512 / 112)
    assert adist.sync_every(8, 7, 8) == 2          # ceil(512 / 448)
    assert adist.sync_every(8, 64, 8) == 1
