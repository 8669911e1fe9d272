"""n-peer replica training with periodic parameter averaging (TEST INFRASTRUCTURE ONLY).

PAPER.md P:410: "allows volunteer nodes to independently train a copy of the
complete model and relies on an periodic allreduce communication to
synchronize copies of the model, in a way similar to data parallelism".
P:563: "The target group size to do the model averaging (ring-allreduce step)".

Readings (R16-R18): every peer holds a full replica (fp32 master,
AdamW m and v); one training step = forward/backward over the step's C
micro-batches (one flat batch of C*b sequences, loss = mean over all step
tokens) followed by AdamW; on a sync step the fp32 master
parameters (only) are replaced by their arithmetic mean over peers, after
that step's update.  m and v stay local.

Host update placement (R37; "CPU AdamW", Hivemind accumulating
gradients up to the target batch): with grad_rounds = R >= 1 a step is one gradient round; the
gradients of R rounds are summed and every R-th round AdamW takes one step with their mean.
"""
from __future__ import annotations

import numpy as np

from . import adamw, gpt


def average(params_list):
    """Equal-weight arithmetic mean of the peers' parameter vectors (fp64)."""
    return np.mean(np.stack([np.asarray(p, dtype=np.float64) for p in params_list]), axis=0)


class Peer:
    def __init__(self, cfg, init_params, hyper: adamw.AdamWHyper, grad_rounds: int = 0):
        self.cfg = cfg
        self.h = hyper
        self.p = np.asarray(init_params, dtype=np.float64).copy()
        self.m = np.zeros_like(self.p)
        self.v = np.zeros_like(self.p)
        self.t = 0
        self.R = grad_rounds
        self.gsum = np.zeros_like(self.p)
        self.rounds = 0

    def step(self, tokens):
        """One training step (or gradient round) on tokens [C*b, T+1]; returns the loss."""
        loss, g = gpt.loss_and_grad(self.cfg, self.p, tokens)
        if self.R <= 0:
            self.t += 1
            self.p, self.m, self.v = adamw.adamw_step(self.h, self.t, self.p, g, self.m, self.v)
            return loss, g
        self.gsum = self.gsum + g
        self.rounds += 1
        if self.rounds == self.R:
            self.t += 1
            self.p, self.m, self.v = adamw.adamw_step(self.h, self.t, self.p, self.gsum / self.R, self.m, self.v)
            self.gsum = np.zeros_like(self.p)
            self.rounds = 0
        return loss, g


def train(cfg, init_params, hyper, token_batches, sync_steps=()):
    """Emulate n peers in one process.

    token_batches[s][r] = tokens of peer r at step s (1-based step = s+1).
    After the update of every step whose 1-based index is in ``sync_steps``,
    all peers' masters are replaced by their mean.
    Returns (peers, losses[s][r]).
    """
    n = len(token_batches[0])
    peers = [Peer(cfg, init_params, hyper) for _ in range(n)]
    losses = []
    for s, batches in enumerate(token_batches):
        losses.append([pr.step(tok)[0] for pr, tok in zip(peers, batches)])
        if (s + 1) in sync_steps:
            mean = average([pr.p for pr in peers])
            for pr in peers:
                pr.p = mean.copy()
    return peers, losses
