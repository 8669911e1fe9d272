"""Measured profile feeding the planner ("the model is profiled
offline", "We empirically determine C offline via profiling for a particular GPU").

The arithmetic lives in the library (csrc/profile.cpp, atom_profile / atom_profile_trace): the
compute rate the step sustains (FLOPs executed / compute-lane busy time), the achieved copy rates
and the per-node cost table, all from the per-op CUDA-event trace of a step run with a first plan.
This module only runs that first plan for a few steps and hands back atom_profile's numbers; the
plan is then recomputed with them (R34).
"""
from . import atom


def measure(cfg, plan, tokens_dev, device: int = 0, steps: int = 3) -> dict:
    """Profile `plan` on this GPU: run `steps` steps on device tokens, then atom_profile on the last
    step. Returns {"flops", "h2d", "d2h", "compute_busy_ms", "executed_flops", "cost_table"}."""
    peer = atom.Peer(cfg, plan, device=device, init_params=None, seed=1234)
    try:
        for s in range(steps):
            peer.step_device(tokens_dev[s % len(tokens_dev)])
        return peer.profile()
    finally:
        import torch
        peer.destroy()
        peer.arena = None          # hand the arena back to the driver before the real plan allocates
        torch.cuda.empty_cache()
