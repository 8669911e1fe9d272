"""Host-side multi-peer plumbing (torch.distributed is only the bootstrap / timing channel).

PAPER.md P:410: peers "independently train a copy of the complete model and [rely] on a
periodic allreduce communication to synchronize copies of the model"; averaging once
a global batch of 512 samples has been processed.  One process per GPU; the parameter
averaging itself is NCCL inside libatom (atom_sync / sync_every); this module only
* distributes libatom's NCCL unique id from rank 0 (``bootstrap_nccl_id``),
* derives the averaging cadence from the global batch (``sync_every``, reading R17),
* reduces a per-rank device time to the max over ranks (``max_over_ranks``).
"""
from __future__ import annotations

import math


def sync_every(world: int, C: int, micro_batch: int, global_batch: int = 512) -> int:
    """Steps between parameter averages: ceil(G / (n C b)); 0 (never) for a single peer."""
    if world <= 1:
        return 0
    return max(1, math.ceil(global_batch / (world * C * micro_batch)))


def bootstrap_nccl_id(make_id, group=None) -> bytes:
    """Rank 0 calls ``make_id()`` (atom_nccl_unique_id) and broadcasts the 128 bytes."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    nid = obj[0]
    if not isinstance(nid, (bytes, bytearray)) or len(nid) != 128:
        raise RuntimeError("NCCL unique id broadcast failed")
    return bytes(nid)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank float over all ranks (the multi-GPU timing rule)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
