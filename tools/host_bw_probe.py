"""Pinned host<->device copy rates when every local GPU copies at once (torchrun, one rank per GPU):
H2D alone, D2H alone, and both directions together, 2 GiB per direction per rank, after a barrier."""
import json, os, time
import torch
import torch.distributed as dist

rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
nb = 2 << 30
h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, ops in [("h2d", [(s1, lambda: d.copy_(h, non_blocking=True))]),
                  ("d2h", [(s2, lambda: h2.copy_(d2, non_blocking=True))]),
                  ("bidir", [(s1, lambda: d.copy_(h, non_blocking=True)), (s2, lambda: h2.copy_(d2, non_blocking=True))])]:
    for rep in range(2):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(); torch.cuda.synchronize()
        t = time.perf_counter()
        for s, fn in ops:
            with torch.cuda.stream(s):
                for _ in range(3):
                    fn()
        torch.cuda.synchronize()
        res[name] = round(3 * nb / (time.perf_counter() - t) / 1e9, 1)
out = [None] * world
if world > 1:
    dist.all_gather_object(out, res)
else:
    out = [res]
if rank == 0:
    print(json.dumps({"world": world, "GBs_per_rank": out}))
if world > 1:
    dist.destroy_process_group()
