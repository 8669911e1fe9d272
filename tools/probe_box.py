"""Probe the GPU box: host, topology, pinned host<->device bandwidth (alone and bidirectional)."""
import json, os, subprocess, sys, time
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {"lscpu": sh("lscpu | head -20"), "free": sh("free -g"), "topo": sh("nvidia-smi topo -m"),
       "smi": sh("nvidia-smi --query-gpu=index,name,memory.total,pcie.link.gen.max,pcie.link.width.max,clocks.max.sm --format=csv"),
       "nproc": os.cpu_count()}
free, total = torch.cuda.mem_get_info()
out["mem_get_info"] = [free, total]
def bw(nbytes, reps=5):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps): fn()
        torch.cuda.synchronize()
        res[name] = nbytes * reps / (time.perf_counter() - t) / 1e9
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res["bidir_each"] = nbytes * reps / (time.perf_counter() - t) / 1e9
    return res
out["pinned_bw_GBs"] = {str(n >> 20) + "MiB": bw(n) for n in (64 << 20, 256 << 20, 1 << 30)}
t = time.perf_counter(); x = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True); out["pin_8GiB_s"] = time.perf_counter() - t
print(json.dumps(out, indent=1))
