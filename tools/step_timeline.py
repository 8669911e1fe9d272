"""One 2.7B training step under torch.profiler (CUPTI: every kernel and runtime call in the process,
libatom's included) -> per-stream busy / gap accounting and the top kernels by device time; the
host side: time spent in CUDA runtime calls during the step.  Usage:
    python tools/step_timeline.py [--config 2.7b] [--out gpurun_out/timeline.json]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2403_10504_b200 import atom  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2.7b")
    ap.add_argument("--out", default="gpurun_out/timeline_trace.json")
    ap.add_argument("--tflops", type=float, default=960.0)
    ap.add_argument("--link-gbs", type=float, default=49.7)
    a = ap.parse_args()
    g = synth.CONFIGS[a.config]
    free, _ = torch.cuda.mem_get_info()
    cfg = atom.make_cfg(g, dtype=atom.BF16, max_C=32, peak_flops=int(a.tflops * 1e12), state_budget=20 * 2 ** 30,
                        lr=1e-4, warmup_steps=3000)
    plan = atom.atom_plan(cfg, int(free - 6 * 2 ** 30), int(a.link_gbs * 1e9))
    peer = atom.Peer(cfg, plan, device=0, init_params=None, seed=1234)
    toks = [torch.tensor(synth.tokens(g, plan.C * g.micro_batch, synth.step_seed(0, s)), device="cuda")
            for s in range(4)]
    for s in range(3):
        peer.step_device(toks[s])
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        peer.step_device(toks[3])
        torch.cuda.synchronize()
    prof.export_chrome_trace(a.out)
    peer.destroy()
    ev = json.load(open(a.out))["traceEvents"]
    kern = [e for e in ev if e.get("cat") == "kernel"]
    mem = [e for e in ev if e.get("cat") in ("gpu_memcpy", "gpu_memset")]
    rt = [e for e in ev if e.get("cat") == "cuda_runtime"]
    by_stream = collections.defaultdict(list)
    for e in kern:
        by_stream[e["args"].get("stream", e.get("tid"))].append((e["ts"], e["ts"] + e["dur"]))
    t0 = min(e["ts"] for e in kern)
    t1 = max(e["ts"] + e["dur"] for e in kern)
    print(f"plan C={plan.C} S={plan.n_seg}; step span (first kernel -> last kernel) {(t1 - t0) / 1000:.1f} ms, "
          f"{len(kern)} kernels, {len(mem)} copies/memsets")
    allk = sorted((s, e) for v in by_stream.values() for s, e in v)
    busy, cs, ce = 0.0, None, None
    for s, e in allk:
        if ce is None or s > ce:
            if ce is not None:
                busy += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    busy += ce - cs
    print(f"any-kernel-running {busy / 1000:.1f} ms ({100 * busy / (t1 - t0):.1f} % of the span)")
    for st, iv in sorted(by_stream.items(), key=lambda kv: -sum(e - s for s, e in kv[1])):
        iv.sort()
        tot = sum(e - s for s, e in iv)
        gaps = [iv[i + 1][0] - iv[i][1] for i in range(len(iv) - 1)]
        small = sum(g for g in gaps if 0 < g < 100)
        print(f"stream {st}: {len(iv)} kernels, {tot / 1000:.1f} ms busy; gaps < 100 us: {small / 1000:.1f} ms "
              f"over {sum(1 for g in gaps if 0 < g < 100)} gaps; median gap {sorted(gaps)[len(gaps) // 2] if gaps else 0:.1f} us")
    names = collections.Counter()
    cnt = collections.Counter()
    for e in kern:
        n = e["name"].split("(")[0][:70]
        names[n] += e["dur"]
        cnt[n] += 1
    print("top kernels (ms, launches, mean us):")
    for n, d in names.most_common(25):
        print(f"  {d / 1000:9.2f} {cnt[n]:6d} {d / cnt[n]:9.1f}  {n}")
    rtn = collections.Counter()
    rtc = collections.Counter()
    for e in rt:
        rtn[e["name"]] += e["dur"]
        rtc[e["name"]] += 1
    print(f"host: {sum(rtn.values()) / 1000:.1f} ms in CUDA runtime calls during the step:")
    for n, d in rtn.most_common(12):
        print(f"  {d / 1000:9.2f} ms {rtc[n]:6d} calls {d / rtc[n]:7.2f} us  {n}")


if __name__ == "__main__":
    main()
