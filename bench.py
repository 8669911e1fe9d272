"""Benchmark: swapped GPT-3 training step on B200 peers (Atom, arXiv 2403.10504).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config xl] [--impl atom|reference]

One process per GPU (torchrun for N > 1).  Every rank is a peer holding a whole-model replica
in pinned host memory; sub-models are swapped through a capped model-state budget (the paper's
sub-model "GPU capacity") and peers average parameters every K_sync steps.
Rank 0 prints ONE JSON line.  Timing: W warm-up steps, then K timed steps bracketed by a
barrier + device synchronize, CUDA events, max over ranks.  Inputs: synthetic tokens
(PCG64, uniform over the vocabulary); init drawn on the device (minGPT law).

--impl reference times the CPU oracle (oracle/, fp64 numpy) as it stands on this host, on a
bounded sample of the same workload (see cpu_sample()).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "train tokens/s per B200 (swapped GPT-3), swap-hidden %, at 1/2/4/8 peers"
UNIT = "tokens/s"
# measured on this pool's B200 box (profiles/box_probe_r01.json): pinned copies, 1 GiB
H2D_GBS, D2H_GBS, BIDIR_GBS = 55.5, 57.2, 49.7


def attention_roofline(g, tok_step, klog, peak_tf):
    f_fwd = tok_step * 2.0 * g.n_layer * g.d_model * (g.seq_len + 1)
    out = {"bound": "tensor", "unit": "TFLOP/s", "peak": peak_tf,
           "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernels timed inside the step)"}
    for k, f in (("attn_fwd", f_fwd), ("attn_bwd", 2.0 * f_fwd)):
        ms = klog.get(k, (0, 0.0))[1]
        tf = f / (ms / 1000.0) / 1e12 if ms > 0 else None
        out[k] = {"flops_per_step": f, "ms_per_step": ms, "achieved": tf, "frac": tf / peak_tf if tf else None}
    return out


def attention_standalone(g, device, burst_tf):
    """The step's attention kernels timed alone at one micro-batch's shape (b, T, h, d_h): the
    persistent forward and the dS^T backward (dK/dV + dQ + D), CUDA events on the launching stream,
    against the burst peak (a kernel timed alone)."""
    import torch
    from paper_2403_10504_b200 import atom
    b, T, h, d = g.micro_batch, g.seq_len, g.n_head, g.d_model
    dh = d // h
    gen = torch.Generator(device=device).manual_seed(5)
    qkv = (torch.randn(b * T, 3 * d, generator=gen, device=device) * 0.5).bfloat16()
    o = torch.empty(b * T, d, device=device, dtype=torch.bfloat16)
    dout = torch.randn(b * T, d, generator=gen, device=device).bfloat16()
    lse = torch.empty(b * h * T, device=device)
    dsum = torch.empty(b * h * T, device=device)
    dqkv = torch.empty_like(qkv)
    st = torch.cuda.current_stream(device).cuda_stream
    f_fwd = 4.0 * b * h * dh * T * (T + 1) / 2
    fwd = lambda: atom.k_attn_fwd(atom.ATTN_TC, atom.BF16, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), b, T, h,
                                  dh, stream=st)
    bwd = lambda: atom.k_attn_bwd(atom.ATTN_TC_DS, atom.BF16, qkv.data_ptr(), o.data_ptr(), dout.data_ptr(),
                                  lse.data_ptr(), dsum.data_ptr(), dqkv.data_ptr(), b, T, h, dh, stream=st)
    out = {"shape": {"b": b, "T": T, "h": h, "d_h": dh}, "unit": "TFLOP/s", "peak": burst_tf,
           "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst: kernels timed alone)"}
    for name, fn, f in (("fwd", fwd, f_fwd), ("bwd", bwd, 2.0 * f_fwd)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(device)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize(device)
        us = e0.elapsed_time(e1) / 10 * 1000.0
        tf = f / (us * 1e-6) / 1e12
        out[name] = {"us": us, "achieved": tf, "frac": tf / burst_tf}
    del qkv, o, dout, lse, dsum, dqkv
    return out


def plan_with_fallback(atom, cfg, hbm_budget, link_bw, notes):
    """atom_plan; when no plan both fits and hides the swap at C <= 32 (a slow shared host link, e.g.
    many peers on one socket), allow C up to 64, and past that drop the compute >= load condition
    (the swap is then only partly hidden): the bench still measures the step it can run."""
    try:
        return atom.atom_plan(cfg, hbm_budget, link_bw)
    except atom.AtomError as ex:
        notes.append(f"C <= {cfg.max_C}: {str(ex)[:120]}")
    cfg.max_C = 64
    try:
        plan = atom.atom_plan(cfg, hbm_budget, link_bw)
        notes.append("planned with C <= 64")
        return plan
    except atom.AtomError as ex:
        notes.append(f"C <= 64: {str(ex)[:120]}")
    cfg.max_C, cfg.overlap_check = 32, 0
    notes.append("planned without the compute >= load condition (swap partly exposed)")
    return atom.atom_plan(cfg, hbm_budget, link_bw)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "fallback": True}


WORKLOADS = {
    # name: (config, model-state cap bytes, description)
    "xl": ("xl", 10 * 2 ** 30, "GPT-3 XL 1.3B (24L, d=2048, 16x128 heads, T=2048, b=8), model state capped at 10 GiB"),
    "2.7b": ("2.7b", 20 * 2 ** 30, "GPT-3 2.7B (32L, d=2560, 32x80 heads, T=2048, b=8), model state capped at "
             "20 GiB (resident would need 50 GB); sub-models, C and the activation policy planned from a "
             "profiled compute rate"),
    "13b": ("13b", 0, "GPT-3 13B (40L, d=5120, 40x128 heads, T=2048, b=4): weights and AdamW state host-resident "
            "(236 GB of device state would be needed), swapped per sub-model through the whole HBM"),
    "small": ("small", 0, "GPT-3 Small 125M (12L, d=768, 12x64 heads, T=2048, b=8) swapped one layer per sub-model "
              "(forced partition, C=8, overlap check off: at 49.7 GB/s no hidden plan exists below the resident "
              "one -- Small's compute per layer is too short to cover its load, the case P:295 describes)"),
    "tiny": ("tiny", 3 * 10 ** 6, "tiny GPT (4L, d=64, T=32, V=256)"),
}


# workloads with a fixed partition instead of the planner's (cfg overrides)
FORCED = {"small": {"forced_ends": list(range(14)), "C_": 8, "overlap_check": 0}}


def host_mem_available():
    """Bytes this process may still pin: MemAvailable, capped by the cgroup limit when one is set."""
    avail = None
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                avail = int(ln.split()[1]) * 1024
    except OSError:
        pass
    try:
        lim = open("/sys/fs/cgroup/memory.max").read().strip()
        if lim != "max":
            used = int(open("/sys/fs/cgroup/memory.current").read())
            avail = min(avail or 1 << 62, int(lim) - used)
    except (OSError, ValueError):
        pass
    return avail


def bind_to_gpu_numa(local):
    """Run this rank on the CPUs NVML reports as local to its GPU, so the pinned host arenas are
    first-touched on that NUMA node (8 peers over two sockets would otherwise share one memory
    controller). No-op when NVML or the affinity call is unavailable."""
    try:
        import pynvml
        import torch
        pr = torch.cuda.get_device_properties(local)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        pass
    return None


def link_probe(local, world, nbytes=2 << 30, reps=3, rounds=3):
    """Pinned host<->device rate per direction when every rank copies both ways at once (the
    backward phase's traffic): host DRAM, not PCIe, is what several peers share (4 GPUs of one
    socket: ~22 GB/s each way per GPU vs 49.7 alone, tools/host_bw_probe.py). Min over ranks."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    rates = []
    for _ in range(rounds):
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            torch.cuda.synchronize()
        t = time.perf_counter()
        with torch.cuda.stream(s1):
            for _ in range(reps):
                d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            for _ in range(reps):
                h2.copy_(d2, non_blocking=True)
        torch.cuda.synchronize()
        rates.append(reps * nbytes / (time.perf_counter() - t))
    rate = statistics.median(rates)   # one slow round (page faults, a neighbour's burst) is not the link
    del h, h2, d, d2
    torch.cuda.empty_cache()
    if world > 1:
        import torch.distributed as dist
        r = torch.tensor([rate], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(r, op=dist.ReduceOp.MIN)
        rate = float(r.item())
    return rate


def f_alg_per_token(g):
    """Algorithmic FLOPs per token: 6(12 L d^2 + d V) + 6 L d (T+1) (causal half)."""
    L, d, V, T = g.n_layer, g.d_model, g.vocab, g.seq_len
    return 6 * (12 * L * d * d + d * V) + 6 * L * d * (T + 1)


class Clocks:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu):
        self.gpu, self.proc, self.lines = gpu, None, []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(g, seconds_hint=20.0, max_steps=3):
    """Time the oracle (fwd + hand bwd + AdamW) in fp32 on one
    sequence of the workload through a layer-reduced copy of the model (L = 2, same d, h, T, V)
    and extrapolate to the full depth by algorithmic FLOPs.  Returns (tokens/s at full depth,
    sample description, cores, wall seconds per timed sample step)."""
    from oracle import adamw as oadamw
    from oracle import gpt as ogpt
    L = min(2, g.n_layer)
    g1 = synth.GPTConfig(g.name + f"-L{L}", L, g.d_model, g.n_head, g.seq_len, g.vocab, 1)
    p = synth.init_params(g1, seed=1, dtype=np.float32)
    toks = synth.tokens(g1, 1, 5)
    h = oadamw.AdamWHyper()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    # BLAS on every host core (torchrun sets OMP_NUM_THREADS=1 for its ranks): the reported core
    # count is the thread count the sample really used
    cores = os.cpu_count()
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        limiter = threadpool_limits(limits=cores)
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        limiter = None
    t0 = time.perf_counter()
    n = 0
    while True:
        loss, grad = ogpt.loss_and_grad(g1, p, toks, dtype=np.float32)
        p, m, v = oadamw.adamw_step(h, n + 1, p, grad, m, v, dtype=np.float32)
        n += 1
        if time.perf_counter() - t0 > seconds_hint or n >= max_steps:
            break
    dt = (time.perf_counter() - t0) / n
    if limiter is not None:
        limiter.unregister()
    rate_sample = g.seq_len / dt
    rate = rate_sample * f_alg_per_token(g1) / f_alg_per_token(g)
    desc = (f"oracle fp32 numpy fwd+bwd+AdamW on 1 sequence (T={g.seq_len}) of a {L}-block copy of the model "
            f"(d={g.d_model}, V={g.vocab}); {n} step(s), {dt:.1f} s each; tokens/s scaled to L={g.n_layer} by "
            f"algorithmic FLOPs per token")
    return rate, desc, cores, dt


def run_reference(args, g, wl_desc):
    """--impl reference: the oracle timed on this host (rank 0 only).  A step = one timed sample
    (one sequence through the L = 2 copy, fp32); ms_per_step is that sample's wall time, value the
    full-depth tokens/s it extrapolates to."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rates, walls = [], []
    for i in range(args.warmup + args.steps):
        r, desc, cores, dt = cpu_sample(g, seconds_hint=0.0, max_steps=1)
        if i >= args.warmup:
            rates.append(r)
            walls.append(dt)
    val = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.mean(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl_desc, "model": g.name, "seq_len": g.seq_len, "sample_tokens_per_step": g.seq_len,
                       "sample": "each step = one sequence through an L=2 copy of the model (fp32 oracle); "
                                 "value = the full-depth tokens/s it extrapolates to by algorithmic FLOPs"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


GEMM_NCU = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_gemm_shapes_ncu.json")


def gemm_traffic():
    """DRAM bytes per GEMM launch from the committed `ncu --set full` captures of the twelve 2.7B
    block GEMM shapes (forward, data gradient, weight gradient of QKV, projection, fc, fc2; one
    launch each, cold L2: tools/runs/gpu_r2_51.sh), averaged like `achieved` over the step's GEMM
    mix (each shape once per block and micro-batch), next to their algorithmic bytes (A + B + C)."""
    try:
        with open(GEMM_NCU) as f:
            caps = json.load(f)
    except OSError:
        return {"traffic": None}
    per = [c["dram_read"] + c["dram_write"] for c in caps]
    alg = [c["algorithmic_bytes"] for c in caps]
    return {"traffic": sum(per) / len(per),
            "traffic_detail": {"shapes": [c["shape"] for c in caps], "dram_bytes": per, "algorithmic_bytes": alg,
                               "mean_over_algorithmic": sum(per) / sum(alg),
                               "tensor_pipe_pct": [round(c["tensor_pipe_pct"], 1) for c in caps],
                               "source": os.path.relpath(GEMM_NCU, os.path.dirname(os.path.abspath(__file__)))}}


def host_link(st, plan, probe_gbs):
    h2d, d2h = st["h2d_ms"], st["d2h_ms"]   # summed copy-op time per lane, last step (atom_get_stats)
    return {"h2d_op_GBs": plan.pred_h2d_B / h2d / 1e6 if h2d > 0 else None,
            "d2h_op_GBs": plan.pred_d2h_B / d2h / 1e6 if d2h > 0 else None,
            "probe_bidir_GBs": probe_gbs, "solo_h2d_GBs": H2D_GBS, "solo_d2h_GBs": D2H_GBS}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--no-attn-standalone", action="store_true",
                    help="skip the attention kernels' standalone timing (attention_roofline.standalone)")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="2.7b", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="atom", choices=["atom", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--link-gbs", type=float, default=0.0,
                    help="host-link GB/s per direction the planner assumes (default: measured, all ranks at once)")
    ap.add_argument("--trace-out", default="", help="write the last step's per-op trace here (rank 0)")
    ap.add_argument("--planner-tflops", type=float, default=0.0,
                    help="compute rate the planner's cost model assumes (default: measured by a profile run)")
    ap.add_argument("--grad-rounds", type=int, default=0,
                    help="host update placement (P:563 CPU AdamW): gradient rounds per update (0 = GPU AdamW every step)")
    ap.add_argument("--op-nodes", action="store_true",
                    help="operator-granular graph: sub-models may end between a block's attention and MLP halves "
                         "(P:332; DESIGN.md R40)")
    ap.add_argument("--dropout", type=float, default=0.0, help="minGPT dropout p at every site (DESIGN.md R38)")
    ap.add_argument("--no-profile", action="store_true",
                    help="plan with the measured bf16 peak instead of a profiled compute rate")
    args = ap.parse_args()
    cfg_name, state_cap, wl_desc = WORKLOADS[args.config]
    g = synth.CONFIGS[cfg_name]
    if args.impl == "reference":
        return run_reference(args, g, wl_desc)

    import torch
    from paper_2403_10504_b200 import atom
    from paper_2403_10504_b200 import dist as adist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    numa_cpus = bind_to_gpu_numa(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # every peer pins 12 B/param (fp32 master, m, v): refuse up front rather than drive the
    # host out of memory (all local ranks check before any of them pins)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    need = local_world * (12 * synth.n_params(g) + 4 * 2 ** 30)
    avail = host_mem_available()
    if avail is not None and need > avail:
        raise SystemExit(f"bench: {local_world} peer(s) of {g.name} need {need / 1e9:.1f} GB of pinned host memory, "
                         f"{avail / 1e9:.1f} GB available")
    if args.link_gbs <= 0:
        args.link_gbs = link_probe(local, world) / 1e9
    pk = peaks()
    free, total = torch.cuda.mem_get_info()
    hbm_budget = int(free - 6 * 2 ** 30)
    # peer averaging cadence from a global batch of 512 sequences (reading R17)
    plan_tf = args.planner_tflops or pk["bf16_tflops"]
    forced = FORCED.get(args.config, {})
    extra = dict(op_nodes=int(args.op_nodes), dropout_p=args.dropout, dropout_seed=7)
    # the profile run always uses the block graph (its plan may need the re-forward, which the
    # half-block graph does not offer, R40); --op-nodes re-plans the half-block graph afterwards
    first = dict(extra, op_nodes=0) if not args.planner_tflops and not args.no_profile and not forced else extra
    cfg = atom.make_cfg(g, dtype=atom.BF16, max_C=32, peak_flops=int(plan_tf * 1e12),
                        state_budget=state_cap, lr=1e-4, warmup_steps=3000, grad_rounds=args.grad_rounds, **forced,
                        **first)
    plan_notes = []
    plan = plan_with_fallback(atom, cfg, hbm_budget, int(args.link_gbs * 1e9), plan_notes)
    profiled = None
    if not args.planner_tflops and not args.no_profile and not forced:
        # measured profile -> plan (R34): run the first plan for a few
        # steps, measure the compute rate it sustains, re-plan with that rate (min over ranks so
        # every peer gets the same plan)
        from paper_2403_10504_b200 import profile as aprof
        toks0 = [torch.tensor(synth.tokens(g, plan.C * g.micro_batch, synth.step_seed(rank, 10 ** 6 + s)),
                              device=f"cuda:{local}") for s in range(2)]
        m = aprof.measure(cfg, plan, toks0, device=local, steps=3)
        del toks0
        rates = [m["flops"], m["h2d"] or args.link_gbs * 1e9, m["d2h"] or args.link_gbs * 1e9]
        if world > 1:
            import torch.distributed as dist
            r = torch.tensor(rates, dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(r, op=dist.ReduceOp.MIN)
            rates = [float(x) for x in r.tolist()]
        table = m["cost_table"]
        if world > 1 and table:   # the slowest rank's per-node times (max), so all plans agree
            import torch.distributed as dist
            t = torch.tensor(table, dtype=torch.int64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            table = [int(x) for x in t.tolist()]
        profiled = {"first_plan": {"C": plan.C, "act_policy": plan.act_policy, "n_recompute": plan.n_recompute,
                                   "sub_models": plan.ends()},
                    "measured_tflops": rates[0] / 1e12, "measured_h2d_GBs": rates[1] / 1e9,
                    "measured_d2h_GBs": rates[2] / 1e9,
                    "cost_table_ms": ({"block_fwd": table[2] / 1e6, "block_bwd": table[3] / 1e6,
                                       "head_fwd": table[-2] / 1e6, "head_bwd": table[-1] / 1e6,
                                       "embed_fwd": table[0] / 1e6, "embed_bwd": table[1] / 1e6}
                                      if table else None)}
        plan_tf = rates[0] / 1e12
        link_bw = int(min(rates[1], args.link_gbs * 1e9))
        # the measured per-block cost table fits the block graph; the half-block graph plans with the
        # measured rates (R40)
        cfg = atom.make_cfg(g, dtype=atom.BF16, max_C=32, peak_flops=int(rates[0]), state_budget=state_cap,
                            lr=1e-4, warmup_steps=3000, cost_table=(table or None) if not args.op_nodes else None,
                            d2h_bw=int(min(rates[2], args.link_gbs * 1e9)), grad_rounds=args.grad_rounds, **extra)
        plan = plan_with_fallback(atom, cfg, hbm_budget, link_bw, plan_notes)
    tok_step = plan.C * g.micro_batch * g.seq_len
    cfg.sync_every = adist.sync_every(world, plan.C, g.micro_batch)     # global batch 512
    nccl_id = adist.bootstrap_nccl_id(atom.atom_nccl_unique_id) if world > 1 else None
    peer = atom.Peer(cfg, plan, device=local, init_params=None, seed=1234, nccl_id=nccl_id, nranks=world, rank=rank)
    n_seq = plan.C * g.micro_batch
    host_batches = [synth.tokens(g, n_seq, synth.step_seed(rank, s)) for s in range(args.warmup + 2 * args.steps)]
    dev_batches = [torch.tensor(b, device=f"cuda:{local}") for b in host_batches]

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            torch.cuda.synchronize()

    if world > 1:
        # the first warm-up step averages too: NCCL sets up its connections on a communicator's
        # first collective (hundreds of ms), which must not land in a timed step
        atom.atom_sync([peer], flush=False)
    for i in range(args.warmup):
        peer.step_device(dev_batches[i])
    barrier()

    def timed(fn, batches):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        losses = [fn(b) for b in batches]
        torch.cuda.synchronize()   # the step's tail runs on the library's streams: device-wide sync
        e1.record()
        torch.cuda.synchronize()
        ms = adist.max_over_ranks(e0.elapsed_time(e1), device=f"cuda:{local}")
        return ms, losses

    # value: inputs resident in HBM; per-GEMM CUDA events on the library's compute stream
    peer.reset_stats(timing=int(os.environ.get("ATOM_BENCH_TIMING", "1")))
    with Clocks(local) as clk:
        ms, losses = timed(peer.step_device, dev_batches[args.warmup:args.warmup + args.steps])
    st = peer.stats()
    gemm_shapes = sorted(peer.gemm_log(), key=lambda r: -r["ms"])
    # e2e: host tokens through atom_step (pinned staging + H2D in the step), loss read back
    ms_e2e, _ = timed(peer.step, host_batches[args.warmup + args.steps:])
    # per kernel category: one more step, outside both timed regions, with events around every
    # launch group (they cost ~8 % of a step, so never inside a timed one)
    peer.reset_stats(timing=2)
    peer.step_device(dev_batches[0])
    klog = peer.kernel_log()
    attn_alone = None
    if rank == 0 and not args.no_attn_standalone:
        try:
            attn_alone = attention_standalone(g, f"cuda:{local}", pk["bf16_tflops"])
        except Exception as ex:  # noqa: BLE001 -- a report field, never a reason to lose the line
            attn_alone = {"error": f"{type(ex).__name__}: {ex}"[:200]}
    value = world * args.steps * tok_step / (ms / 1000.0)
    e2e = world * args.steps * tok_step / (ms_e2e / 1000.0)

    gemm_tf = st["gemm_flops"] / (st["gemm_ms"] / 1000.0) / 1e12 if st["gemm_ms"] > 0 else None
    peak_tf = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    ms_step = ms / args.steps
    # the slower of the FLOPs at tensor peak and the plan's swapped bytes over the host link (per
    # direction, the link alone): ~14 N in / 12 N out with the GPU AdamW (less the resident
    # sub-model 1), 12 N / 4 N with host gradient sums (--grad-rounds)
    def t_roof_at(tflops):   # ms
        return 1000.0 * max(tok_step * f_alg_per_token(g) / (tflops * 1e12),
                            plan.pred_h2d_B / (H2D_GBS * 1e9), plan.pred_d2h_B / (D2H_GBS * 1e9))

    t_roof = t_roof_at(pk["bf16_tflops"]) / 1000.0
    trace = peer.trace()
    if rank == 0 and args.trace_out:
        with open(args.trace_out, "w") as f:
            f.write(trace)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            r, desc, cores, _ = cpu_sample(g)
            cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": wl_desc, "model": g.name, "global_batch": world * n_seq, "seq_len": g.seq_len,
                       "micro_batch": g.micro_batch, "C": plan.C, "sub_models": plan.ends(),
                       "graph": ("operator-granular (node 2l+1 = attention half, 2l+2 = MLP half of block l)"
                                 if args.op_nodes else "block nodes"),
                       "mid_block_cuts": ([e for e in plan.ends()[:-1] if e % 2 == 1] if args.op_nodes else []),
                       "dropout_p": args.dropout,
                       "act_policy": {0: "auto", 1: "stash", 2: "recompute", 3: "hybrid"}.get(plan.act_policy),
                       "n_recompute": plan.n_recompute,
                       "planner_tflops": plan_tf, "profile": profiled,
                       "state_budget_bytes": state_cap, "device_arena_bytes": plan.device_bytes,
                       "plan_fallback": plan_notes or None,
                       "parallelism": f"peers{world}", "sync_every": cfg.sync_every,
                       "update": (f"host: CPU AdamW every {args.grad_rounds} gradient rounds (a step = one round)"
                                  if args.grad_rounds else "GPU AdamW on every swapped-in sub-model, every step"),
                       "link_GBs_bidir_probe": args.link_gbs, "numa_cpus": numa_cpus,
                       "l2": "inputs larger than L2 (weights/activations stream through HBM every step)"},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 4 * n_seq * (g.seq_len + 1),
                    "d2h_bytes_per_step": 4},
            # value is the whole-job aggregate over all peers (the bench contract); per B200 here
            "value_per_gpu": value / world,
            "gpu_launches": st["kernel_launches"],
            "roofline": {"bound": "tensor", "kernel": "gemm_tc2_kernel (tcgen05, 2-CTA 256x256 tiles; all GEMM launches of the timed steps)", "achieved": gemm_tf,
                         "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": (gemm_tf / peak_tf) if gemm_tf else None, **gemm_traffic(),
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                         "gemm_share_of_step": st["gemm_ms"] / ms if ms else None,
                         "by_shape": [[r["M"], r["N"], r["K"], r["a_mn"], r["b_mn"], r["epilogue"], r["launches"],
                                       round(r["ms"], 2), round(r["tflops"], 1)] for r in gemm_shapes],
                         "by_shape_fields": "M N K a_mn b_mn epilogue launches ms TFLOP/s"},
            "step_roofline": {"t_roof_ms": t_roof * 1000.0, "frac": t_roof * 1000.0 / ms_step,
                              "peak_tflops": pk["bf16_tflops"], "peak": "MEASURED_PEAKS.json bf16_tflops (burst)",
                              # the same step against the sustained measured peak and the datasheet
                              "frac_vs_sustained": t_roof_at(pk.get("bf16_tflops_sustained", pk["bf16_tflops"])) / ms_step,
                              "frac_vs_datasheet_2250": t_roof_at(2250.0) / ms_step,
                              "flops_per_token": f_alg_per_token(g),
                              # the same bound with the host link as all ranks see it at once
                              # (link_probe: host DRAM shared by the peers of one socket)
                              "t_roof_contended_ms": 1000.0 * max(t_roof, plan.pred_d2h_B / (args.link_gbs * 1e9)),
                              "frac_contended": 1000.0 * max(t_roof, plan.pred_d2h_B / (args.link_gbs * 1e9)) / ms_step},
            # device time per kernel category in one extra (untimed) step: CUDA events around each
            # launch group on its stream (the side streams overlap the main one: the sum exceeds the step)
            "kernel_ms_per_step": {k: round(v[1], 2) for k, v in klog.items()},
            # the attention kernels (the furthest below peak): algorithmic FLOPs of one step's causal
            # attention, forward 2 L d (T + 1) per token and backward twice that (its recomputed S is
            # not counted), over the same per-category event times (concurrent streams: an upper
            # bound on the kernels' time, so a lower bound on their rate)
            "attention_roofline": {**attention_roofline(g, tok_step, klog, peak_tf),
                                   "standalone": attn_alone},
            "swap_hidden_pct": (100.0 * st["copy_hidden_ms"] / st["copy_ms"]) if st["copy_ms"] else None,
            "swap_hidden": {"h2d_pct": 100.0 * st["h2d_hidden_ms"] / st["h2d_ms"] if st["h2d_ms"] else None,
                            "d2h_pct": 100.0 * st["d2h_hidden_ms"] / st["d2h_ms"] if st["d2h_ms"] else None,
                            "combined_pct": (100.0 * st["copy_hidden_ms"] / st["copy_ms"]) if st["copy_ms"] else None,
                            "h2d_ms": st["h2d_ms"], "d2h_ms": st["d2h_ms"],
                            "of": "last timed step: copy time overlapping compute-lane FWD/BWD ops (per-op CUDA events)"},
            "compute_busy_pct": (100.0 * st["compute_busy_ms"] / st["compute_span_ms"]) if st["compute_span_ms"] else None,
            "host_issue_ms_per_step": st["host_issue_ms"],
            "hbm_arena": {"total_bytes": plan.device_bytes, "resident_submodel1_bytes": plan.r1_bytes,
                          "slots_bytes": plan.nslot * plan.slot_bytes, "nslot": plan.nslot,
                          "stash_bytes": plan.stash_bytes, "work_bytes": plan.work_bytes},
            "h2d_GBs": st["h2d_bytes"] / (ms / 1000.0) / 1e9, "d2h_GBs": st["d2h_bytes"] / (ms / 1000.0) / 1e9,
            # while a copy runs (planned bytes of the last step / busy time of its copy lane) vs the
            # link as every rank sees it at once (link_probe) and alone (profiles/box_probe_r01.json)
            "host_link": host_link(st, plan, args.link_gbs),
            "loss_first_last": [losses[0], losses[-1]],
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    peer.destroy()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
