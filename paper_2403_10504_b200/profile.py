"""Measured profile feeding the planner ("the model is profiled
offline", "We empirically determine C offline via profiling for a particular GPU").

The planner's cost table is analytic (FLOPs / rate, bytes / link). Profiling here measures the
one number that table needs from this GPU and these kernels: the compute rate the step actually
sustains, i.e. the FLOPs a step executes (including a re-forward, if the plan has one) divided by
the busy time of the compute stream, taken from the library's per-op CUDA-event trace of a few
steps run with a first plan. The plan is then recomputed with that rate (R34).
"""
from . import atom


def compute_busy_ms(trace: str) -> float:
    """Union of the compute-lane intervals of a step trace (atom_get_trace), in ms."""
    iv = sorted((float(f[5]), float(f[6])) for f in (l.split() for l in trace.splitlines())
                if len(f) >= 7 and f[0] == "compute")
    busy, cur_s, cur_e = 0.0, None, None
    for a, b in iv:
        if cur_e is None or a > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    if cur_e is not None:
        busy += cur_e - cur_s
    return busy / 1000.0


def compute_span_ms(trace: str) -> float:
    """First compute-lane op start -> last compute-lane op end, in ms."""
    iv = [(float(f[5]), float(f[6])) for f in (l.split() for l in trace.splitlines())
          if len(f) >= 7 and f[0] == "compute"]
    return (max(b for _, b in iv) - min(a for a, _ in iv)) / 1000.0 if iv else 0.0


def executed_flops(g, plan) -> float:
    """FLOPs one step executes: 6 N-style model FLOPs per token (plan.pred_flops) plus the
    re-forward of the plan's n_recompute blocks (R28, R35: the QKV,
    attention-projection and fc GEMMs, 16 d^2 per token, and the attention forward,
    2 d (T + 1) per token)."""
    d, T = g.d_model, g.seq_len
    tokens = plan.C * g.micro_batch * T
    return float(plan.pred_flops) + plan.n_recompute * tokens * (16.0 * d * d + 2.0 * d * (T + 1))


def lane_ms(trace: str, lane: str) -> float:
    """Summed op durations of one lane (copies do not overlap within a lane), in ms."""
    return sum(float(f[6]) - float(f[5]) for f in (l.split() for l in trace.splitlines())
               if len(f) >= 7 and f[0] == lane) / 1000.0


def op_means_us(trace: str, lane: str = "compute") -> dict:
    """Mean duration (us) of each (KIND, segment) op of one lane over its micro-batches."""
    acc = {}
    for f in (l.split() for l in trace.splitlines()):
        if len(f) >= 7 and f[0] == lane:
            key = (f[1], int(f[2]))
            n, t = acc.get(key, (0, 0.0))
            acc[key] = (n + 1, t + float(f[6]) - float(f[5]))
    return {k: t / n for k, (n, t) in acc.items()}


def cost_table_from_trace(trace: str, plan, n_layer: int) -> list:
    """Per-node {t_f_ns, t_b_ns} (one micro-batch) for atom_model_cfg.cost_table, from the traced
    FWD / BWD op of every segment (execution time per layer, profiled).

    Node order E, B_0..B_{L-1}, H. Blocks share one cost: the blocks-only segments' times divided
    by their block counts (the backward without the re-forwards of the plan's n_recompute blocks,
    which the planner adds back, R28, R35). E and H get what is left of their segments: FWD(1) / BWD(1)
    minus its blocks; FWD(S) carries the head's forward and backward (run back to back per
    micro-batch), split 1 : 2 as their FLOPs are. Returns [] when no segment holds only
    blocks (the caller falls back to the single measured rate)."""
    ops = op_means_us(trace)
    ends = plan.ends()
    S, L = len(ends), n_layer
    lo = [0] + [e + 1 for e in ends[:-1]]
    nblk = [sum(1 for v in range(lo[k], ends[k] + 1) if 1 <= v <= L) for k in range(S)]
    # re-forwarded blocks per segment: blocks 1..n_recompute
    nrc = [sum(1 for v in range(lo[k], ends[k] + 1) if 1 <= v <= plan.n_recompute) if k < S - 1 else 0
           for k in range(S)]
    mids = [k for k in range(S) if all(1 <= v <= L for v in range(lo[k], ends[k] + 1))
            and ("FWD", k + 1) in ops and ("BWD", k + 1) in ops and k < S - 1]
    if not mids:
        return []
    nb = sum(nblk[k] for k in mids)
    tf_b = sum(ops[("FWD", k + 1)] for k in mids) / nb
    tb_b = (sum(ops[("BWD", k + 1)] for k in mids) - tf_b * sum(nrc[k] for k in mids)) / nb
    tf_e = max(ops.get(("FWD", 1), 0.0) - nblk[0] * tf_b, 0.0) if lo[0] == 0 else 0.0
    tb_e = max(ops.get(("BWD", 1), 0.0) - nblk[0] * tb_b - nrc[0] * tf_b, 0.0)
    head = max(ops.get(("FWD", S), 0.0) - nblk[S - 1] * tf_b, 0.0)
    ns = lambda us: max(int(round(us * 1000.0)), 1)
    table = [ns(tf_e), ns(tb_e)]
    for _ in range(L):
        table += [ns(tf_b), ns(tb_b)]
    table += [ns(head / 3.0), ns(2.0 * head / 3.0)]
    return table


def measure(cfg, plan, tokens_dev, device: int = 0, steps: int = 3) -> dict:
    """Profile `plan` on this GPU: run `steps` steps on device tokens and read the last step's
    trace. Returns the sustained compute rate (FLOPs executed / compute-lane busy time) and the
    achieved host->device and device->host copy rates (planned bytes / copy-lane busy time): the
    per-layer execution and loading times of P:329 folded into the cost model's two rates."""
    peer = atom.Peer(cfg, plan, device=device, init_params=None, seed=1234)
    try:
        for s in range(steps):
            peer.step_device(tokens_dev[s % len(tokens_dev)])
        tr = peer.trace()
    finally:
        import torch
        peer.destroy()
        peer.arena = None          # hand the arena back to the driver before the real plan allocates
        torch.cuda.empty_cache()
    busy = compute_busy_ms(tr)
    h2d, d2h = lane_ms(tr, "h2d"), lane_ms(tr, "d2h")
    return {"flops": executed_flops(cfg, plan) / (busy / 1000.0),
            "h2d": plan.pred_h2d_B / (h2d / 1000.0) if h2d > 0 else 0.0,
            "d2h": plan.pred_d2h_B / (d2h / 1000.0) if d2h > 0 else 0.0,
            "cost_table": cost_table_from_trace(tr, plan, cfg.n_layer)}
