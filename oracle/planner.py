"""Partition planner oracle (TEST INFRASTRUCTURE ONLY).

Follows PAPER.md §III-D "Model Partitioning and Code Generation":

* Problem: split the topologically sorted graph into
  contiguous sub-models so that (1) every sub-model fits the GPU memory,
  (2) the compute of a sub-model overlaps the loading of the next one,
  C * sum t^{f|b} >= sum t^{load} (C = gradient-accumulation degree), and
  (3) the total size of the cut tensors is minimal.
* Algorithm 1 is the paper's recursive search; ``alg1_enumerate``
  writes it out literally (readings R5-R6 of DESIGN.md fix its loop bounds).
* Selection: "selects the one that minimizes the total tensor sizes
  between sub-models"; ties: fewer segments, then lexicographically smallest
  end-index vector.
* C: "We empirically determine C offline"; reading R8: the smallest
  C in [1, max_C] admitting a feasible plan.

Two layers live here:

1. ``Chain`` + ``valid_constraints`` / ``alg1_enumerate`` /
   ``brute_force_chain`` / ``determine_C``: the paper's generic formulation on
   an abstract chain of nodes (m_i, t_i^f, t_i^u) -- SPEC S:135-188's model.
2. ``plan``: the B200 cost model of SURVEY §8(c) c.1 / DESIGN.md §4 (nodes
   E, B_0..B_{L-1}, H; analytic integer costs; static device arena of
   persistent segment-1 weights + NSLOT rotating slots + activation stash +
   working set) with ``brute_force_plan`` and the exact ``dp_plan``.  The C++
   planner in libatom must return the identical plan (bit-exact).

All arithmetic is on Python ints (no floating point anywhere).
"""
from __future__ import annotations

import dataclasses
import itertools
from typing import List, Optional, Sequence

# ----------------------------------------------------------------------------
# 1. the paper's abstract formulation
# ----------------------------------------------------------------------------


@dataclasses.dataclass
class Chain:
    mem: List[int]      # m_i   ("max working memory size")
    t_fwd: List[int]    # t_i^f
    t_load: List[int]   # t_i^u ("loading time ... from host memory to device memory")

    @property
    def n(self):
        return len(self.mem)


def seg_sum(v: Sequence[int], s: int, e: int) -> int:
    """sum of v over the inclusive node range [s, e] (G.mem / G.comp_t / G.load_t)."""
    return sum(v[s:e + 1])


def valid_constraints(g: Chain, cs, ce, ls, le, cap, C) -> bool:
    """Alg. 1 ValidConstraints with C included (reading R5)."""
    return (seg_sum(g.mem, cs, ce) <= cap and seg_sum(g.mem, ls, le) <= cap
            and C * seg_sum(g.t_fwd, cs, ce) >= seg_sum(g.t_load, ls, le))


def alg1_enumerate(g: Chain, cap, C):
    """Algorithm 1 written out, returning the set of end-index tuples.

    Readings (R6): Main's l_e loop starts at num_nodes-1 (the printed
    ``G.num_nodes`` is one past the last node); PartitionModel's loop runs
    l^_e from num_nodes-1 down to l_e+1 (the next window must be non-empty);
    the recorded result is the full end-index vector, the first window
    included; a one-segment plan is not produced by Alg. 1 (it always splits).
    """
    n = g.n
    partitions = set()

    def partition_model(cs, ce, ls, le, t):
        if not valid_constraints(g, cs, ce, ls, le, cap, C):
            return
        if le == n - 1:
            partitions.add(tuple(t) + (le,))
            return
        # "squeeze boundary to keep more nodes within a certain range"
        for le_hat in range(n - 1, le, -1):
            t.append(le)                 # t.insert((l_s,l_e),(l_e+1,l^_e)) -- record boundary l_e
            partition_model(ls, le, le + 1, le_hat, t)
            t.pop()                      # backtracking

    cs = 0
    for ce in range(n - 2, cs - 1, -1):
        ls = ce + 1
        for le in range(n - 1, ls - 1, -1):
            partition_model(cs, ce, ls, le, [ce])
    return partitions


def all_partitions(n):
    """Every contiguous partition of n nodes as an end-index tuple (2^(n-1) of them)."""
    for mask in range(1 << (n - 1)):
        ends = [i for i in range(n - 1) if mask >> i & 1] + [n - 1]
        yield tuple(ends)


def brute_force_chain(g: Chain, cap, C, min_segments=2):
    """Filter all partitions by Alg. 1's pairwise predicate."""
    out = set()
    for ends in all_partitions(g.n):
        if len(ends) < min_segments:
            continue
        starts = [0] + [e + 1 for e in ends[:-1]]
        ok = all(valid_constraints(g, starts[k], ends[k], starts[k + 1], ends[k + 1], cap, C)
                 for k in range(len(ends) - 1))
        if len(ends) == 1:
            ok = seg_sum(g.mem, 0, g.n - 1) <= cap
        if ok:
            out.add(ends)
    return out


def select_best(plans, cut_bytes_of):
    """P:399 min total cut size; ties: fewer segments, then lexicographic ends."""
    plans = list(plans)
    if not plans:
        raise ValueError("EmptyInput")
    return min(plans, key=lambda e: (cut_bytes_of(e), len(e), tuple(e)))


def determine_C(t_fwd_segs, t_load_segs, max_C=64):
    """Smallest C with C * fwd(k) >= load(k+1) for all adjacent pairs."""
    for C in range(1, max_C + 1):
        if all(C * t_fwd_segs[k] >= t_load_segs[k + 1] for k in range(len(t_fwd_segs) - 1)):
            return C
    return None


# ----------------------------------------------------------------------------
# 2. the B200 cost model
# ----------------------------------------------------------------------------
FP32, BF16 = 0, 1
ACT_AUTO, ACT_STASH, ACT_RECOMPUTE, ACT_HYBRID = 0, 1, 2, 3


def ceil_div(a: int, b: int) -> int:
    return -((-a) // b)


def al(x: int, a: int) -> int:
    return ceil_div(x, a) * a


def al64(x):
    return al(x, 64)


def al256(x):
    return al(x, 256)


@dataclasses.dataclass
class PlanCfg:
    n_layer: int
    d_model: int
    n_head: int
    seq_len: int
    vocab: int
    micro_batch: int
    dtype: int = BF16
    C: int = 0                    # 0 = smallest feasible
    max_C: int = 64
    overlap_check: int = 1
    peak_flops: int = 1606 * 10 ** 12
    d2h_bw: int = 0               # 0 = link_bw
    cost_table: Optional[List[int]] = None    # per node [t_f_ns, t_b_ns] flattened
    state_budget: int = 0         # 0 = none; else cap on R1 + NSLOT*slot (model state on device)
    act_policy: int = ACT_AUTO    # AUTO: fewest re-forwarded blocks R = 0 (stash), 1, ..., L (reading R35)
    forced_ends: Optional[List[int]] = None
    n_recompute: int = 0          # ACT_HYBRID: re-forward blocks 1..n_recompute (those before the last segment)
    grad_rounds: int = 0          # > 0: host gradient sums + CPU AdamW (reading R37): bwd loads 8 B, stores 4 B
    op_nodes: int = 0             # 1: operator-granular graph ("a node ... is a layer or an operator"):
    #                               every block is two nodes, its attention half A_l (LN1, QKV, attention,
    #                               output projection) and its MLP half M_l (LN2, fc, GELU, fc2), so a
    #                               sub-model may end in the middle of a block (reading R40)

    @classmethod
    def from_gpt(cls, g, **kw):
        return cls(g.n_layer, g.d_model, g.n_head, g.seq_len, g.vocab, g.micro_batch, **kw)


def n_nodes(c: PlanCfg) -> int:
    """E, the block nodes (L, or 2L operator-granular halves), H."""
    return (2 if c.op_nodes else 1) * c.n_layer + 2


def node_params(c: PlanCfg):
    """Padded parameter count per node: each tensor starts on a 64-element boundary.
    Operator-granular: the attention half holds ln1.g, ln1.b, W_qkv, b_qkv, W_o, b_o, the MLP half
    ln2.g, ln2.b, W_fc, b_fc, W_pr, b_pr (the canonical block order split in two)."""
    d, V, T, L = c.d_model, c.vocab, c.seq_len, c.n_layer
    pE = al64(V * d) + al64(T * d)
    pA = al64(d) * 2 + al64(3 * d * d) + al64(3 * d) + al64(d * d) + al64(d)
    pM = al64(d) * 2 + al64(4 * d * d) + al64(4 * d) + al64(4 * d * d) + al64(d)
    pH = al64(d) * 2 + al64(V * d)
    return [pE] + ([pA, pM] * L if c.op_nodes else [pA + pM] * L) + [pH]


def node_flops_fwd(c: PlanCfg):
    """F^f per micro-batch: blocks 24 d^2 M + 2 d T (T+1) b (causal half); head 2 d V M.
    Operator-granular: attention half 8 d^2 M + 2 d T (T+1) b (QKV, attention, projection),
    MLP half 16 d^2 M (fc, fc2)."""
    d, V, T, b, L = c.d_model, c.vocab, c.seq_len, c.micro_batch, c.n_layer
    M = b * T
    fA = 8 * d * d * M + 2 * d * T * (T + 1) * b
    fM = 16 * d * d * M
    fH = 2 * d * V * M
    return [0] + ([fA, fM] * L if c.op_nodes else [fA + fM] * L) + [fH]


def node_flops_recompute(c: PlanCfg):
    """Re-forward a block needs inside its backward under ACT_RECOMPUTE: the QKV, attention
    projection and fc GEMMs (16 d^2 M) and the attention forward (the MLP projection's output is
    not needed by the backward)."""
    d, T, b, L = c.d_model, c.seq_len, c.micro_batch, c.n_layer
    M = b * T
    if c.op_nodes:   # unused: the operator-granular graph plans with the full stash only (R40)
        return [0] + [8 * d * d * M + 2 * d * T * (T + 1) * b, 8 * d * d * M] * L + [0]
    return [0] + [16 * d * d * M + 2 * d * T * (T + 1) * b] * L + [0]


@dataclasses.dataclass
class Costs:
    P: List[int]
    tf: List[int]
    tb: List[int]
    tlf: List[int]
    tlb: List[int]
    tmv: List[int]
    ts: List[int]
    ff: List[int]
    tbr: List[int]      # backward time including the block re-forward (ACT_RECOMPUTE)


def node_costs(c: PlanCfg, link_bw: int) -> Costs:
    P = node_params(c)
    n = len(P)
    ff = node_flops_fwd(c)
    fr = node_flops_recompute(c)
    if c.cost_table is not None:
        tf = [c.cost_table[2 * i] for i in range(n)]
        tb = [c.cost_table[2 * i + 1] for i in range(n)]
        tbr = [tb[i] + (tf[i] if 1 <= i < n - 1 else 0) for i in range(n)]
    else:
        tf = [ceil_div(f * 10 ** 9, c.peak_flops) for f in ff]
        tb = [ceil_div(2 * f * 10 ** 9, c.peak_flops) for f in ff]
        tbr = [ceil_div((2 * f + r) * 10 ** 9, c.peak_flops) for f, r in zip(ff, fr)]
    d2h = c.d2h_bw if c.d2h_bw > 0 else link_bw
    tlf = [ceil_div(4 * p * 10 ** 9, link_bw) for p in P]
    # host update placement (R37): the backward loads master + gradient sum (last segment: the sum)
    # and stores the sum; else master + m + v in (m + v), all three out
    hu = c.grad_rounds > 0
    tlb = [ceil_div((8 if hu else 12) * p * 10 ** 9, link_bw) for p in P]
    tmv = [ceil_div((4 if hu else 8) * p * 10 ** 9, link_bw) for p in P]
    ts = [ceil_div((4 if hu else 12) * p * 10 ** 9, d2h) for p in P]
    return Costs(P, tf, tb, tlf, tlb, tmv, ts, ff, tbr)


def wbytes(c):
    return 4 if c.dtype == FP32 else 2


def seg_need(c: PlanCfg, P_seg: int) -> int:
    """Bytes of one segment's full state on device:
    [compute-dtype weights | fp32 grad | fp32 master | AdamW m | AdamW v].
    Segment 1 holds it permanently (R1); segments 2..S rent a slot of this size."""
    return al256(wbytes(c) * P_seg) + 4 * al256(4 * P_seg)


def stash_blk_bytes(c: PlanCfg) -> int:
    """Per-block, per-micro-batch activation stash:
    x, qkv, o, x2, u (activation dtype) + LN1/LN2 stats (2 x fp32 per token) + LSE fp32 [b,h,T]."""
    ab = wbytes(c)
    d, M = c.d_model, c.micro_batch * c.seq_len
    return (al256(ab * M * d) + al256(ab * M * 3 * d) + al256(ab * M * d) + al256(ab * M * d)
            + al256(ab * M * 4 * d) + al256(8 * M) + al256(8 * M)
            + al256(4 * c.micro_batch * c.n_head * c.seq_len))


def hfin_bytes(c):
    return al256(wbytes(c) * c.micro_batch * c.seq_len * c.d_model)


def n_rc(c: PlanCfg, R: int, nb_last: int) -> int:
    """Re-forwarded blocks of a plan: blocks 1..R, but never one of the interleaved last segment."""
    return min(R, c.n_layer - nb_last)


def stash_bytes(c: PlanCfg, C: int, nb_last: int, S: int, R: int = 0) -> int:
    """Block stashes (C micro-batches for blocks before the last segment, 1 for blocks of the
    interleaved last segment) + [M, d] activation buffers at the last segment's boundary:
    its input for all C micro-batches (S >= 2) and the final hidden state (when the last
    segment has blocks; it is the input itself when the last segment is the head alone).
    The first R blocks before the last segment (R = L: all of them, ACT_RECOMPUTE) keep only
    their input (C copies); one full stash entry is then shared by their backward re-forwards."""
    L = c.n_layer
    nh = 1 if S == 1 else (C if nb_last == 0 else C + 1)
    nb_pre = L - nb_last
    r = n_rc(c, R, nb_last)
    return (stash_blk_bytes(c) * (C * (nb_pre - r) + nb_last) + hfin_bytes(c) * C * r + hfin_bytes(c) * nh
            + (stash_blk_bytes(c) if r > 0 else 0))


RED_ROWS = 128   # rows per partial-sum chunk in the deterministic column reductions


def work_bytes(c: PlanCfg, C: int) -> int:
    """Working set: token buffer, boundary-gradient buffer (all C micro-batches),
    per-token losses, max(block-backward scratch, head scratch), reduction
    partials, embedding-backward counting-sort scratch, small scalars.  The block-backward
    scratch of the bf16 path includes the attention backward's dS^T [b, h, T, T] (written by
    the dK/dV kernel, read by the dQ kernel)."""
    ab = wbytes(c)
    d, V, T, b, h = c.d_model, c.vocab, c.seq_len, c.micro_batch, c.n_head
    M = b * T
    Vp = al(V, 8)
    tokens = al256(4 * C * b * (T + 1))
    dh = al256(ab * C * M * d)
    losses = al256(4 * C * M)
    bwd_s = al256(ab * M * 4 * d) + 4 * al256(ab * M * d) + al256(4 * b * h * T) + al256(ab * M * 4 * d)
    if c.dtype == BF16:   # the attention backward's dS^T [b, h, T, T] (bf16) between its dK/dV and dQ kernels
        bwd_s += al256(2 * b * h * T * T)
    head_s = al256(ab * M * Vp) + 2 * al256(ab * M * d) + al256(8 * M)
    scratch = max(bwd_s, head_s)
    red = al256(4 * ceil_div(M, RED_ROWS) * 4 * d)
    emb = al256(4 * (3 * V + 1 + M))
    small = 256
    return tokens + dh + losses + scratch + red + emb + small


def nslot(S):
    """Rotating slots for the swapped segments 2..S: none when everything is resident,
    2 for a single swapped segment (next step's prefetch overlaps the current store),
    3 otherwise (executing + prefetching + draining)."""
    return 0 if S == 1 else (2 if S == 2 else 3)


@dataclasses.dataclass
class Plan:
    n_seg: int
    seg_end: List[int]
    C: int
    nslot: int
    cut_bytes: int
    r1_bytes: int
    slot_bytes: int
    stash_bytes: int
    work_bytes: int
    device_bytes: int
    pred_h2d_B: int
    pred_d2h_B: int
    pred_flops: int
    act_policy: int = ACT_STASH
    n_recompute: int = 0
    pred_step_ns: int = 0
    pred_hidden_ppm: int = 0


def _seg_tables(c: PlanCfg, k: Costs):
    n = len(k.P)

    def pre(v):
        s = [0]
        for x in v:
            s.append(s[-1] + x)
        return s
    return {name: pre(getattr(k, name)) for name in ("P", "tf", "tb", "tbr", "tlf", "tlb", "tmv", "ts")}, n


class Evaluator:
    """Feasibility of a partition under the cost model (memory + per-phase overlap)."""

    def __init__(self, c: PlanCfg, budget: int, link_bw: int, R: int = 0):
        """R: blocks 1..R are re-forwarded inside their backward (those before the last segment)."""
        self.c, self.budget, self.R = c, budget, R
        self.k = node_costs(c, link_bw)
        self.pre, self.n = _seg_tables(c, self.k)
        self.L = c.n_layer
        tbx = [self.k.tbr[v] if 1 <= v <= R and not c.op_nodes else self.k.tb[v] for v in range(self.n)]
        self.pre["tbx"] = _seg_tables(c, dataclasses.replace(self.k, tbr=tbx))[0]["tbr"]

    def tbn(self, i, j):
        """backward time of a segment that is not the last one (its re-forwarded blocks included)"""
        return self.s("tbx", i, j)

    def s(self, name, i, j):
        p = self.pre[name]
        return p[j + 1] - p[i]

    def need(self, i, j):
        return seg_need(self.c, self.s("P", i, j))

    def nblocks(self, i, j):
        """Whole blocks inside nodes [i..j] (block nodes 1..L; operator-granular: block l is the node
        pair 2l+1, 2l+2, counted when both halves are inside)."""
        if self.c.op_nodes:
            return sum(1 for l in range(self.L) if i <= 2 * l + 1 and 2 * l + 2 <= j)
        lo, hi = max(i, 1), min(j, self.L)
        return max(0, hi - lo + 1)

    def r1(self, e1):
        """R1: segment 1 [0..e1] stays fully resident (reading R11)."""
        return self.need(0, e1)

    def mem_fixed(self, C, e1, il, S, Q):
        """device bytes for first segment [0..e1], last [il..n-1], S segments, max need Q."""
        return (self.r1(e1) + nslot(S) * al256(Q) + stash_bytes(self.c, C, self.nblocks(il, self.n - 1), S, self.R)
                + work_bytes(self.c, C))

    def pair_ok(self, C, a, b, last):
        """a=(i,j), b=(j+1,k) adjacent segments; ``last``: b is the final segment.

        fwd:        C t_f(a) >= t_loadF(b); for a = segment 1 the prefetch of
                    segment 2 may start once the previous step's store of segment 2
                    has landed (during the backward of segment 1), so it overlaps the
                    rest of that backward and the forward of segment 1:
                    C (t_f(a) + t_b(a)) >= t_store(b) + t_loadF(b)
        bwd store:  C t_b(a) >= t_store(b)
        bwd load:   C t_b(b) >= t_loadB(a) (no load when a is the resident segment 1);
                    for the final, interleaved segment b:
                    C (t_f(b) + t_b(b)) >= t_mv(b) + t_loadB(a)."""
        if not self.c.overlap_check:
            return True
        (i, j), (j1, kk) = a, b
        first = i == 0
        if first:
            if C * (self.s("tf", i, j) + self.tbn(i, j)) < self.s("ts", j1, kk) + self.s("tlf", j1, kk):
                return False
        elif C * self.s("tf", i, j) < self.s("tlf", j1, kk):
            return False
        if C * self.tbn(i, j) < self.s("ts", j1, kk):
            return False
        load_a = 0 if first else self.s("tlb", i, j)
        if last:
            return C * (self.s("tf", j1, kk) + self.s("tb", j1, kk)) >= self.s("tmv", j1, kk) + load_a
        return C * self.tbn(j1, kk) >= load_a

    def segments(self, ends):
        starts = [0] + [e + 1 for e in ends[:-1]]
        return list(zip(starts, ends))

    def slot_need(self, ends):
        """Q = the largest swapped segment's state (0 when S = 1)."""
        segs = self.segments(ends)
        return max([self.need(i, j) for i, j in segs[1:]], default=0)

    def device_bytes(self, C, ends):
        segs = self.segments(ends)
        return self.mem_fixed(C, ends[0], segs[-1][0], len(ends), self.slot_need(ends))

    def violation(self, C, ends):
        """None if feasible, else the name of the first violated constraint."""
        segs = self.segments(ends)
        if self.device_bytes(C, ends) > self.budget:
            return "memory"
        if self.c.state_budget > 0:
            Q = self.slot_need(ends)
            if self.r1(ends[0]) + nslot(len(ends)) * al256(Q) > self.c.state_budget:
                return "state memory"
        for k in range(len(segs) - 1):
            if not self.pair_ok(C, segs[k], segs[k + 1], k + 1 == len(segs) - 1):
                return f"overlap(seg {k + 1}, seg {k + 2})"
        return None

    def make_plan(self, C, ends) -> Plan:
        c, segs = self.c, self.segments(ends)
        S = len(ends)
        Q = self.slot_need(ends)
        nb_last = self.nblocks(segs[-1][0], self.n - 1)
        st = stash_bytes(c, C, nb_last, S, self.R)
        r = n_rc(c, self.R, nb_last)
        pol = ACT_STASH if r == 0 else (ACT_RECOMPUTE if r == self.L - nb_last else ACT_HYBRID)
        wk = work_bytes(c, C)
        r1 = self.r1(ends[0])
        M = c.micro_batch * c.seq_len
        P = [self.s("P", i, j) for i, j in segs]
        # forward loads fp32 masters of 2..S; backward loads master+m+v of 2..S-1 and m+v of S
        # (host update placement: master + gradient sum, and the sum of S; stores the sum)
        hu = c.grad_rounds > 0
        h2d = (sum(4 * p for p in P[1:]) + sum((8 if hu else 12) * p for p in P[1:-1])
               + (4 if hu else 8) * P[-1]) if S >= 2 else 0
        d2h = sum((4 if hu else 12) * p for p in P[1:])
        return Plan(S, list(ends), C, nslot(S), (S - 1) * wbytes(c) * M * c.d_model, r1, al256(Q), st, wk,
                    r1 + nslot(S) * al256(Q) + st + wk, h2d, d2h,
                    C * sum(3 * f for f in self.k.ff), pol, r)


def policies(c: PlanCfg):
    """Re-forward counts R to try, in order. ACT_AUTO: R = 0 (full stash), 1, ..., L (R = L
    re-forwards every block before the last segment, ACT_RECOMPUTE): every re-forwarded block
    costs its forward again, so the fewest that make a plan feasible wins, then the smallest C
    (readings R28, R35)."""
    if c.op_nodes:   # operator-granular graph: the full stash only (reading R40)
        return [0] if c.act_policy in (ACT_AUTO, ACT_STASH) else []
    if c.act_policy == ACT_AUTO:
        return list(range(c.n_layer + 1))
    return {ACT_STASH: [0], ACT_RECOMPUTE: [c.n_layer], ACT_HYBRID: [c.n_recompute]}[c.act_policy]


def brute_force_plan(c: PlanCfg, budget: int, link_bw: int) -> Optional[Plan]:
    """Enumerate every contiguous partition x every C (SURVEY §8(c) c.5 pin)."""
    for pol in policies(c):
        ev = Evaluator(c, budget, link_bw, pol)
        Cs = [c.C] if c.C > 0 else range(1, c.max_C + 1)
        for C in Cs:
            feas = [e for e in all_partitions(ev.n) if ev.violation(C, list(e)) is None]
            if c.forced_ends is not None:
                feas = [e for e in feas if list(e) == list(c.forced_ends)]
            if feas:
                best = min(feas, key=lambda e: ((len(e) - 1) * wbytes(c), len(e), e))
                return ev.make_plan(C, list(best))
    return None


def _dp_for_C(ev: Evaluator, C: int):
    """Exact optimum (min S, then lexicographically smallest ends) for one C.

    S = 1 and S = 2 are enumerated directly (their arenas hold 1 and 2 slots).
    For S >= 3 (3 slots) the memory bound is
        W1(first) + 3*al256(Q) + stash(last) + work <= budget,   Q = max segment need,
    so for every candidate Q (a distinct segment need) and every first segment
    [0..e1] a right-to-left DP over states (i, j) = "current segment [i..j]"
    computes the fewest segments that complete the chain through pairwise-valid
    transitions to an admissible last segment.  The lexicographically smallest
    ends are then read greedily off the DP table."""
    n, budget = ev.n, ev.budget
    # S = 1
    if ev.violation(C, [n - 1]) is None:
        return [n - 1]
    if n < 2:
        return None
    for e in range(n - 1):
        if ev.violation(C, [e, n - 1]) is None:
            return [e, n - 1]
    if n < 3:
        return None
    needs = sorted({ev.need(i, j) for i in range(1, n) for j in range(i, n)})
    best_ans = None
    INF = 1 << 30
    wk = work_bytes(ev.c, C)
    for Q in needs:
        base = 3 * al256(Q) + wk
        if base > budget:
            break
        sb = ev.c.state_budget
        for e1 in range(n - 2):
            if sb > 0 and 3 * al256(Q) + ev.r1(e1) > sb:
                break
            rem = budget - base - ev.r1(e1)
            if rem < 0:
                break
            # admissible last segments [il..n-1]
            term = [il for il in range(e1 + 2, n)
                    if ev.need(il, n - 1) <= Q
                    and stash_bytes(ev.c, C, ev.nblocks(il, n - 1), 3, ev.R) <= rem]
            if not term:
                continue
            tset = set(term)
            # best[(i, j)] = fewest segments after [i..j] to finish (INF if impossible)
            best = {}

            def transition(i, j):
                v = INF
                if (j + 1) in tset and ev.pair_ok(C, (i, j), (j + 1, n - 1), True):
                    v = 1
                for k in range(j + 1, n - 1):
                    r = best[(j + 1, k)]
                    if r + 1 < v and ev.pair_ok(C, (i, j), (j + 1, k), False):
                        v = r + 1
                return v

            # middle states (i, j), e1 < i <= j <= n-2, by decreasing end j
            for j in range(n - 2, e1, -1):
                for i in range(e1 + 1, j + 1):
                    best[(i, j)] = INF if ev.need(i, j) > Q else transition(i, j)
            best[(0, e1)] = transition(0, e1)
            r0 = best.get((0, e1), INF)
            if r0 >= INF:
                continue
            S = r0 + 1
            # greedy lexicographic reconstruction
            ends, cur, left = [e1], (0, e1), r0
            while left > 0:
                i, j = cur
                if left == 1:
                    ends.append(n - 1)
                    break
                for k in range(j + 1, n - 1):
                    if best.get((j + 1, k), INF) == left - 1 and ev.pair_ok(C, (i, j), (j + 1, k), False):
                        ends.append(k)
                        cur = (j + 1, k)
                        left -= 1
                        break
                else:
                    raise AssertionError("inconsistent DP table")
            cand = (S, ends)
            if best_ans is None or cand < best_ans:
                best_ans = cand
    return None if best_ans is None else best_ans[1]


def dp_plan(c: PlanCfg, budget: int, link_bw: int) -> Optional[Plan]:
    for pol in policies(c):
        ev = Evaluator(c, budget, link_bw, pol)
        Cs = [c.C] if c.C > 0 else range(1, c.max_C + 1)
        for C in Cs:
            if c.forced_ends is not None:
                if ev.violation(C, list(c.forced_ends)) is None:
                    return ev.make_plan(C, list(c.forced_ends))
                continue
            ends = _dp_for_C(ev, C)
            if ends is not None:
                return ev.make_plan(C, ends)
    return None


def plan_R(c: PlanCfg, p: Plan) -> int:
    """The R an evaluator needs to reproduce plan p (its re-forwarded blocks are 1..n_recompute)."""
    return p.n_recompute


def plan(c: PlanCfg, budget: int, link_bw: int) -> Optional[Plan]:
    """The planner's answer: the optimum of the cost model (exact DP), with the
    schedule simulation attached."""
    p = dp_plan(c, budget, link_bw)
    if p is not None:
        from . import schedule
        ev = Evaluator(c, budget, link_bw, plan_R(c, p))
        sim = schedule.simulate(schedule.emit(p.n_seg, p.C, False), ev, p)
        p.pred_step_ns, p.pred_hidden_ppm = sim["makespan"], sim["hidden_ppm"]
    return p
