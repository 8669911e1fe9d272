"""Thin ctypes binding of libatom (include/atom.h, include/atom_kernels.h).

Argument marshalling only: every step of the training path runs in libatom's kernels.
There is no fallback: if libatom.so is missing or fails to load, importing this module
raises (build it with ``python -m paper_2403_10504_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ATOM_LIB: an alternative build of the same library (tools/build_variant.py A/B experiments)
LIB_PATH = os.environ.get("ATOM_LIB") or os.path.join(HERE, "libatom.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libatom.so not built at {LIB_PATH}; run `python -m paper_2403_10504_b200.build`")
lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants
ATOM_OK, ATOM_E_INVALID, ATOM_E_INFEASIBLE, ATOM_E_CAPACITY = 0, -1, -2, -3
ATOM_E_CUDA, ATOM_E_NCCL, ATOM_E_OOM, ATOM_E_STATE = -4, -5, -6, -7
FP32, BF16 = 0, 1
ACT_AUTO, ACT_STASH, ACT_RECOMPUTE, ACT_HYBRID = 0, 1, 2, 3
MAX_SEG = 256
IMPL_TC, IMPL_SIMT = 0, 1
EPI_STORE, EPI_BIAS, EPI_BIAS_RES, EPI_BIAS_GELU, EPI_DGELU, EPI_ACC_F32 = range(6)


class AtomError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"atom status {code}: {msg}")
        self.code = code


def _err():
    f = getattr(lib, "atom_last_error", None)
    if f is None:
        return ""
    f.restype = C.c_char_p
    m = f()
    return m.decode() if m else ""


def check(code):
    if code != ATOM_OK:
        raise AtomError(code, _err())
    return code


# ---------------------------------------------------------------- kernels ABI
lib.atom_k_gemm.restype = C.c_int
lib.atom_k_gemm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_long, C.c_int,
                            C.c_void_p, C.c_long, C.c_int, C.c_int, C.c_void_p, C.c_long, C.c_void_p, C.c_long,
                            C.c_void_p, C.c_void_p, C.c_long, C.c_void_p, C.c_long, C.c_int, C.c_void_p]
lib.atom_k_cpu_adamw.restype = C.c_int
lib.atom_k_cpu_adamw.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_long, C.c_float, C.c_float,
                                 C.c_float, C.c_float, C.c_float, C.c_long, C.c_float, C.c_int]


def k_cpu_adamw(p, g, m, v, lr_t, b1, b2, eps, wd, t, gscale=1.0, threads=0):
    """atom_k_cpu_adamw on float32 numpy arrays (p, m, v updated in place)."""
    for a in (p, g, m, v):
        assert a.dtype == np.float32 and a.flags.c_contiguous
    return check(lib.atom_k_cpu_adamw(p.ctypes.data, g.ctypes.data, m.ctypes.data, v.ctypes.data, p.size, lr_t, b1,
                                      b2, eps, wd, t, gscale, threads))


lib.atom_k_launch_count.restype = C.c_ulonglong


def k_gemm(impl, dtype, M, N, K, A, lda, a_mn, B, ldb, b_mn, mode, out, ldo, out2=0, ldo2=0, bias=0, res=0, ldr=0,
           aux=0, ldx=0, force_bn=0, stream=0):
    return check(lib.atom_k_gemm(impl, dtype, M, N, K, A, lda, int(a_mn), B, ldb, int(b_mn), mode, out, ldo,
                                 out2 or None, ldo2, bias or None, res or None, ldr, aux or None, ldx, force_bn,
                                 stream or None))


def launch_count():
    return int(lib.atom_k_launch_count())


lib.atom_k_launch_log.restype = C.c_int
lib.atom_k_launch_log.argtypes = [C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]


def launch_log() -> dict:
    """{kernel family: launches since load} (atom_k_launch_log)."""
    n = C.c_int64(0)
    lib.atom_k_launch_log(None, 0, C.byref(n))
    buf = C.create_string_buffer(int(n.value) + 1)
    check(lib.atom_k_launch_log(buf, n.value + 1, C.byref(n)))
    out = {}
    for line in buf.value.decode().splitlines():
        k, v = line.rsplit(" ", 1)
        out[k] = int(v)
    return out


# ---------------------------------------------------------------- training ABI
class ModelCfg(C.Structure):
    _fields_ = [("n_layer", C.c_int32), ("d_model", C.c_int32), ("n_head", C.c_int32), ("seq_len", C.c_int32),
                ("vocab", C.c_int32), ("micro_batch", C.c_int32), ("dtype", C.c_int32), ("C", C.c_int32),
                ("max_C", C.c_int32), ("act_policy", C.c_int32), ("overlap_check", C.c_int32),
                ("peak_flops", C.c_int64), ("d2h_bw", C.c_int64), ("state_budget", C.c_int64),
                ("cost_table", C.POINTER(C.c_int64)), ("forced_ends", C.POINTER(C.c_int32)),
                ("n_forced", C.c_int32), ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("weight_decay", C.c_float), ("warmup_steps", C.c_int32),
                ("sync_every", C.c_int32), ("n_recompute", C.c_int32), ("grad_rounds", C.c_int32),
                ("cpu_threads", C.c_int32), ("dropout_p", C.c_float), ("op_nodes", C.c_int32),
                ("dropout_seed", C.c_uint64)]


class Plan(C.Structure):
    _fields_ = [("n_seg", C.c_int32), ("seg_end", C.c_int32 * MAX_SEG), ("C", C.c_int32), ("nslot", C.c_int32),
                ("act_policy", C.c_int32), ("cut_bytes", C.c_int64), ("r1_bytes", C.c_int64), ("slot_bytes", C.c_int64),
                ("stash_bytes", C.c_int64), ("work_bytes", C.c_int64), ("device_bytes", C.c_int64),
                ("pred_step_ns", C.c_int64), ("pred_hidden_ppm", C.c_int64), ("pred_h2d_B", C.c_int64),
                ("pred_d2h_B", C.c_int64), ("pred_flops", C.c_int64), ("hbm_budget", C.c_int64),
                ("link_bw", C.c_int64), ("n_recompute", C.c_int32), ("reserved", C.c_int32)]

    def ends(self):
        return [self.seg_end[i] for i in range(self.n_seg)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f not in ("seg_end", "reserved")}
        d["seg_end"] = self.ends()
        return d


def make_cfg(g, dtype=BF16, C_=0, max_C=64, overlap_check=1, peak_flops=1606 * 10 ** 12, d2h_bw=0,
             state_budget=0, cost_table=None, forced_ends=None, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8,
             weight_decay=0.01, warmup_steps=3000, sync_every=0, act_policy=0, n_recompute=0, grad_rounds=0,
             cpu_threads=0, dropout_p=0.0, dropout_seed=0, op_nodes=0):
    """atom_model_cfg from a synth.GPTConfig-like object (keeps ctypes arrays alive on the struct)."""
    c = ModelCfg()
    c.n_layer, c.d_model, c.n_head, c.seq_len, c.vocab, c.micro_batch = (
        g.n_layer, g.d_model, g.n_head, g.seq_len, g.vocab, g.micro_batch)
    c.dtype, c.C, c.max_C, c.act_policy, c.overlap_check = dtype, C_, max_C, act_policy, overlap_check
    c.peak_flops, c.d2h_bw, c.state_budget = peak_flops, d2h_bw, state_budget
    if cost_table is not None:
        arr = (C.c_int64 * len(cost_table))(*cost_table)
        c._ct = arr
        c.cost_table = C.cast(arr, C.POINTER(C.c_int64))
    if forced_ends is not None:
        arr = (C.c_int32 * len(forced_ends))(*forced_ends)
        c._fe = arr
        c.forced_ends = C.cast(arr, C.POINTER(C.c_int32))
        c.n_forced = len(forced_ends)
    c.lr, c.beta1, c.beta2, c.eps, c.weight_decay = lr, beta1, beta2, eps, weight_decay
    c.warmup_steps, c.sync_every, c.n_recompute = warmup_steps, sync_every, n_recompute
    c.grad_rounds, c.cpu_threads = grad_rounds, cpu_threads
    c.dropout_p, c.dropout_seed, c.op_nodes = dropout_p, dropout_seed, op_nodes
    return c


lib.atom_plan.restype = C.c_int
lib.atom_plan.argtypes = [C.POINTER(ModelCfg), C.c_int64, C.c_int64, C.POINTER(Plan)]
lib.atom_plan_schedule.restype = C.c_int
lib.atom_plan_schedule.argtypes = [C.POINTER(Plan), C.c_int32, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]


def atom_plan(cfg: ModelCfg, hbm_budget: int, link_bw: int) -> Plan:
    p = Plan()
    check(lib.atom_plan(C.byref(cfg), int(hbm_budget), int(link_bw), C.byref(p)))
    return p


class Profile(C.Structure):
    _fields_ = [("flops_per_s", C.c_double), ("h2d_bytes_per_s", C.c_double), ("d2h_bytes_per_s", C.c_double),
                ("compute_busy_ms", C.c_double), ("executed_flops", C.c_double), ("n_nodes", C.c_int32),
                ("have_table", C.c_int32)]


lib.atom_profile.restype = C.c_int
lib.atom_profile.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int64, C.POINTER(Profile)]
lib.atom_profile_trace.restype = C.c_int
lib.atom_profile_trace.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_int64,
                                   C.POINTER(Profile)]


def _profile_dict(pr, table):
    return {"flops": pr.flops_per_s, "h2d": pr.h2d_bytes_per_s, "d2h": pr.d2h_bytes_per_s,
            "compute_busy_ms": pr.compute_busy_ms, "executed_flops": pr.executed_flops,
            "cost_table": [int(x) for x in table] if pr.have_table else []}


def atom_profile_trace(trace: str, cfg: ModelCfg, plan: Plan) -> dict:
    """atom_profile_trace: the measured profile (rates, per-node cost table) of a traced step."""
    n = 2 * (cfg.n_layer + 2)
    table = (C.c_int64 * n)()
    pr = Profile()
    check(lib.atom_profile_trace(trace.encode(), C.byref(cfg), C.byref(plan), table, n, C.byref(pr)))
    return _profile_dict(pr, table)


def atom_plan_schedule(plan: Plan, sync=False) -> str:
    n = C.c_int64(0)
    lib.atom_plan_schedule(C.byref(plan), int(sync), None, 0, C.byref(n))
    buf = C.create_string_buffer(n.value + 1)
    check(lib.atom_plan_schedule(C.byref(plan), int(sync), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


class Stats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("kernel_launches", C.c_int64), ("gemm_launches", C.c_int64),
                ("gemm_ms", C.c_double), ("gemm_flops", C.c_double), ("h2d_bytes", C.c_double),
                ("d2h_bytes", C.c_double), ("copy_ms", C.c_double), ("copy_hidden_ms", C.c_double),
                ("step_ms", C.c_double), ("h2d_ms", C.c_double), ("h2d_hidden_ms", C.c_double),
                ("d2h_ms", C.c_double), ("d2h_hidden_ms", C.c_double), ("compute_busy_ms", C.c_double),
                ("compute_span_ms", C.c_double), ("host_issue_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = C.c_void_p
lib.atom_nccl_unique_id.restype = C.c_int
lib.atom_nccl_unique_id.argtypes = [C.c_void_p]
lib.atom_peer_create.restype = C.c_int
lib.atom_peer_create.argtypes = [C.POINTER(ModelCfg), C.POINTER(Plan), C.c_int32, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_uint64, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(_P)]
lib.atom_step.restype = C.c_int
lib.atom_step.argtypes = [_P, C.c_void_p, C.POINTER(C.c_float)]
lib.atom_step_device.restype = C.c_int
lib.atom_step_device.argtypes = [_P, C.c_void_p, C.POINTER(C.c_float)]
lib.atom_sync.restype = C.c_int
lib.atom_sync.argtypes = [C.POINTER(_P), C.c_int32, C.c_int32]
lib.atom_get_params.restype = C.c_int
lib.atom_get_params.argtypes = [_P, C.c_void_p, C.c_void_p, C.c_void_p]
lib.atom_get_trace.restype = C.c_int
lib.atom_get_trace.argtypes = [_P, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
lib.atom_get_gemm_log.restype = C.c_int
lib.atom_get_gemm_log.argtypes = [_P, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
lib.atom_get_kernel_log.restype = C.c_int
lib.atom_get_kernel_log.argtypes = [_P, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
lib.atom_get_stats.restype = C.c_int
lib.atom_get_stats.argtypes = [_P, C.POINTER(Stats)]
lib.atom_reset_stats.restype = C.c_int
lib.atom_reset_stats.argtypes = [_P, C.c_int32]
lib.atom_peer_destroy.restype = C.c_int
lib.atom_peer_destroy.argtypes = [_P]


lib.atom_comm_reset.restype = C.c_int
lib.atom_comm_reset.argtypes = [_P, C.c_void_p, C.c_int32, C.c_int32]
lib.atom_comm_shrink.restype = C.c_int
lib.atom_comm_shrink.argtypes = [_P, C.POINTER(C.c_int32), C.c_int32, C.c_int32]
lib.atom_broadcast_state.restype = C.c_int
lib.atom_broadcast_state.argtypes = [_P, C.c_int32, C.c_int32]
lib.atom_peer_info.restype = C.c_int
lib.atom_peer_info.argtypes = [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64)]


def atom_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib.atom_nccl_unique_id(buf))
    return buf.raw


def n_params(g) -> int:
    L, d, T, V = g.n_layer, g.d_model, g.seq_len, g.vocab
    return V * d + T * d + L * (12 * d * d + 13 * d) + 2 * d + V * d


class Peer:
    """One whole-model replica (atom_peer) on one GPU.  The device arena is a torch allocation."""

    def __init__(self, cfg: ModelCfg, plan: Plan, device: int = 0, init_params=None, seed: int = 0,
                 nccl_id: bytes = None, nranks: int = 1, rank: int = 0):
        import torch
        self.cfg, self.plan = cfg, plan
        self.N = n_params(cfg)
        self.arena = torch.empty(plan.device_bytes, dtype=torch.uint8, device=f"cuda:{device}")
        torch.cuda.synchronize(device)
        self._init = None
        ip = None
        if init_params is not None:
            self._init = np.ascontiguousarray(init_params, dtype=np.float32)
            assert self._init.size == self.N
            ip = self._init.ctypes.data
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        h = _P()
        check(lib.atom_peer_create(C.byref(cfg), C.byref(plan), device, self.arena.data_ptr(), plan.device_bytes,
                                   ip, seed, idbuf, nranks, rank, C.byref(h)))
        self.h = h

    def step(self, tokens) -> float:
        t = np.ascontiguousarray(tokens, dtype=np.int32)
        want = (self.plan.C * self.cfg.micro_batch, self.cfg.seq_len + 1)
        assert t.shape == want, (t.shape, want)
        loss = C.c_float()
        check(lib.atom_step(self.h, t.ctypes.data, C.byref(loss)))
        return loss.value

    def step_device(self, tokens_dev) -> float:
        loss = C.c_float()
        check(lib.atom_step_device(self.h, tokens_dev.data_ptr(), C.byref(loss)))
        return loss.value

    def params(self, which=("master", "m", "v")):
        out = {w: np.empty(self.N, dtype=np.float32) for w in which}
        ptr = lambda k: out[k].ctypes.data if k in out else None
        check(lib.atom_get_params(self.h, ptr("master"), ptr("m"), ptr("v")))
        return out

    def trace(self) -> str:
        n = C.c_int64(0)
        lib.atom_get_trace(self.h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        check(lib.atom_get_trace(self.h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def profile(self) -> dict:
        """atom_profile: rates and per-node cost table measured from this peer's last step."""
        n = 2 * (self.cfg.n_layer + 2)
        table = (C.c_int64 * n)()
        pr = Profile()
        check(lib.atom_profile(self.h, table, n, C.byref(pr)))
        return _profile_dict(pr, table)

    def kernel_log(self) -> dict:
        """Per kernel category since the last reset_stats(timing=True): {category: (groups, ms)}."""
        n = C.c_int64(0)
        lib.atom_get_kernel_log(self.h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        check(lib.atom_get_kernel_log(self.h, buf, n.value + 1, C.byref(n)))
        out = {}
        for line in buf.value.decode().splitlines():
            k, cnt, ms = line.split()
            out[k] = (int(cnt), float(ms))
        return out

    def gemm_log(self) -> list:
        """Per-shape GEMM timing since the last reset_stats(timing=True): dicts with M, N, K,
        a_mn, b_mn, epilogue, launches, ms, tflops."""
        n = C.c_int64(0)
        lib.atom_get_gemm_log(self.h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        check(lib.atom_get_gemm_log(self.h, buf, n.value + 1, C.byref(n)))
        keys = ("M", "N", "K", "a_mn", "b_mn", "epilogue", "launches", "ms", "tflops")
        out = []
        for line in buf.value.decode().splitlines():
            f = line.split()
            out.append({k: (float(v) if k in ("ms", "tflops") else int(v)) for k, v in zip(keys, f)})
        return out

    def comm_reset(self, nccl_id: bytes, nranks: int, rank: int):
        """atom_comm_reset: leave the current averaging communicator, join a new one."""
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        check(lib.atom_comm_reset(self.h, idbuf, nranks, rank))

    def comm_shrink(self, exclude_ranks, abort_ops=False):
        """atom_comm_shrink: ncclCommShrink without the given (failed / leaving) ranks."""
        ex = (C.c_int32 * max(len(exclude_ranks), 1))(*exclude_ranks)
        check(lib.atom_comm_shrink(self.h, ex, len(exclude_ranks), int(abort_ops)))

    def broadcast_state(self, root: int, adopt: bool):
        """atom_broadcast_state (collective): root sends master, m, v and step count; adopt=True
        overwrites this peer's state with root's (a joiner)."""
        check(lib.atom_broadcast_state(self.h, root, int(adopt)))

    def info(self) -> dict:
        r, n, t = C.c_int32(), C.c_int32(), C.c_int64()
        check(lib.atom_peer_info(self.h, C.byref(r), C.byref(n), C.byref(t)))
        return {"rank": r.value, "nranks": n.value, "step": t.value}

    def stats(self) -> dict:
        s = Stats()
        check(lib.atom_get_stats(self.h, C.byref(s)))
        return s.as_dict()

    def reset_stats(self, timing=0):
        """timing: 0 off, 1 per-GEMM CUDA events, 2 also per kernel category (kernel_log)."""
        check(lib.atom_reset_stats(self.h, int(timing)))

    def destroy(self):
        if getattr(self, "h", None):
            lib.atom_peer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def atom_sync(peers, flush=False):
    arr = (_P * len(peers))(*[p.h for p in peers])
    check(lib.atom_sync(arr, len(peers), int(flush)))


ATTN_TC, ATTN_MMA, ATTN_SIMT, ATTN_TC_DS = 0, 1, 2, 3
lib.atom_k_attn_fwd.restype = C.c_int
lib.atom_k_attn_fwd.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                C.c_int, C.c_void_p]
lib.atom_k_attn_bwd.restype = C.c_int
lib.atom_k_attn_bwd.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]


def k_attn_fwd(impl, dtype, qkv, o, lse, B, T, h, dh, stream=0):
    return check(lib.atom_k_attn_fwd(impl, dtype, qkv, o, lse, B, T, h, dh, stream or None))


def k_attn_bwd(impl, dtype, qkv, o, dout, lse, dsum, dqkv, B, T, h, dh, stream=0):
    return check(lib.atom_k_attn_bwd(impl, dtype, qkv, o, dout, lse, dsum, dqkv, B, T, h, dh, stream or None))


DROP_EMBD, DROP_ATTN, DROP_RESID_ATTN, DROP_RESID_MLP = 0, 1, 2, 3
lib.atom_k_dropout.restype = C.c_int
lib.atom_k_dropout.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_long, C.c_double, C.c_ulonglong, C.c_int,
                               C.c_int, C.c_int, C.c_void_p]


def k_dropout(dtype, x, y, n, p, seed, site, layer, micro_step, stream=0):
    """atom_k_dropout on device pointers x, y (x == y allowed): y = x * keep / (1 - p)."""
    return check(lib.atom_k_dropout(dtype, x, y, n, p, seed, site, layer, micro_step, stream or None))
