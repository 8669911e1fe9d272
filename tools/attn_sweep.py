"""Causal attention forward / backward time (default 32 heads x d_h = 80; argv: h dh) over sequence lengths with B*T fixed, to split
the kernels' time into a per-CTA fixed cost and a per-key-block cost (least squares over the
sweep), next to library kernels on the same shapes (cuDNN SDPA, flash_attn) as reference points.
FLOPs counted causally: fwd 4 B h T^2/2 dh, bwd 2x fwd (algorithmic, S recompute not counted)."""
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom  # noqa: E402


def bench(fn, it=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3   # us


h, dh = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (32, 80)
tokens = 16384
d = h * dh
rows = []
TS = [int(t) for t in os.environ.get("ATOM_SWEEP_T", "512,1024,2048,4096,8192").split(",")]
for T in TS:
    B = tokens // T
    qkv = (torch.randn(B * T, 3 * d, device="cuda") * 0.5).bfloat16()
    o = torch.empty(B * T, d, device="cuda", dtype=torch.bfloat16)
    do = torch.randn(B * T, d, device="cuda").bfloat16()
    lse = torch.empty(B * h * T, device="cuda")
    ds = torch.empty(B * h * T, device="cuda")
    dqkv = torch.empty_like(qkv)
    fl = 4.0 * B * h * T * T / 2 * dh
    tf = bench(lambda: atom.k_attn_fwd(atom.ATTN_TC, atom.BF16, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, h,
                                       dh))
    tb = bench(lambda: atom.k_attn_bwd(atom.ATTN_TC_DS, atom.BF16, qkv.data_ptr(), o.data_ptr(), do.data_ptr(),
                                       lse.data_ptr(), ds.data_ptr(), dqkv.data_ptr(), B, T, h, dh))
    npair = (T + 255) // 256
    ncta = B * h * npair
    nblk = B * h * sum(2 * qp + 2 for qp in range(npair))   # key blocks of 128 for both query tiles
    line = f"T={T:5d} B={B:3d}: ours fwd {tf:7.1f} us {fl / tf / 1e6:6.1f} TF  bwd {tb:7.1f} us {2 * fl / tb / 1e6:6.1f} TF"
    q, k, v = (t.reshape(B, T, h, dh).transpose(1, 2) for t in qkv.view(B * T, 3, d).unbind(1))
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    for name, be in (("cudnn", torch.nn.attention.SDPBackend.CUDNN_ATTENTION),
                     ("flash", torch.nn.attention.SDPBackend.FLASH_ATTENTION)):
        try:
            with torch.nn.attention.sdpa_kernel(be):
                t1 = bench(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True))
                qq, kk, vv = (x.detach().requires_grad_() for x in (q, k, v))
                y = F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
                g = torch.randn_like(y)
                t2 = bench(lambda: torch.autograd.grad(y, (qq, kk, vv), g, retain_graph=True))
            line += f" | {name} fwd {fl / t1 / 1e6:6.1f} bwd {2 * fl / t2 / 1e6:6.1f} TF"
        except Exception as ex:  # noqa: BLE001
            line += f" | {name} n/a ({type(ex).__name__})"
    print(line, flush=True)
    # dK/dV kernel: one CTA per (b, h, 128-key block kb), 64-query blocks from the diagonal on
    ncta_b = B * h * (T // 128)
    nblk_b = B * h * sum((T - 128 * kb) // 64 for kb in range(T // 128))
    rows.append((ncta, nblk, tf, ncta_b, nblk_b, tb))
for i, nm in ((0, "fwd"), (3, "bwd")):
    A = np.array([[r[i], r[i + 1]] for r in rows], dtype=float)
    y = np.array([r[i + 2] for r in rows])
    (c_cta, c_blk), *_ = np.linalg.lstsq(A, y, rcond=None)
    print(f"{nm}: per CTA {c_cta * 1e3 * 148:.1f} ns, per block {c_blk * 1e3 * 148:.1f} ns (one SM's time; fwd block = "
          f"128 keys x 2 query tiles, bwd block = 64 queries x 128 keys, dK/dV + dQ + D together)")
