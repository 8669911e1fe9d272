"""Time the causal attention kernels (tcgen05 / mma.sync) on the GPT-3 shapes with CUDA events,
next to flash_attn (library reference point, if importable). FLOPs counted causally:
fwd 2 * 2 * B*h*T^2/2*dh, bwd 2.5x fwd."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom


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
    return s.elapsed_time(e) / it


shapes = [("xl", 8, 2048, 16, 128), ("2.7b", 8, 2048, 32, 80), ("dh64", 8, 2048, 32, 64)]
if len(sys.argv) > 1:
    shapes = [s for s in shapes if s[0] in sys.argv[1:]]
try:
    import flash_attn
    fa = flash_attn.flash_attn_func
except Exception:  # noqa: BLE001
    fa = None
for name, B, T, h, dh in shapes:
    d = h * dh
    qkv = (torch.randn(B * T, 3 * d, device="cuda") * 0.5).bfloat16()
    o = torch.empty(B * T, d, device="cuda", dtype=torch.bfloat16)
    do = torch.randn(B * T, d, device="cuda").bfloat16()
    lse = torch.empty(B * h * T, device="cuda")
    ds = torch.empty(B * h * T, device="cuda")
    dqkv = torch.empty_like(qkv)
    fl = 4.0 * B * h * T * T / 2 * dh
    out = [f"{name:5s} B={B} T={T} h={h} dh={dh}"]
    for impl, nm in ((atom.ATTN_TC, "tc"), (atom.ATTN_MMA, "mma")):
        tf = bench(lambda: atom.k_attn_fwd(impl, atom.BF16, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, h, dh))
        tb = bench(lambda: atom.k_attn_bwd(impl, atom.BF16, qkv.data_ptr(), o.data_ptr(), do.data_ptr(),
                                           lse.data_ptr(), ds.data_ptr(), dqkv.data_ptr(), B, T, h, dh))
        out.append(f"{nm}: fwd {tf*1e3:7.1f} us {fl/tf/1e9:6.1f} TF  bwd {tb*1e3:7.1f} us {2.5*fl/tb/1e9:6.1f} TF")
    if fa is not None:
        q, k, v = qkv.view(B, T, 3, h, dh).unbind(2)
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        tf = bench(lambda: fa(q, k, v, causal=True))
        q.requires_grad_(); k.requires_grad_(); v.requires_grad_()
        y = fa(q, k, v, causal=True)
        g = torch.randn_like(y)
        tb = bench(lambda: torch.autograd.grad(y, (q, k, v), g, retain_graph=True))
        out.append(f"flash_attn2: fwd {fl/tf/1e9:6.1f} TF  bwd {2.5*fl/tb/1e9:6.1f} TF")
    print("  |  ".join(out), flush=True)
