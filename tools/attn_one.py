"""One causal attention forward + backward (tcgen05 path) at B T h dh, for ncu captures:
python tools/attn_one.py 8 2048 16 128"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom

B, T, h, dh = (int(a) for a in sys.argv[1:5])
impl = int(sys.argv[5]) if len(sys.argv) > 5 else atom.ATTN_TC
d = h * dh
qkv = (torch.randn(B * T, 3 * d, device="cuda") * 0.5).bfloat16()
o = torch.empty(B * T, d, device="cuda", dtype=torch.bfloat16)
do = torch.randn(B * T, d, device="cuda").bfloat16()
lse = torch.empty(B * h * T, device="cuda")
ds = torch.empty(B * h * T, device="cuda")
dqkv = torch.empty_like(qkv)
atom.k_attn_fwd(impl, atom.BF16, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, h, dh)
atom.k_attn_bwd(impl, atom.BF16, qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), ds.data_ptr(),
                dqkv.data_ptr(), B, T, h, dh)
torch.cuda.synchronize()
print("ok", float(o.float().abs().mean()), float(dqkv.float().abs().mean()))
