"""Per-kernel device time of the attention backward (dsum, dK/dV, dQ) at the 2.7B shape, for the
recomputing dQ kernel (ATTN_TC) and the dQ-from-dS^T kernel (ATTN_TC_DS), from a CUPTI trace."""
import collections
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom  # noqa: E402

B, T, h, dh = 8, 2048, 32, 80
d = h * dh
qkv = (torch.randn(B * T, 3 * d, device="cuda") * 0.5).bfloat16()
o = torch.empty(B * T, d, device="cuda", dtype=torch.bfloat16)
do = torch.randn(B * T, d, device="cuda").bfloat16()
lse = torch.empty(B * h * T, device="cuda")
ds = torch.empty(B * h * T, device="cuda")
dqkv = torch.empty_like(qkv)
atom.k_attn_fwd(atom.ATTN_TC, atom.BF16, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, h, dh)
import os
IMPLS = [(atom.ATTN_TC, "recompute dQ"), (atom.ATTN_TC_DS, "dQ from dS^T")]
if os.environ.get("ATOM_BWD_ONLY"):   # "tc" or "ds": one path only (e.g. builds without the dS^T staging)
    IMPLS = IMPLS[:1] if os.environ["ATOM_BWD_ONLY"] == "tc" else IMPLS[1:]
for impl, nm in IMPLS:
    for _ in range(3):
        atom.k_attn_bwd(impl, atom.BF16, qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), ds.data_ptr(),
                        dqkv.data_ptr(), B, T, h, dh)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            atom.k_attn_bwd(impl, atom.BF16, qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(),
                            ds.data_ptr(), dqkv.data_ptr(), B, T, h, dh)
        torch.cuda.synchronize()
    prof.export_chrome_trace("/tmp/attn_bwd.json")
    ev = [e for e in json.load(open("/tmp/attn_bwd.json"))["traceEvents"] if e.get("cat") == "kernel"]
    tot = collections.defaultdict(float)
    for e in ev:
        tot[e["name"].split("(")[0]] += e["dur"] / 5
    print(nm, {k: round(v, 1) for k, v in tot.items()}, "sum us", round(sum(tot.values()), 1), flush=True)
