"""Where the dK/dV kernel's time goes: clock64 stamps of the pipeline events of the heaviest CTAs
(key block 0 of the first 8 heads, 32 query blocks at T = 2048), from a build with -DATOM_DKV_TRACE=1
(tools/build_variant.py dkvtrace attn_tc.cu -DATOM_DKV_TRACE=1; ATOM_LIB=.../libatom_dkvtrace.so)."""
import ctypes
import sys

import numpy as np
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
IMPL = atom.ATTN_TC if os.environ.get("ATOM_BWD_ONLY") == "tc" else atom.ATTN_TC_DS
for _ in range(3):
    atom.k_attn_bwd(IMPL, atom.BF16, qkv.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(),
                    ds.data_ptr(), dqkv.data_ptr(), B, T, h, dh)
torch.cuda.synchronize()
tr = np.zeros((8, 12, 64, 4), dtype=np.uint64)
assert atom.lib.atom_k_dkv_trace(ctypes.c_void_p(tr.ctypes.data)) == 0
tr = tr.astype(np.int64)
nblk = 32
lo, hi = 4, 28   # steady state
def med(x):
    return float(np.median(np.array(x))) if len(x) else float("nan")
prod_wait, prod_load, mma_wait, mma_issue = [], [], [], []
ew = {"flush+gap": [], "st_full": [], "s_full": [], "compute": []}
cyc = []
for c in range(8):
    t = tr[c]
    base = t[0, 0, 0]
    for it in range(lo, hi):
        prod_wait.append(t[0, it, 1] - t[0, it, 0])
        prod_load.append(t[0, it, 2] - t[0, it, 1])
        mma_wait.append(t[1, it, 1] - t[1, it, 0])
        mma_issue.append(t[1, it, 2] - t[1, it, 1])
        cyc.append(t[1, it + 1, 1] - t[1, it, 1])
    for w in range(4, 12):
        wg = (w - 4) >> 2
        its = [i for i in range(lo, hi) if i % 2 == wg]
        for i in its:
            ew["st_full"].append(t[w, i, 1] - t[w, i, 0])
            ew["s_full"].append(t[w, i, 2] - t[w, i, 1])
            ew["compute"].append(t[w, i, 3] - t[w, i, 2])
            if i + 2 < nblk:
                ew["flush+gap"].append(t[w, i + 2, 0] - t[w, i, 3])
print(f"cycles per block (MMA p_full to p_full): median {med(cyc):.0f}")
print(f"producer: wait st_empty {med(prod_wait):.0f}, TMA issue + L/D loads + arrive {med(prod_load):.0f}")
print(f"MMA warp: wait p_full {med(mma_wait):.0f}, dV/dK issue + wait st_full + S^T/dP^T issue {med(mma_issue):.0f}")
print("elementwise warps (per own block, 2 blocks per cycle pair): " +
      ", ".join(f"{k} {med(v):.0f}" for k, v in ew.items()))
# one CTA's timeline for the first 8 blocks
t = tr[0]
b0 = t[1, 0, 0]
for it in range(8):
    w = 4 + (it % 2) * 4
    print(f"block {it}: prod empty-wait {t[0,it,0]-b0:7d}..{t[0,it,1]-b0:7d} arrive {t[0,it,2]-b0:7d} | "
          f"ew{w} st {t[w,it,0]-b0:7d}..{t[w,it,1]-b0:7d} s {t[w,it,2]-b0:7d} done {t[w,it,3]-b0:7d} | "
          f"mma p {t[1,it,0]-b0:7d}..{t[1,it,1]-b0:7d} next {t[1,it,2]-b0:7d}")
