"""Achieved HBM GB/s of atom_k_dropout at the 2.7B site shapes (CUDA events, warm, L2-sized inputs
exceeded).  Algorithmic bytes: 2 x sizeof(T) per element (read x, write y).  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2403_10504_b200 import atom

peaks = json.load(open("MEASURED_PEAKS.json"))
rows = []
for name, n, dt, tdt in [("resid_2.7B_bf16", 8 * 2048 * 2560, atom.BF16, torch.bfloat16),
                         ("attn_2.7B_bf16", 8 * 32 * 2048 * 2048, atom.BF16, torch.bfloat16),
                         ("resid_2.7B_fp32", 8 * 2048 * 2560, atom.FP32, torch.float32)]:
    x = torch.randn(n, device="cuda").to(tdt)
    y = torch.empty_like(x)
    for _ in range(3):
        atom.k_dropout(dt, x.data_ptr(), y.data_ptr(), n, 0.1, 1, 3, 0, 0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = 20
    torch.cuda.synchronize()
    s.record()
    for i in range(it):
        atom.k_dropout(dt, x.data_ptr(), y.data_ptr(), n, 0.1, 1, 3, 0, i)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / it
    gbs = 2 * x.element_size() * n / ms / 1e6
    rows.append({"site": name, "n": n, "us": round(ms * 1e3, 1), "GB/s": round(gbs, 1)})
print(json.dumps({"kernel": "dropout_kernel", "rows": rows, "peak": peaks}))
