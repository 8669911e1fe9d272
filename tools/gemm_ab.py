"""Time a few GEMM shapes (auto tile choice) with CUDA events, many iterations: A/B of library variants
(ATOM_LIB). python tools/gemm_ab.py"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom

shapes = [("dgrad_fc", 16384, 2560, 10240, 0, 1), ("fc2", 16384, 2560, 10240, 0, 0),
          ("dgrad_qkv", 16384, 2560, 7680, 0, 1), ("dgrad_pr", 16384, 10240, 2560, 0, 1)]
for name, M, N, K, amn, bmn in shapes:
    lda = K
    ldb = N if bmn else K
    A = torch.randn(M, lda, device="cuda").bfloat16()
    B = torch.randn((K, ldb) if bmn else (N, ldb), device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    f = lambda: atom.k_gemm(atom.IMPL_TC, atom.BF16, M, N, K, A.data_ptr(), lda, amn, B.data_ptr(), ldb, bmn,
                            atom.EPI_STORE, out.data_ptr(), N)
    for _ in range(5):
        f()
    res = []
    for rep in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(20):
            f()
        e.record()
        torch.cuda.synchronize()
        res.append(2.0 * M * N * K / (s.elapsed_time(e) / 20) / 1e9)
    print(f"{name} {min(res):.0f} {sorted(res)[2]:.0f} {max(res):.0f}", flush=True)
