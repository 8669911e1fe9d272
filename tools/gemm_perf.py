"""Time the tcgen05 GEMM variants on the GPT-3 shapes (CUDA events) vs torch.matmul (cuBLAS)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom

def bench(fn, it=20):
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it

shapes = [("qkv", 16384, 7680, 2560, 0, 0), ("proj", 16384, 2560, 2560, 0, 0), ("fc", 16384, 10240, 2560, 0, 0),
          ("fc2", 16384, 2560, 10240, 0, 0), ("dgrad_fc", 16384, 2560, 10240, 0, 1), ("wgrad_fc", 10240, 2560, 16384, 1, 1),
          ("wgrad_qkv", 7680, 2560, 16384, 1, 1), ("lm_head", 16384, 50257, 2560, 0, 0), ("lm_dgrad", 16384, 2560, 50257, 0, 1),
          ("lm_wgrad", 50257, 2560, 16384, 1, 1), ("xl_qkv", 16384, 6144, 2048, 0, 0), ("xl_proj", 16384, 2048, 2048, 0, 0),
          ("sq8192", 8192, 8192, 8192, 0, 0)]
for name, M, N, K, amn, bmn in shapes:
    lda = (M + 7) // 8 * 8 if amn else (K + 7) // 8 * 8
    ldb = (N + 7) // 8 * 8 if bmn else (K + 7) // 8 * 8
    A = torch.randn((K, lda) if amn else (M, lda), device="cuda").bfloat16()
    B = torch.randn((K, ldb) if bmn else (N, ldb), device="cuda").bfloat16()
    ld = (N + 7) // 8 * 8
    out = torch.empty(M, ld, device="cuda", dtype=torch.bfloat16)
    res = {}
    for bn in (0, 128, 256, 512):
        f = lambda: atom.k_gemm(atom.IMPL_TC, atom.BF16, M, N, K, A.data_ptr(), lda, amn, B.data_ptr(), ldb, bmn,
                                atom.EPI_STORE, out.data_ptr(), ld, force_bn=bn)
        res[bn] = bench(f)
    At = A[:, :M].T if amn else A[:, :K]
    Bt = B[:, :N] if bmn else B[:, :K].T
    tt = bench(lambda: torch.matmul(At, Bt))
    fl = 2.0 * M * N * K
    print(f"{name:10s} M={M} N={N} K={K} auto {fl/res[0]/1e9:7.1f} TF  1cta128 {fl/res[128]/1e9:7.1f}  1cta256 {fl/res[256]/1e9:7.1f}  2cta {fl/res[512]/1e9:7.1f}  torch {fl/tt/1e9:7.1f}", flush=True)
