"""Time the tcgen05 GEMM on the GPT-3 shapes (CUDA events, warm L2 excluded by size) vs torch.matmul."""
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
          ("lm_head", 16384, 50257, 2560, 0, 0), ("xl_qkv", 16384, 6144, 2048, 0, 0), ("sq8192", 8192, 8192, 8192, 0, 0)]
for name, M, N, K, amn, bmn in shapes:
    A = torch.randn((K, M) if amn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if bmn else (N, K), device="cuda").bfloat16()
    ld = (N + 7) // 8 * 8
    out = torch.empty(M, ld, device="cuda", dtype=torch.bfloat16)
    lda = M if amn else K
    ldb = N if bmn else K
    res = {}
    for bn in (0, 128, 256):
        f = lambda: atom.k_gemm(atom.IMPL_TC, atom.BF16, M, N, K, A.data_ptr(), lda, amn, B.data_ptr(), ldb, bmn,
                                atom.EPI_STORE, out.data_ptr(), ld, force_bn=bn)
        res[bn] = bench(f)
    At = A.T if amn else A
    Bt = B if bmn else B.T
    tt = bench(lambda: torch.matmul(At, Bt))
    fl = 2.0 * M * N * K
    print(f"{name:10s} M={M} N={N} K={K} auto {fl/res[0]/1e9:7.1f} TF  bn128 {fl/res[128]/1e9:7.1f}  bn256 {fl/res[256]/1e9:7.1f}  torch {fl/tt/1e9:7.1f} TF", flush=True)
