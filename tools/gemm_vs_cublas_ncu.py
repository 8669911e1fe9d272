"""One GEMM shape through libatom's tcgen05 kernel and through cuBLAS (torch.matmul), for an ncu capture
comparing L2 / DRAM traffic, cluster shape and tensor-pipe activity:
    ncu --metrics ... python tools/gemm_vs_cublas_ncu.py M N K [a_mn b_mn]
(a_mn / b_mn = 1: the operand is stored K-rows-outer, M / N contiguous, as the weight gradients read
dY^T and X)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom  # noqa: E402

M, N, K = (int(a) for a in sys.argv[1:4])
amn, bmn = (int(a) for a in sys.argv[4:6]) if len(sys.argv) > 5 else (0, 0)
A = torch.randn((K, M) if amn else (M, K), device="cuda").bfloat16()
B = torch.randn((K, N) if bmn else (N, K), device="cuda").bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
At = A.T if amn else A          # [M, K]
Bt = B if bmn else B.T          # [K, N]
for _ in range(2):
    atom.k_gemm(atom.IMPL_TC, atom.BF16, M, N, K, A.data_ptr(), M if amn else K, amn, B.data_ptr(), N if bmn else K,
                bmn, atom.EPI_STORE, out.data_ptr(), N)
    torch.matmul(At, Bt, out=out)
torch.cuda.synchronize()
print("ok")
