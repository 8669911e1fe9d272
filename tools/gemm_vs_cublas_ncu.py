"""One GEMM shape through libatom's tcgen05 kernel and through cuBLAS (torch.matmul), for an ncu capture
comparing L2 / DRAM traffic, cluster shape and tensor-pipe activity:
    ncu --metrics ... python tools/gemm_vs_cublas_ncu.py M N K"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom  # noqa: E402

M, N, K = (int(a) for a in sys.argv[1:4])
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    atom.k_gemm(atom.IMPL_TC, atom.BF16, M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, atom.EPI_STORE,
                out.data_ptr(), N)
    torch.matmul(A, B.t(), out=out)
torch.cuda.synchronize()
print("ok")
