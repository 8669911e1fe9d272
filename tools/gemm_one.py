"""Run one GEMM shape a few times (for ncu): python tools/gemm_one.py M N K amn bmn force_bn"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom
M, N, K, amn, bmn, bn = map(int, sys.argv[1:7])
lda = (M + 7) // 8 * 8 if amn else (K + 7) // 8 * 8
ldb = (N + 7) // 8 * 8 if bmn else (K + 7) // 8 * 8
A = torch.randn((K, lda) if amn else (M, lda), device="cuda").bfloat16()
B = torch.randn((K, ldb) if bmn else (N, ldb), device="cuda").bfloat16()
out = torch.empty(M, (N + 7) // 8 * 8, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    atom.k_gemm(atom.IMPL_TC, atom.BF16, M, N, K, A.data_ptr(), lda, amn, B.data_ptr(), ldb, bmn, atom.EPI_STORE,
                out.data_ptr(), (N + 7) // 8 * 8, force_bn=bn)
torch.cuda.synchronize()
print("ok")
