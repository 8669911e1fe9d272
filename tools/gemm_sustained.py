"""Sustained (power-capped) GEMM throughput: each 2.7B step shape run back to back for ~1.5 s, ours
(tcgen05, automatic tile choice, the step's epilogue-free store) vs torch.matmul (cuBLAS), with the
SM clock sampled by nvidia-smi during each run -> TF/s and TF/s per GHz."""
import statistics
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2403_10504_b200 import atom  # noqa: E402


class Clock:
    def __enter__(self):
        self.p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                                   "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        self.v = []
        self.t = threading.Thread(target=lambda: [self.v.append(l) for l in self.p.stdout], daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.p.terminate()

    def mhz(self):
        xs = [float(l.split(",")[0]) for l in self.v[2:] if l.strip()]
        pw = [float(l.split(",")[1]) for l in self.v[2:] if l.strip()]
        return (statistics.median(xs) if xs else float("nan")), (statistics.median(pw) if pw else float("nan"))


def run(fn, secs=1.5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n, t0 = 0, time.time()
    with Clock() as c:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        while time.time() - t0 < secs:
            for _ in range(10):
                fn()
            n += 10
            torch.cuda.synchronize()
        e.record()
        torch.cuda.synchronize()
    mhz, pw = c.mhz()
    return s.elapsed_time(e) / n, mhz, pw


D, M = 2560, 16384
shapes = [("qkv", M, 3 * D, D, 0, 0), ("proj", M, D, D, 0, 0), ("fc", M, 4 * D, D, 0, 0), ("fc2", M, D, 4 * D, 0, 0),
          ("dgrad_qkv", M, D, 3 * D, 0, 1), ("dgrad_proj", M, D, D, 0, 1), ("dgrad_fc", M, 4 * D, D, 0, 1),
          ("dgrad_fc2", M, D, 4 * D, 0, 1), ("wgrad_qkv", 3 * D, D, M, 1, 1), ("wgrad_proj", D, D, M, 1, 1),
          ("wgrad_fc", 4 * D, D, M, 1, 1), ("wgrad_fc2", D, 4 * D, M, 1, 1), ("sq8192", 8192, 8192, 8192, 0, 0)]
only = sys.argv[1:]
for name, Mg, N, K, amn, bmn in shapes:
    if only and name not in only:
        continue
    lda = (Mg + 7) // 8 * 8 if amn else K
    ldb = (N + 7) // 8 * 8 if bmn else K
    A = torch.randn((K, lda) if amn else (Mg, lda), device="cuda").bfloat16()
    B = torch.randn((K, ldb) if bmn else (N, ldb), device="cuda").bfloat16()
    out = torch.empty(Mg, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * Mg * N * K
    ours = run(lambda: atom.k_gemm(atom.IMPL_TC, atom.BF16, Mg, N, K, A.data_ptr(), lda, amn, B.data_ptr(), ldb, bmn,
                                   atom.EPI_STORE, out.data_ptr(), N))
    At = A[:, :Mg].T if amn else A
    Bt = B[:, :N] if bmn else B.T
    cub = run(lambda: torch.matmul(At, Bt, out=out))
    print(f"{name:11s} {Mg:6d} {N:6d} {K:6d}  ours {fl / ours[0] / 1e9:7.1f} TF/s @ {ours[1]:6.0f} MHz {ours[2]:5.0f} W "
          f"({fl / ours[0] / 1e9 / ours[1] * 1000:6.1f} TF/s/GHz)   cuBLAS {fl / cub[0] / 1e9:7.1f} @ {cub[1]:6.0f} MHz "
          f"{cub[2]:5.0f} W ({fl / cub[0] / 1e9 / cub[1] * 1000:6.1f}/GHz)", flush=True)
    del A, B, out
