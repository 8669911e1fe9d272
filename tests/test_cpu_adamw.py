"""libatom's CPU AdamW (host update placement, "CPU AdamW"; R37) against the
fp64 oracle (oracle/adamw.py), through the C-ABI test entry atom_k_cpu_adamw -- no GPU needed."""
import numpy as np

from oracle import adamw as oadamw
from paper_2403_10504_b200 import atom


def test_cpu_adamw_matches_oracle_over_steps():
    rng = np.random.default_rng(5)
    n = 300_001   # ragged against the worker split
    h = oadamw.AdamWHyper(lr=1e-3, warmup_steps=4)
    p = rng.normal(0, 0.02, n)
    m = np.zeros(n)
    v = np.zeros(n)
    p32, m32, v32 = p.astype(np.float32), m.astype(np.float32), v.astype(np.float32)
    R = 3
    for t in range(1, 7):
        gsum = rng.normal(0, 1e-2, n) * R
        p, m, v = oadamw.adamw_step(h, t, p, gsum / R, m, v)
        g32 = gsum.astype(np.float32)
        atom.k_cpu_adamw(p32, g32, m32, v32, oadamw.lr_at(h, t), h.beta1, h.beta2, h.eps, h.weight_decay, t,
                         gscale=1.0 / R, threads=7)
        # v carries the fp32 rounding of beta2 (1 - fp32(0.999) = 0.00099998713: 1.3e-5 relative),
        # as the GPU kernel does (the step parity tests allow 2e-4 on v)
        for a, b, tol in ((p32, p, 1e-5), (m32, m, 1e-5), (v32, v, 5e-5)):
            assert np.linalg.norm(a - b) <= tol * np.linalg.norm(b), t


def test_cpu_adamw_threads_do_not_change_bits():
    rng = np.random.default_rng(6)
    n = 1 << 18
    base = [rng.normal(0, 1, n).astype(np.float32) for _ in range(2)] + [np.abs(rng.normal(0, 1, n)).astype(np.float32)]
    outs = []
    for th in (1, 3, 16):
        p, g, v = (b.copy() for b in base)
        m = np.zeros(n, np.float32)
        atom.k_cpu_adamw(p, g, m, v, 1e-3, 0.9, 0.999, 1e-8, 0.01, 2, 0.5, th)
        outs.append((p, m, v))
    for o in outs[1:]:
        assert all(np.array_equal(a, b) for a, b in zip(o, outs[0]))
