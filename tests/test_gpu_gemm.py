"""GEMM kernels (tcgen05 and SIMT) against a plain PyTorch fp32 reference, through the C-ABI."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2403_10504_b200 import atom  # noqa: E402

GELU_C = math.sqrt(2 / math.pi)


def gelu(u):
    return 0.5 * u * (1 + torch.tanh(GELU_C * (u + 0.044715 * u ** 3)))


def gelu_grad(u):
    th = torch.tanh(GELU_C * (u + 0.044715 * u ** 3))
    return 0.5 * (1 + th) + 0.5 * u * (1 - th * th) * GELU_C * (1 + 3 * 0.044715 * u * u)


def _operand(rows, K, mn, dt, gen):
    """logical [rows, K] and its storage (K-major [rows, K] or MN-major [K, rows_pad])."""
    x = torch.randn(rows, K, generator=gen, device="cuda").to(dt)
    if not mn:
        ld = (K + 7) // 8 * 8
        st = torch.zeros(rows, ld, device="cuda", dtype=dt)
        st[:, :K] = x
        return x, st, ld
    ld = (rows + 7) // 8 * 8
    st = torch.zeros(K, ld, device="cuda", dtype=dt)
    st[:, :rows] = x.T
    return x, st, ld


def _run(impl, dt, M, N, K, a_mn, b_mn, mode, force_bn=0, seed=0):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    A, As, lda = _operand(M, K, a_mn, dt, gen)
    B, Bs, ldb = _operand(N, K, b_mn, dt, gen)
    D = A.float() @ B.float().T
    ld = (N + 7) // 8 * 8
    out = torch.zeros(M, ld, device="cuda", dtype=torch.float32 if mode == atom.EPI_ACC_F32 else dt)
    out2 = torch.zeros(M, ld, device="cuda", dtype=dt)
    bias = (torch.randn(ld, generator=gen, device="cuda")).to(dt)
    res = torch.randn(M, ld, generator=gen, device="cuda").to(dt)
    aux = torch.randn(M, ld, generator=gen, device="cuda").to(dt)
    if mode == atom.EPI_ACC_F32:
        out.copy_(torch.randn(M, ld, generator=gen, device="cuda"))
    base = out.clone()
    dtype = atom.BF16 if dt == torch.bfloat16 else atom.FP32
    atom.k_gemm(impl, dtype, M, N, K, As.data_ptr(), lda, a_mn, Bs.data_ptr(), ldb, b_mn, mode, out.data_ptr(), ld,
                out2.data_ptr(), ld, bias.data_ptr(), res.data_ptr(), ld, aux.data_ptr(), ld, force_bn)
    torch.cuda.synchronize()
    b = bias[:N].float()
    if mode == atom.EPI_STORE:
        ref, got = D, out[:, :N].float()
    elif mode == atom.EPI_BIAS:
        ref, got = D + b, out[:, :N].float()
    elif mode == atom.EPI_BIAS_RES:
        ref, got = D + b + res[:, :N].float(), out[:, :N].float()
    elif mode == atom.EPI_BIAS_GELU:
        u = D + b
        ref = torch.cat([u, gelu(u)], 1)
        got = torch.cat([out[:, :N].float(), out2[:, :N].float()], 1)
    elif mode == atom.EPI_DGELU:
        ref, got = D * gelu_grad(aux[:, :N].float()), out[:, :N].float()
    else:
        ref, got = base[:, :N] + D, out[:, :N]
    # padding columns untouched
    if ld > N and mode != atom.EPI_ACC_F32:
        assert torch.all(out[:, N:] == 0)
    return ref, got


def _close(ref, got, dt, K):
    scale = ref.abs().max().item() + 1e-6
    err = (ref - got).abs().max().item()
    tol = (1e-5 * math.sqrt(K) if dt == torch.float32 else 1.2e-2) * scale
    assert err <= tol, (err, scale)


SHAPES = [(128, 256, 64), (256, 512, 192), (300, 200, 100), (1000, 776, 520), (2048, 2304, 768)]
MAJORS = [(False, False), (False, True), (True, True), (True, False)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("majors", MAJORS)
@pytest.mark.parametrize("bn", [128, 256, 512], ids=["1cta-128", "1cta-256", "2cta-256x256"])
def test_tc_gemm_store(shape, majors, bn):
    M, N, K = shape
    ref, got = _run(atom.IMPL_TC, torch.bfloat16, M, N, K, *majors, atom.EPI_STORE, bn)
    _close(ref, got, torch.bfloat16, K)


@pytest.mark.parametrize("mode", [atom.EPI_BIAS, atom.EPI_BIAS_RES, atom.EPI_BIAS_GELU, atom.EPI_DGELU,
                                  atom.EPI_ACC_F32])
@pytest.mark.parametrize("majors", [(False, False), (False, True), (True, True)])
@pytest.mark.parametrize("bn", [0, 512], ids=["auto", "2cta"])
def test_tc_gemm_epilogues(mode, majors, bn):
    M, N, K = 384, 520, 256
    ref, got = _run(atom.IMPL_TC, torch.bfloat16, M, N, K, *majors, mode, bn)
    _close(ref, got, torch.bfloat16, K)


def test_tc_gemm_large_ragged_vocab():
    """lm_head shape class: N = 50257 (odd), row pitch padded to a multiple of 8."""
    M, N, K = 512, 50257, 768
    ref, got = _run(atom.IMPL_TC, torch.bfloat16, M, N, K, False, False, atom.EPI_STORE)
    _close(ref, got, torch.bfloat16, K)


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("mode", [atom.EPI_STORE, atom.EPI_BIAS_RES, atom.EPI_BIAS_GELU, atom.EPI_DGELU,
                                  atom.EPI_ACC_F32])
@pytest.mark.parametrize("majors", MAJORS)
def test_simt_gemm(dt, mode, majors):
    M, N, K = 133, 97, 71
    ref, got = _run(atom.IMPL_SIMT, dt, M, N, K, *majors, mode)
    _close(ref, got, dt, K)


def test_tc_gemm_deterministic():
    M, N, K = 1024, 1024, 1024
    gen = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(M, K, generator=gen, device="cuda").bfloat16()
    B = torch.randn(N, K, generator=gen, device="cuda").bfloat16()
    outs = []
    for _ in range(2):
        o = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        atom.k_gemm(atom.IMPL_TC, atom.BF16, M, N, K, A.data_ptr(), K, 0, B.data_ptr(), K, 0, atom.EPI_STORE,
                    o.data_ptr(), N)
        outs.append(o)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


_SPLITK_CHILD = r"""
import sys, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from paper_2403_10504_b200 import atom
import test_gpu_gemm as t
M, N, K, amn, bmn = {args}
ref, got = t._run(atom.IMPL_TC, torch.bfloat16, M, N, K, amn, bmn, atom.EPI_ACC_F32, 512)
t._close(ref, got, torch.bfloat16, K)
ref2, got2 = t._run(atom.IMPL_TC, torch.bfloat16, M, N, K, amn, bmn, atom.EPI_ACC_F32, 512)
assert torch.equal(got, got2)
log = atom.launch_log()
assert any(k.startswith("gemm_tc2_splitk<") for k in log), log
print("splitk ok")
"""


# ragged: 11 x 9 = 99 tiles of 256 x 256 on 74 CTA pairs, a 25-tile tail split in two (ragged M and N)
@pytest.mark.parametrize("shape", [(3840, 2560, 2048), (4096, 4096, 1024), (2560 + 200, 2048 + 52, 1536)],
                         ids=["tail2-P8", "tail34-P2", "ragged"])
@pytest.mark.parametrize("majors", [(True, True), (False, False)], ids=["wgrad", "kmajor"])
def test_tc_gemm_acc_f32_streamk_tail(shape, majors):
    """Weight-gradient GEMMs (fp32 accumulate) whose last wave is split along K (stream-K tail,
    gemm_tc.cu SplitK, off by default; ATOM_GEMM_SPLITK=1 is read once per process, so the check
    runs in a child process with it set): same result as the unsplit math within fp32 rounding,
    deterministic, and the launch log proves the split kernel ran."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _SPLITK_CHILD.format(root=root, tests=os.path.join(root, "tests"), args=(*shape, *majors))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, ATOM_GEMM_SPLITK="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "splitk ok" in r.stdout, r.stdout + r.stderr
