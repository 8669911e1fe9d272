"""Parity at BASELINE.json's full sizes (GPT-3 2.7B: d = 2560, 32 heads x 80, T = 2048, b = 8),
in the launch configuration bench.py times, on sampled outputs or through properties that hold at
any size:

* the tcgen05 GEMMs at every 2.7B block shape and operand layout (forward, data gradient, weight
  gradient; automatic tile choice = the bench's), sampled entries vs fp64 dot products of the
  same bf16 operands;
* the tcgen05 attention forward and backward at (8, 2048, 32, 80), two sampled heads vs the
  fp32 PyTorch reference of those heads;
* a whole 2.7B training step: the bench's 11-sub-model partition vs the resident model (S = 1),
  three steps with the same tokens -- bit-identical losses (every parameter after the first two
  updates feeds the next loss), and the first loss at its closed form ln V + var(logits) / 2
  for the minGPT init (logits of a unit-variance LN output through N(0, 0.02^2) weights).
"""
import math

import pytest
import torch

import synth
from paper_2403_10504_b200 import atom

pytestmark = pytest.mark.gpu

G27 = synth.CONFIGS["2.7b"]
M, D = 8 * 2048, 2560
GEMMS = [  # name, M, N, K, a_mn, b_mn (the block's GEMMs and their gradients at 2.7B)
    ("qkv", M, 3 * D, D, False, False), ("proj", M, D, D, False, False), ("fc", M, 4 * D, D, False, False),
    ("fc2", M, D, 4 * D, False, False), ("dgrad_qkv", M, D, 3 * D, False, True),
    ("dgrad_fc2", M, 4 * D, D, False, True), ("wgrad_fc", 4 * D, D, M, True, True),
    ("wgrad_qkv", 3 * D, D, M, True, True), ("lm_head", M, 50257, D, False, False)]


@pytest.mark.parametrize("name,Mg,N,K,amn,bmn", GEMMS, ids=[g[0] for g in GEMMS])
def test_gemm_full_size_sampled(name, Mg, N, K, amn, bmn):
    gen = torch.Generator(device="cuda").manual_seed(11)
    lda = (Mg + 7) // 8 * 8 if amn else K
    ldb = (N + 7) // 8 * 8 if bmn else K
    A = torch.randn((K, lda) if amn else (Mg, lda), generator=gen, device="cuda").bfloat16()
    B = torch.randn((K, ldb) if bmn else (N, ldb), generator=gen, device="cuda").bfloat16()
    ld = (N + 7) // 8 * 8
    out = torch.zeros(Mg, ld, device="cuda", dtype=torch.bfloat16)
    atom.k_gemm(atom.IMPL_TC, atom.BF16, Mg, N, K, A.data_ptr(), lda, amn, B.data_ptr(), ldb, bmn, atom.EPI_STORE,
                out.data_ptr(), ld)
    torch.cuda.synchronize()
    rows = torch.randint(0, Mg, (64,), generator=gen, device="cuda")
    cols = torch.randint(0, N, (64,), generator=gen, device="cuda")
    Ar = (A[:, rows].T if amn else A[rows, :K]).double()          # [64, K]
    Bc = (B[:, cols] if bmn else B[cols, :K].T).double()          # [K, 64]
    ref = Ar @ Bc                                                  # all 64 x 64 pairs
    got = out[rows][:, cols].double()
    # per entry: the bf16 rounding of the output (half an ulp: 2^-9 relative, 4e-3 with margin)
    # plus fp32 accumulation error over K unit-variance products
    excess = (got - ref).abs() - (4e-3 * ref.abs() + 5e-4 * math.sqrt(K))
    assert excess.max().item() <= 0, (name, excess.max().item())


def _ref_heads(qkv, B, T, h, dh, heads, dout=None):
    x = qkv.float().view(B, T, 3, h, dh)[:, :, :, heads]           # [B, T, 3, nh, dh]
    x = x.detach().requires_grad_(dout is not None)
    q, k, v = (x[:, :, i].transpose(1, 2) for i in range(3))
    s = q @ k.transpose(-1, -2) / math.sqrt(dh)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=qkv.device), 1)
    s = s.masked_fill(mask, float("-inf"))
    o = torch.softmax(s, -1) @ v                                    # [B, nh, T, dh]
    lse = torch.logsumexp(s, -1)
    gq = None
    if dout is not None:
        do = dout.float().view(B, T, h, dh)[:, :, heads].transpose(1, 2)
        o.backward(do)
        gq = x.grad                                                 # [B, T, 3, nh, dh]
    return o.transpose(1, 2), lse, gq


def test_attention_full_size_sampled_heads():
    B, T, h, dh = 8, 2048, 32, 80
    gen = torch.Generator(device="cuda").manual_seed(12)
    qkv = (torch.randn(B * T, 3 * h * dh, generator=gen, device="cuda")).bfloat16()
    dout = torch.randn(B * T, h * dh, generator=gen, device="cuda").bfloat16()
    o = torch.zeros(B * T, h * dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(B, h, T, device="cuda")
    dsum = torch.zeros(B, h, T, device="cuda")
    dqkv = torch.zeros(B * T, 3 * h * dh, device="cuda", dtype=torch.bfloat16)
    atom.k_attn_fwd(atom.ATTN_TC, atom.BF16, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, h, dh)
    atom.k_attn_bwd(atom.ATTN_TC, atom.BF16, qkv.data_ptr(), o.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                    dsum.data_ptr(), dqkv.data_ptr(), B, T, h, dh)
    torch.cuda.synchronize()
    heads = [0, 29]
    ro, rl, gq = _ref_heads(qkv, B, T, h, dh, heads, dout)
    got_o = o.float().view(B, T, h, dh)[:, :, heads]
    assert (got_o - ro).abs().max().item() < 2e-2 * max(1.0, ro.abs().max().item())
    assert (lse[:, heads] - rl).abs().max().item() < 2e-2
    got_g = dqkv.float().view(B, T, 3, h, dh)[:, :, :, heads]
    err = (got_g - gq).abs().max().item()
    assert err < 3e-2 * max(1.0, gq.abs().max().item()), err


def _peer_27b(ends, C):
    cfg = atom.make_cfg(G27, dtype=atom.BF16, C_=C, overlap_check=0, forced_ends=ends, lr=1e-4, warmup_steps=0)
    plan = atom.atom_plan(cfg, 178 * 10 ** 9, 50 * 10 ** 9)
    return atom.Peer(cfg, plan, device=0, init_params=None, seed=1234)


def test_27b_swapped_equals_resident_and_initial_loss():
    C = 1
    toks = [synth.tokens(G27, C * G27.micro_batch, synth.step_seed(0, s)) for s in range(3)]
    runs = {}
    for name, ends in (("resident", None), ("swapped", [4, 7, 10, 13, 16, 19, 22, 25, 28, 31, 33])):
        p = _peer_27b(ends, C)
        assert p.plan.n_seg == (1 if ends is None else len(ends))
        runs[name] = [p.step(t) for t in toks]
        p.destroy()
        del p
        torch.cuda.empty_cache()
    assert runs["swapped"] == runs["resident"], runs
    # minGPT init: LN output ~ unit variance per feature, lm_head ~ N(0, 0.02^2): logits ~ N(0, s2),
    # s2 = 0.02^2 d; E[CE] = E[logsumexp] - E[z_y] ~ ln V + s2 / 2 for small s2 (targets independent)
    s2 = 0.02 ** 2 * G27.d_model
    want = math.log(G27.vocab) + s2 / 2
    assert abs(runs["resident"][0] - want) < 0.02 * want, (runs["resident"][0], want)
