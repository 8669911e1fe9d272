"""An independently written minGPT-style torch module (torch.nn.functional ops), test-only.

Used two ways: in fp64 on the CPU as the library-routine pin of the oracle's hand-written backward
(tests/test_oracle_gpt.py), and in bf16 on the GPU as the yardstick of what bf16 arithmetic does to
the gradient (tests/test_gpu_fullwidth_oracle.py): the CUDA path's bf16 gradient error against the
fp64 oracle must stay within a small factor of PyTorch's own bf16 error on the same step.
"""
import numpy as np
import torch
import torch.nn.functional as F

import synth


class TorchGPT(torch.nn.Module):
    """An independently written minGPT-style module (torch.nn.functional ops)."""

    def __init__(self, cfg, flat, dtype=torch.float64, device="cpu"):
        super().__init__()
        self.cfg = cfg
        t = torch.tensor(flat, dtype=torch.float64).to(device=device, dtype=dtype)
        self.params = torch.nn.ParameterList()
        self.names = []
        off = 0
        for node, name, shp, _ in synth.param_layout(cfg):
            n = int(np.prod(shp))
            self.params.append(torch.nn.Parameter(t[off:off + n].reshape(shp).clone()))
            self.names.append((node, name))
            off += n

    def get(self, node, name):
        return self.params[self.names.index((node, name))]

    def forward(self, toks):
        cfg = self.cfg
        x, y = toks[:, :-1], toks[:, 1:]
        B, T = x.shape
        d, h = cfg.d_model, cfg.n_head
        hcur = F.embedding(x, self.get(0, "wte")) + self.get(0, "wpe")[:T]
        for l in range(cfg.n_layer):
            n = l + 1
            a = F.layer_norm(hcur, (d,), self.get(n, "ln1_g"), self.get(n, "ln1_b"), eps=1e-5)
            qkv = F.linear(a, self.get(n, "w_qkv"), self.get(n, "b_qkv"))
            q, k, v = qkv.split(d, dim=-1)
            q, k, v = (t_.view(B, T, h, d // h).transpose(1, 2) for t_ in (q, k, v))
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            o = o.transpose(1, 2).reshape(B, T, d)
            hcur = hcur + F.linear(o, self.get(n, "w_o"), self.get(n, "b_o"))
            a2 = F.layer_norm(hcur, (d,), self.get(n, "ln2_g"), self.get(n, "ln2_b"), eps=1e-5)
            u = F.linear(a2, self.get(n, "w_fc"), self.get(n, "b_fc"))
            hcur = hcur + F.linear(F.gelu(u, approximate="tanh"), self.get(n, "w_pr"), self.get(n, "b_pr"))
        L1 = cfg.n_layer + 1
        z = F.layer_norm(hcur, (d,), self.get(L1, "lnf_g"), self.get(L1, "lnf_b"), eps=1e-5)
        logits = F.linear(z, self.get(L1, "w_lm"))
        return F.cross_entropy(logits.reshape(-1, cfg.vocab), y.reshape(-1))
