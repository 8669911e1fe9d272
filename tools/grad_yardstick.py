"""bf16 gradient accuracy: the CUDA path (atom_step, bf16) and PyTorch bf16 (tests/torch_gpt.py on
the GPU, the same step) against the fp64 oracle, per tensor.  Prints max and 99.9th-percentile of
|g - g_ref| / (|g_ref| + rms(g_ref)) and the relative L2 error for both."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import synth  # noqa: E402
from oracle import gpt as ogpt  # noqa: E402
from paper_2403_10504_b200 import atom  # noqa: E402
from torch_gpt import TorchGPT  # noqa: E402

CFGS = {
    "tiny": (synth.CONFIGS["tiny"], 2, [2, 5]),
    "mini": (synth.GPTConfig("mini", n_layer=3, d_model=128, n_head=2, seq_len=128, vocab=1000, micro_batch=2), 2,
             [1, 2, 4]),
    "wide": (synth.GPTConfig("wide-2.7b", n_layer=2, d_model=2560, n_head=32, seq_len=2048, vocab=50257,
                             micro_batch=1), 2, [1, 2, 3]),
}


def stats(g, ref, cfg):
    out = {}
    off = 0
    for node, name, shp in ogpt.shapes(cfg):
        n = int(np.prod(shp))
        x, y = g[off:off + n].astype(np.float64), ref[off:off + n]
        rms = float(np.sqrt(np.mean(y * y)))
        e = np.abs(x - y) / (np.abs(y) + rms + 1e-300)
        out[(node, name)] = (float(e.max()), float(np.quantile(e, 0.999)),
                             float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)))
        off += n
    return out


def main(names):
    for nm in names:
        g, C, ends = CFGS[nm]
        cfg = atom.make_cfg(g, dtype=atom.BF16, C_=C, overlap_check=0, forced_ends=ends, lr=1e-3, warmup_steps=0)
        plan = atom.atom_plan(cfg, 10 ** 12, 10 ** 10)
        init = synth.init_params(g, seed=1234, perturb=True)
        toks = synth.tokens(g, C * g.micro_batch, synth.step_seed(0, 0))
        peer = atom.Peer(cfg, plan, init_params=init)
        loss = peer.step(toks)
        ours = peer.params()["m"] / 0.1
        peer.destroy()
        ref_loss, ref = ogpt.loss_and_grad(g, init.astype(np.float64), toks)
        m = TorchGPT(g, init, dtype=torch.bfloat16, device="cuda")
        tl = m(torch.tensor(toks, dtype=torch.long, device="cuda"))
        tl.backward()
        tg = torch.cat([q.grad.reshape(-1).double() for q in m.params]).cpu().numpy()
        del m
        torch.cuda.empty_cache()
        so, st = stats(ours, ref, g), stats(tg, ref, g)
        print(f"== {nm}: loss ours {loss:.6f} torch-bf16 {tl.item():.6f} oracle {ref_loss:.6f}")
        print(f"{'tensor':22s} {'ours max':>9s} {'torch max':>9s} {'ours p999':>9s} {'torch p999':>10s} "
              f"{'ours relL2':>10s} {'torch relL2':>11s}")
        for k in so:
            a, b = so[k], st[k]
            print(f"{str(k):22s} {a[0]:9.3e} {b[0]:9.3e} {a[1]:9.3e} {b[1]:10.3e} {a[2]:10.3e} {b[2]:11.3e}")
        ratio = max(so[k][0] / max(st[k][0], 1e-30) for k in so)
        print(f"worst max-ratio ours/torch: {ratio:.3f}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["tiny", "mini", "wide"])
