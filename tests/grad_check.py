"""bf16 gradient check against the fp64 oracle (test helper; DESIGN.md §3 "bf16 gradient bound").

The bf16 path stores weights and activations in bf16 (unit roundoff 2^-9) and accumulates in fp32;
every gradient element passes through a chain of such roundings from the loss, so its error is a
few 2^-9 relative to the scale of the terms that make it up, not to its own (possibly cancelled)
value.  Two bars per tensor, both against the oracle's exact gradient g_ref:

* REL_L2 = 2^-6: ||g - g_ref|| / ||g_ref||.  PyTorch's own bf16 step of the same model (tests/
  torch_gpt.py on the GPU) measured 4e-3 .. 1.35e-2 on tiny / mini / full-width (tools/
  grad_yardstick.py, profiles/r02_grad_yardstick.txt); the CUDA path 3.7e-3 .. 1.29e-2.
* ELEM = 2^-2: every element |g - g_ref| <= ELEM (|g_ref| + s), s = the rms of g_ref over the
  tensor's non-zero rows (the embedding gradient has a row per vocabulary entry, most of them
  exactly zero in both; a 1-D tensor is one row).  Measured worst: 0.17 (full-width lm_head;
  PyTorch bf16: 0.18); a sign flip of any element with |g_ref| >= s / 3, or a dropped term,
  exceeds it.

A gradient that is wrong (a dropped term, a transposed operand, a wrong scale) fails the first bar
by orders of magnitude; the second catches localised errors the norm would hide.
"""
import numpy as np

from oracle import gpt as ogpt

REL_L2 = 2.0 ** -6
ELEM = 2.0 ** -2


def gradient_errors(g, g_ref, cfg):
    """{(node, name): (max element-wise normalised error, relative L2 error)}"""
    out = {}
    off = 0
    for node, name, shp in ogpt.shapes(cfg):
        n = int(np.prod(shp))
        x = np.asarray(g[off:off + n], dtype=np.float64).reshape(shp)
        y = np.asarray(g_ref[off:off + n], dtype=np.float64).reshape(shp)
        y2 = y.reshape(shp[0], -1) if len(shp) == 2 else y.reshape(1, -1)
        rows = y2[np.any(y2 != 0, axis=1)]
        s = float(np.sqrt(np.mean(rows * rows))) if rows.size else 0.0
        elem = float(np.max(np.abs(x - y) / (np.abs(y) + s + 1e-300)))
        rel = float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))
        out[(node, name)] = (elem, rel)
        off += n
    return out


def check_bf16_gradient(g, g_ref, cfg):
    errs = gradient_errors(g, g_ref, cfg)
    we = max(errs.items(), key=lambda kv: kv[1][0])
    wr = max(errs.items(), key=lambda kv: kv[1][1])
    assert we[1][0] <= ELEM, ("element-wise", we)
    assert wr[1][1] <= REL_L2, ("relative L2", wr)
    return errs
