"""Plain fp64 GPT-3 forward and hand-written backward (TEST INFRASTRUCTURE ONLY).

The model is minGPT's pre-LN decoder ("We constructed the GPT-3
computation graph through ... minGPT"), written as the plain definition
(SURVEY §8(c) c.3):

  h0_t   = wte[x_t] + wpe[t]
  a      = LN(h; g1, b1)
  [q|k|v]= a W_qkv^T + b_qkv          heads j = columns j*dh .. (j+1)*dh-1
  S_ts   = q_t.k_s / sqrt(dh) (s <= t), -inf otherwise;  o_t = sum_s softmax_s(S)_ts v_s
  h     <- h + o W_o^T + b_o
  u      = LN(h; g2, b2) W_fc^T + b_fc
  h     <- h + GELU(u) W_pr^T + b_pr,   GELU = tanh approximation (minGPT NewGELU)
  z      = LN(h; gf, bf);  logits = z W_lm^T  (untied, no bias)
  loss   = mean over all tokens of (logsumexp(logits_t) - logits_t[y_t])
  LN(x)  = (x - mu) / sqrt(var + 1e-5) * g + b   (biased variance over d)

Dropout (minGPT sites) is off by default (``drop=None``,
the hot path's p = 0).  With ``drop = Dropout(p, seed, micro_step)`` the
minGPT sites are applied with the Philox keep-masks of oracle/philox.py (R38):

  h0 <- D_embd(h0);  o_t = sum_s D_attn(softmax(S))_ts v_s;
  h  <- h + D_resid_attn(o W_o^T + b_o);  h <- h + D_resid_mlp(GELU(u) W_pr^T + b_pr)

The gradient is the exact derivative of ``loss`` (for a fixed mask), computed by hand (chain
rule written out op by op).
"""
from __future__ import annotations

import math

import numpy as np

from . import philox

LN_EPS = 1e-5
GELU_C = math.sqrt(2.0 / math.pi)


# ----------------------------------------------------------------------------
# parameters: canonical order (SURVEY §8(b) "Parameter order")
# ----------------------------------------------------------------------------
BLOCK_NAMES = ["ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o",
               "ln2_g", "ln2_b", "w_fc", "b_fc", "w_pr", "b_pr"]


def block_shapes(d):
    return {"ln1_g": (d,), "ln1_b": (d,), "w_qkv": (3 * d, d), "b_qkv": (3 * d,),
            "w_o": (d, d), "b_o": (d,), "ln2_g": (d,), "ln2_b": (d,),
            "w_fc": (4 * d, d), "b_fc": (4 * d,), "w_pr": (d, 4 * d), "b_pr": (d,)}


def shapes(cfg):
    """[(node, name, shape)] in canonical order: E, B_0..B_{L-1}, H."""
    d = cfg.d_model
    out = [(0, "wte", (cfg.vocab, d)), (0, "wpe", (cfg.seq_len, d))]
    bs = block_shapes(d)
    for l in range(cfg.n_layer):
        out += [(1 + l, n, bs[n]) for n in BLOCK_NAMES]
    out += [(cfg.n_layer + 1, "lnf_g", (d,)), (cfg.n_layer + 1, "lnf_b", (d,)),
            (cfg.n_layer + 1, "w_lm", (cfg.vocab, d))]
    return out


def unflatten(cfg, flat, dtype=np.float64):
    """flat vector -> {"E": {...}, "B": [{...}], "H": {...}} (views into a copy of dtype: fp64 for
    parity; fp32 only for bench.py's cpu_baseline timing)."""
    flat = np.asarray(flat, dtype=dtype)
    p = {"E": {}, "B": [dict() for _ in range(cfg.n_layer)], "H": {}}
    off = 0
    for node, name, shp in shapes(cfg):
        n = int(np.prod(shp))
        t = flat[off:off + n].reshape(shp)
        off += n
        if node == 0:
            p["E"][name] = t
        elif node == cfg.n_layer + 1:
            p["H"][name] = t
        else:
            p["B"][node - 1][name] = t
    assert off == flat.size, (off, flat.size)
    return p


def flatten(cfg, p):
    parts = []
    for node, name, _ in shapes(cfg):
        if node == 0:
            parts.append(p["E"][name].ravel())
        elif node == cfg.n_layer + 1:
            parts.append(p["H"][name].ravel())
        else:
            parts.append(p["B"][node - 1][name].ravel())
    return np.concatenate(parts)


def node_ranges(cfg):
    """[(start, end)) of each node's parameters in the flat canonical vector."""
    r, off, cur, start = [], 0, 0, 0
    for node, _, shp in shapes(cfg):
        if node != cur:
            r.append((start, off))
            cur, start = node, off
        off += int(np.prod(shp))
    r.append((start, off))
    return r


# ----------------------------------------------------------------------------
# elementary ops (definitions, fp64)
# ----------------------------------------------------------------------------
def layernorm(x, g, b):
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xhat = (x - mu) * rstd
    return xhat * g + b, (xhat, rstd)


def layernorm_bwd(dy, g, cache):
    xhat, rstd = cache
    d = xhat.shape[-1]
    dg = (dy * xhat).reshape(-1, d).sum(axis=0)
    db = dy.reshape(-1, d).sum(axis=0)
    dxhat = dy * g
    dx = rstd * (dxhat - dxhat.mean(axis=-1, keepdims=True)
                 - xhat * (dxhat * xhat).mean(axis=-1, keepdims=True))
    return dx, dg, db


def gelu(u):
    return 0.5 * u * (1.0 + np.tanh(GELU_C * (u + 0.044715 * u ** 3)))


def gelu_grad(u):
    th = np.tanh(GELU_C * (u + 0.044715 * u ** 3))
    return 0.5 * (1.0 + th) + 0.5 * u * (1.0 - th ** 2) * GELU_C * (1.0 + 3 * 0.044715 * u ** 2)


class Dropout:
    """p in [0, 1); seed (uint64) and micro_step (uint32) select the Philox stream."""

    def __init__(self, p, seed, micro_step=0):
        assert 0.0 <= p < 1.0
        self.p, self.seed, self.micro_step = float(p), int(seed), int(micro_step)

    def scale(self, shape, site, layer):
        """fp64 multiplier (0 or 1/(1-p)) for one site tensor, or None when p = 0."""
        if self.p == 0.0:
            return None
        return philox.keep_scale(shape, self.p, site, layer, self.micro_step, self.seed)


def _apply(x, m):
    return x if m is None else x * m


def attention(q, k, v, m=None):
    """q, k, v: [B, h, T, dh] -> o [B, h, T, dh], probabilities A [B, h, T, T].
    m: the attention-dropout multiplier of A (None = no dropout)."""
    T, dh = q.shape[-2], q.shape[-1]
    s = q @ np.swapaxes(k, -1, -2) / math.sqrt(dh)
    mask = np.triu(np.ones((T, T), dtype=bool), k=1)
    s = np.where(mask, -np.inf, s)
    s = s - s.max(axis=-1, keepdims=True)
    e = np.exp(s)
    a = e / e.sum(axis=-1, keepdims=True)
    return _apply(a, m) @ v, a


def attention_bwd(do, q, k, v, a, m=None):
    dh = q.shape[-1]
    dv = np.swapaxes(_apply(a, m), -1, -2) @ do
    da = _apply(do @ np.swapaxes(v, -1, -2), m)
    ds = a * (da - (da * a).sum(axis=-1, keepdims=True))   # softmax Jacobian
    ds = ds / math.sqrt(dh)
    dq = ds @ k
    dk = np.swapaxes(ds, -1, -2) @ q
    return dq, dk, dv


def split_heads(x, h):
    B, T, d = x.shape
    return x.reshape(B, T, h, d // h).transpose(0, 2, 1, 3)


def merge_heads(x):
    B, h, T, dh = x.shape
    return x.transpose(0, 2, 1, 3).reshape(B, T, h * dh)


# ----------------------------------------------------------------------------
# model
# ----------------------------------------------------------------------------
def forward(cfg, p, tokens, want_cache=True, drop=None):
    """tokens [B, T+1] int -> (loss, logits, cache).  loss is the mean CE.
    drop: None (p = 0) or a Dropout (minGPT sites, Philox masks)."""
    x_ids = tokens[:, :-1]
    y_ids = tokens[:, 1:]
    B, T = x_ids.shape
    h = cfg.n_head
    E = p["E"]
    mk = (lambda shape, site, layer: None) if drop is None else drop.scale
    hcur = E["wte"][x_ids] + E["wpe"][np.arange(T)][None]
    m_embd = mk(hcur.shape, philox.SITE_EMBD, 0)
    hcur = _apply(hcur, m_embd)
    caches = []
    for li, blk in enumerate(p["B"]):
        x_in = hcur
        a, ln1c = layernorm(x_in, blk["ln1_g"], blk["ln1_b"])
        qkv = a @ blk["w_qkv"].T + blk["b_qkv"]
        d = cfg.d_model
        q, k, v = (split_heads(qkv[..., i * d:(i + 1) * d], h) for i in range(3))
        m_att = mk(q.shape[:3] + (q.shape[2],), philox.SITE_ATTN, li)
        o4, att = attention(q, k, v, m_att)
        o = merge_heads(o4)
        m_r1 = mk(x_in.shape, philox.SITE_RESID_ATTN, li)
        m_r2 = mk(x_in.shape, philox.SITE_RESID_MLP, li)
        x2 = x_in + _apply(o @ blk["w_o"].T + blk["b_o"], m_r1)
        a2, ln2c = layernorm(x2, blk["ln2_g"], blk["ln2_b"])
        u = a2 @ blk["w_fc"].T + blk["b_fc"]
        g = gelu(u)
        hcur = x2 + _apply(g @ blk["w_pr"].T + blk["b_pr"], m_r2)
        caches.append((x_in, a, ln1c, q, k, v, att, o, x2, a2, ln2c, u, g, m_att, m_r1, m_r2))
    H = p["H"]
    z, lnfc = layernorm(hcur, H["lnf_g"], H["lnf_b"])
    logits = z @ H["w_lm"].T
    mx = logits.max(axis=-1, keepdims=True)
    lse = (mx + np.log(np.exp(logits - mx).sum(axis=-1, keepdims=True)))[..., 0]
    tgt = np.take_along_axis(logits, y_ids[..., None], axis=-1)[..., 0]
    loss = float((lse - tgt).mean())
    cache = (x_ids, y_ids, caches, hcur, z, lnfc, logits, lse, m_embd) if want_cache else None
    return loss, logits, cache


def backward(cfg, p, cache):
    """Exact gradient of the mean CE loss w.r.t. every parameter (same structure as p)."""
    x_ids, y_ids, caches, hL, z, lnfc, logits, lse, m_embd = cache
    B, T = x_ids.shape
    n_tok = B * T
    h = cfg.n_head
    d = cfg.d_model
    H = p["H"]
    # d loss / d logits = (softmax - onehot) / n_tok
    dlogits = np.exp(logits - lse[..., None])
    np.put_along_axis(dlogits, y_ids[..., None],
                      np.take_along_axis(dlogits, y_ids[..., None], axis=-1) - 1.0, axis=-1)
    dlogits /= n_tok
    gH = {"w_lm": dlogits.reshape(-1, cfg.vocab).T @ z.reshape(-1, d)}
    dz = dlogits @ H["w_lm"]
    dh, gH["lnf_g"], gH["lnf_b"] = layernorm_bwd(dz, H["lnf_g"], lnfc)
    gB = [None] * cfg.n_layer
    for l in reversed(range(cfg.n_layer)):
        blk = p["B"][l]
        (x_in, a, ln1c, q, k, v, att, o, x2, a2, ln2c, u, g, m_att, m_r1, m_r2) = caches[l]
        gb = {}
        # h_out = x2 + D(g W_pr^T + b_pr)
        dy = _apply(dh, m_r2)
        gb["w_pr"] = dy.reshape(-1, d).T @ g.reshape(-1, 4 * d)
        gb["b_pr"] = dy.reshape(-1, d).sum(axis=0)
        dg = dy @ blk["w_pr"]
        du = dg * gelu_grad(u)
        gb["w_fc"] = du.reshape(-1, 4 * d).T @ a2.reshape(-1, d)
        gb["b_fc"] = du.reshape(-1, 4 * d).sum(axis=0)
        da2 = du @ blk["w_fc"]
        dx2_ln, gb["ln2_g"], gb["ln2_b"] = layernorm_bwd(da2, blk["ln2_g"], ln2c)
        dx2 = dh + dx2_ln
        # x2 = x_in + D(o W_o^T + b_o)
        dy = _apply(dx2, m_r1)
        gb["w_o"] = dy.reshape(-1, d).T @ o.reshape(-1, d)
        gb["b_o"] = dy.reshape(-1, d).sum(axis=0)
        do = dy @ blk["w_o"]
        dq, dk, dv = attention_bwd(split_heads(do, h), q, k, v, att, m_att)
        dqkv = np.concatenate([merge_heads(dq), merge_heads(dk), merge_heads(dv)], axis=-1)
        gb["w_qkv"] = dqkv.reshape(-1, 3 * d).T @ a.reshape(-1, d)
        gb["b_qkv"] = dqkv.reshape(-1, 3 * d).sum(axis=0)
        da = dqkv @ blk["w_qkv"]
        dx_ln, gb["ln1_g"], gb["ln1_b"] = layernorm_bwd(da, blk["ln1_g"], ln1c)
        dh = dx2 + dx_ln
        gB[l] = gb
    # embeddings: h0 = D(wte[x] + wpe[t])
    dh = _apply(dh, m_embd)
    dwte = np.zeros_like(p["E"]["wte"])
    np.add.at(dwte, x_ids.ravel(), dh.reshape(-1, d))
    dwpe = np.zeros_like(p["E"]["wpe"])
    dwpe[:T] = dh.sum(axis=0)
    return {"E": {"wte": dwte, "wpe": dwpe}, "B": gB, "H": gH}


def loss_and_grad(cfg, flat_params, tokens, drop=None, dtype=np.float64):
    """Flat-vector convenience wrapper: (loss, flat_grad) in fp64 (dtype=np.float32: the same
    arithmetic in fp32, used only to time the oracle as the CPU baseline)."""
    p = unflatten(cfg, flat_params, dtype)
    loss, _, cache = forward(cfg, p, np.asarray(tokens), drop=drop)
    g = backward(cfg, p, cache)
    return loss, flatten(cfg, g)


def loss_only(cfg, flat_params, tokens, drop=None):
    p = unflatten(cfg, flat_params)
    return forward(cfg, p, np.asarray(tokens), want_cache=False, drop=drop)[0]
