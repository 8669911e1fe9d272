"""GPU parity of atom_k_dropout (R38) against the oracle's Philox masks.

The keep decision is integer work (a 16-bit Philox half against floor(p 2^16)): bit-exact.  fp32 values
match the fp64 oracle within 1e-6 relative (one fp32 product); bf16 values match a plain torch
fp32 product rounded to bf16 bit for bit.
"""
import numpy as np
import pytest
import torch

from oracle import philox

pytestmark = pytest.mark.gpu

from paper_2403_10504_b200 import atom  # noqa: E402

DEV = "cuda:0"
SEED = (0x0BADF00D << 32) | 0x12345678


def _run(x, p, site, layer, step, seed=SEED, out=None):
    y = torch.empty_like(x) if out is None else out
    dt = atom.FP32 if x.dtype == torch.float32 else atom.BF16
    atom.k_dropout(dt, x.data_ptr(), y.data_ptr(), x.numel(), p, seed, site, layer, step)
    torch.cuda.synchronize()
    return y


@pytest.mark.parametrize("n", [1, 3, 4, 8, 13, 4099, 1_000_003])
@pytest.mark.parametrize("p", [0.1, 0.5])
def test_fp32_matches_oracle(n, p):
    g = torch.Generator().manual_seed(n)
    x = torch.randn(n, generator=g, dtype=torch.float64)
    x[x == 0] = 1.0
    ref = x.numpy() * philox.keep_scale((n,), p, philox.SITE_RESID_ATTN, 7, 3, SEED)
    y = _run(x.float().to(DEV), p, philox.SITE_RESID_ATTN, 7, 3).double().cpu().numpy()
    assert np.array_equal(y == 0, ref == 0)
    np.testing.assert_allclose(y, ref, rtol=1e-6, atol=0)


@pytest.mark.parametrize("n", [5, 8 * 2 * 64 * 64 + 3])
def test_bf16_matches_torch_product_bitwise(n):
    p = 0.1
    g = torch.Generator().manual_seed(1)
    x = torch.randn(n, generator=g).to(torch.bfloat16)
    m = torch.tensor(philox.keep_scale((n,), p, philox.SITE_ATTN, 2, 0, SEED) != 0)
    scale = torch.tensor(1.0 / (1.0 - p), dtype=torch.float64).float()
    ref = torch.where(m, x.float() * scale, torch.zeros(())).to(torch.bfloat16)
    y = _run(x.to(DEV), p, philox.SITE_ATTN, 2, 0).cpu()
    assert torch.equal(y.view(torch.int16), ref.view(torch.int16))


def test_in_place_and_backward_reuse_the_mask():
    n, p = 10_007, 0.3
    x = torch.randn(n, device=DEV)
    y = _run(x, p, 3, 1, 4)
    z = x.clone()
    _run(z, p, 3, 1, 4, out=z)                       # in place
    assert torch.equal(y, z)
    dy = torch.randn(n, device=DEV)
    dx = _run(dy, p, 3, 1, 4)                        # backward = same multiplier
    assert torch.equal((dx == 0), (y == 0))


def test_p_zero_is_identity_and_empty_is_noop():
    x = torch.randn(4097, device=DEV)
    assert torch.equal(_run(x, 0.0, 0, 0, 0), x)
    e = torch.empty(0, device=DEV)
    _run(e, 0.5, 0, 0, 0)


def test_invalid_arguments_fail_loudly():
    x = torch.randn(16, device=DEV)
    for p in (1.0, -0.1):
        with pytest.raises(Exception):
            atom.k_dropout(atom.FP32, x.data_ptr(), x.data_ptr(), 16, p, 0, 0, 0, 0)
    with pytest.raises(Exception):                   # misaligned fp32 vector
        atom.k_dropout(atom.FP32, x.data_ptr() + 4, x.data_ptr() + 4, 8, 0.1, 0, 0, 0, 0)


@pytest.mark.parametrize("shape,site", [((8, 2048, 2560), philox.SITE_RESID_MLP),
                                        ((8, 32, 2048, 2048), philox.SITE_ATTN)],
                         ids=["resid_2.7B", "attn_2.7B"])
def test_full_size_sampled(shape, site):
    """2.7B site tensors (b = 8, T = 2048): sampled elements vs the oracle's Philox words, the
    keep rate of the whole tensor within 6 sigma (the attention site has > 2^30 elements)."""
    n = int(np.prod(shape))
    p, layer, step = 0.1, 31, 4
    x = torch.ones(n, dtype=torch.bfloat16, device=DEV)
    _run(x, p, site, layer, step, out=x)
    rng = np.random.default_rng(0)
    idx = np.concatenate([rng.integers(0, n, 4096), np.arange(n - 9, n), np.arange(0, 9)]).astype(np.uint64)
    w = philox.philox4x32_10((idx >> np.uint64(3), np.full_like(idx, site), np.full_like(idx, layer),
                              np.full_like(idx, step)), (SEED & 0xFFFFFFFF, SEED >> 32))
    words = np.stack(w, axis=-1)[np.arange(idx.size), ((idx >> np.uint64(1)) & np.uint64(3)).astype(np.int64)]
    halves = np.where(idx % np.uint64(2) == 1, words >> 16, words & 0xFFFF)
    keep_ref = halves >= int(np.floor(p * 2.0 ** 16))
    got = x[torch.tensor(idx.astype(np.int64), device=DEV)].cpu().float().numpy() != 0
    assert np.array_equal(got, keep_ref)
    dropped = n - int((x != 0).sum().item())
    p_eff = np.floor(p * 2.0 ** 16) / 2.0 ** 16      # the 16-bit threshold's drop probability
    sd = (n * p_eff * (1 - p_eff)) ** 0.5
    assert abs(dropped - n * p_eff) <= 6 * sd
