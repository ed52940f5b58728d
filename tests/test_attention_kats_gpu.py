"""Stage-(d) known answers:

* an all-ones mask is dense attention (fp32 path within 1e-6 of a float64
  evaluation of the same formula);
* uniform logits (Q = 0) give the plain average of V over the active keys,
  padded (zero) keys included -- the "two keys -> their average" answer
  generalised to any block mask (fp32 within 1e-6, bf16 within one bf16 ulp
  of the fp32 average);
* exact and soft variants coincide on an all-ones mask.
"""
import numpy as np
import pytest
import torch

from oracle import pyoracle
from paper_2604_20470_b200 import radialplan as rp

pytestmark = pytest.mark.gpu


def _dense_f64(q, k, v, Sp):
    S, H, d = q.shape
    pad = lambda x: np.concatenate([x, np.zeros((Sp - S, H, d), x.dtype)]).astype(np.float64)
    qp, kp, vp = pad(q), pad(k), pad(v)
    out = np.empty((Sp, H, d))
    for h in range(H):
        lg = (qp[:, h] @ kp[:, h].T) / np.sqrt(d)
        lg -= lg.max(axis=1, keepdims=True)
        p = np.exp(lg)
        out[:, h] = (p @ vp[:, h]) / p.sum(axis=1, keepdims=True)
    return out


def test_all_ones_mask_is_dense(cuda, port):
    nf, nt, bs, H, d = 3, 100, 32, 2, 32
    q, k, v = port.random_batch(nf * nt, H, d, 3, threads=2)
    g = rp.make_grid(nf, nt, bs)
    m = rp.BlockMask(g.blocks_per_dim)
    for r in range(g.blocks_per_dim):
        for c in range(g.blocks_per_dim):
            m.set(r, c)
    ex = rp.masked_attention_exact(g, m, q, k, v)
    want = _dense_f64(q, k, v, g.padded_tokens)
    assert np.abs(ex - want).max() < 1e-6
    soft = rp.masked_attention(g, m, q, k, v, epsilon=1e-10)
    assert np.abs(soft - ex).max() < 1e-6


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_uniform_logits_average_active_values(cuda, port, dtype):
    nf, nt, H = 4, 300, 2
    bs, d = (32, 32) if dtype == "f32" else (128, 64)
    g = rp.make_grid(nf, nt, bs)
    cfg = pyoracle.Cfg(0, 1.0, 0.5, 1e-6, 0.75, 0.2, 0.4, 0.4)
    bits = port.build_mask(nf, nt, bs, cfg, 11)
    dense = pyoracle.unpack_bits(bits, g.blocks_per_dim)
    _, _, v = port.random_batch(nf * nt, H, d, 8, threads=2)
    q = np.zeros_like(v)
    if dtype == "bf16":
        vb = torch.from_numpy(v).to(torch.bfloat16)
        v = vb.float().numpy()
        zb = torch.zeros_like(vb).view(torch.uint16).numpy()
        out = rp.masked_attention_exact(g, rp.BlockMask(g.blocks_per_dim, bits), zb, zb,
                                        vb.view(torch.uint16).numpy())
        out = torch.from_numpy(out).view(torch.bfloat16).float().numpy()
    else:
        out = rp.masked_attention_exact(g, rp.BlockMask(g.blocks_per_dim, bits), q, q, v)
    Sp = g.padded_tokens
    vp = np.concatenate([v, np.zeros((Sp - v.shape[0], H, d), np.float32)]).astype(np.float64)
    tok = np.kron(dense, np.ones((bs, bs))).astype(np.float64)
    want = np.einsum("rc,chd->rhd", tok, vp) / tok.sum(axis=1)[:, None, None]
    if dtype == "f32":
        assert np.abs(out - want).max() < 1e-6
    else:  # one bf16 rounding of the fp32-accumulated average (plus P = 1 exactly)
        assert np.all(np.abs(out - want) <= 2.0 ** -8 * np.abs(want) + 1e-5)
