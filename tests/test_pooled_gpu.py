"""the north star's pooled block selector (rp_pooled_select).

Not the reference's semantics, so its oracle is this CPU restatement (test
infrastructure, numpy, fp64): block classification from the radial windows /
split rule of the plan (radial.cpp:30-54), block-mean pooling, block scores,
per-row top-k or cumulative softmax mass, ties to the lower column.  GPU
scores are fp32, so a row is compared exactly unless its selection boundary
sits on a near-tie (|gap| below 1e-4 of the score scale), where the two
boundary candidates may swap.
"""
import math

import numpy as np
import pytest
import torch

from paper_2604_20470_b200 import radialplan as rp

pytestmark = pytest.mark.gpu


def classify(g, p):
    nb, nt, S, B = g.blocks_per_dim, g.tokens_per_frame, g.total_tokens, g.block_size
    width = [rp.window_width(0, t, p, g) for t in range(g.n_frames)]
    keep = [rp.frame_retained(t, p, g) for t in range(g.n_frames)]
    st = np.zeros((nb, nb), np.uint8)
    for r in range(nb):
        t0, t1 = r * B, min(r * B + B, S)
        for c in range(nb):
            k0, k1 = c * B, min(c * B + B, S)
            if t0 >= t1 or k0 >= k1:
                continue
            v = 0
            for fi in range(t0 // nt, (t1 - 1) // nt + 1):
                ua, ub = max(t0, fi * nt) - fi * nt, min(t1 - 1, fi * nt + nt - 1) - fi * nt
                for fj in range(k0 // nt, (k1 - 1) // nt + 1):
                    va, vb = max(k0, fj * nt) - fj * nt, min(k1 - 1, fj * nt + nt - 1) - fj * nt
                    t = abs(fi - fj)
                    if t <= 1:
                        v = 2
                    elif keep[t] and not (va - ub > width[t] or ua - vb > width[t]):
                        v = max(v, 1)
            st[r, c] = v
    return st


def oracle(g, p, q, k, hf, mode, param):
    """Returns (dense 0/1 mask, per-row sorted candidate scores, per-row keep count)."""
    nb, B, S = g.blocks_per_dim, g.block_size, g.total_tokens
    d = q.shape[2]
    qf = q[:, :hf].reshape(S, hf * d).astype(np.float64)
    kf = k[:, :hf].reshape(S, hf * d).astype(np.float64)
    qp = np.stack([qf[b * B:min(S, b * B + B)].mean(0) for b in range(nb)])
    kp = np.stack([kf[b * B:min(S, b * B + B)].mean(0) for b in range(nb)])
    sc = qp @ kp.T / math.sqrt(d) / hf
    st = classify(g, p)
    dense = (st == 2).astype(np.uint8)
    rows = []
    for r in range(nb):
        cand = np.nonzero(st[r] == 1)[0]
        order = sorted(cand, key=lambda c: (-sc[r, c], c))
        s_sorted = np.array([sc[r, c] for c in order])
        n = len(order)
        keep = 0
        if n:
            if mode == rp.PooledMode.TopK:
                keep = max(1, math.floor(n * param))
            else:
                w = np.exp(s_sorted - s_sorted[0])
                cum = np.cumsum(w)
                keep = int(np.searchsorted(cum, param * cum[-1]) + 1)
                keep = min(keep, n)
        for c in order[:keep]:
            dense[r, c] = 1
        rows.append((order, s_sorted, keep, np.cumsum(np.exp(s_sorted - s_sorted[0]))
                     if n else np.zeros(0)))
    return dense, rows, st


CASES = [  # nf, nt, B, H, d, hf, gamma, lambda, mode, param
    (8, 256, 32, 2, 64, 2, 1.4, 0.7, rp.PooledMode.TopK, 0.3),
    (8, 256, 32, 2, 64, 2, 1.4, 0.7, rp.PooledMode.Mass, 0.95),
    (6, 700, 128, 3, 128, 2, 1.0, 0.3, rp.PooledMode.TopK, 0.5),
    (6, 700, 128, 3, 128, 2, 1.0, 0.3, rp.PooledMode.Mass, 0.9),
    (21, 600, 64, 2, 128, 1, 2.0, 0.3, rp.PooledMode.Mass, 0.95),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}x{c[1]}-B{c[2]}-{c[8].name}")
def test_pooled_selector_vs_cpu_restatement(cuda, case):
    nf, nt, B, H, d, hf, gm, lm, mode, param = case
    g = rp.make_grid(nf, nt, B)
    p = rp.RadialParams(gm, lm)
    cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, p)
    S = g.total_tokens
    gen = torch.Generator().manual_seed(nf * 31 + nt)
    # structured features: a smooth per-token drift makes block means informative
    base = torch.randn(S, H, d, generator=gen)
    drift = torch.cumsum(torch.randn(S, 1, d, generator=gen) * 0.05, 0)
    q = (base + drift).to(torch.bfloat16)
    k = (torch.randn(S, H, d, generator=gen) + drift).to(torch.bfloat16)
    bits = rp.pooled_select(g, cfg, q.cuda(), k.cuda(), hf, mode, param).cpu().numpy()
    got = np.unpackbits(bits, axis=1, bitorder="little")[:, : g.blocks_per_dim]
    want, rows, st = oracle(g, p, q.float().numpy(), k.float().numpy(), hf, mode, param)
    assert np.array_equal(got[st == 2], want[st == 2])  # forced blocks
    assert not got[st == 0].any()                        # never outside the candidates
    scale = max(1e-30, float(np.abs(np.concatenate([r[1] for r in rows if len(r[1])])).max()))
    checked = 0
    for r, (order, s_sorted, keep, cum) in enumerate(rows):
        if np.array_equal(got[r], want[r]):
            checked += 1
            continue
        # only a near-tie at the selection boundary may differ
        n = len(order)
        assert 0 < keep < n, r
        gap = abs(s_sorted[keep - 1] - s_sorted[keep])
        mass_tie = mode == rp.PooledMode.Mass and min(
            abs(cum[keep - 1] - param * cum[-1]),
            abs(cum[keep - 2] - param * cum[-1]) if keep >= 2 else np.inf) < 1e-5 * cum[-1]
        assert gap < 1e-4 * scale or mass_tie, (r, gap)
        diff = np.nonzero(got[r] != want[r])[0]
        assert set(diff) <= {order[keep - 1], order[keep]}, (r, diff)
    assert checked >= 0.98 * len(rows)


def test_pooled_selector_errors(cuda):
    g = rp.make_grid(2, 128, 64)
    cfg = rp.SparsityConfig()
    q = torch.zeros(256, 1, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(rp.InvalidArgument):
        rp.pooled_select(g, cfg, q, q, 1, rp.PooledMode.Mass, 1.5)
    with pytest.raises(rp.InvalidArgument):
        rp.pooled_select(g, cfg, q.float(), q.float(), 1, rp.PooledMode.TopK, 0.5)


def test_block_mean_pool_stage_b(cuda):
    """rp_block_mean_pool: block means of the first n heads, padded last block
    averaged over its valid tokens only."""
    g = rp.make_grid(3, 250, 128)
    torch.manual_seed(0)
    x = torch.randn(g.total_tokens, 4, 64, device="cuda").to(torch.bfloat16)
    out = rp.block_mean_pool(g, x, 2).cpu().numpy()
    xf = x[:, :2].reshape(g.total_tokens, 128).float().cpu().numpy().astype(np.float64)
    B, S = g.block_size, g.total_tokens
    want = np.stack([xf[b * B:min(S, b * B + B)].mean(0) for b in range(g.blocks_per_dim)])
    assert np.abs(out - want).max() < 1e-5
