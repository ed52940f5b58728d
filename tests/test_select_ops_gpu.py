"""The per-frame-pair selection operators on the GPU (rp_static_select,
rp_proxy_scores, rp_normalize_scores, rp_dynamic_select) against the
reference's own static_select / proxy_scores / normalize_scores /
dynamic_select (oracle/_ref): identical pair lists, bit-identical scores, z
values and stats (selection.cpp:61-185)."""
import numpy as np
import pytest

from oracle import pyoracle
from paper_2604_20470_b200 import radialplan as rp

pytestmark = pytest.mark.gpu

CASES = [  # nf, nt, bs, gamma, lambda, (i, j)
    (4, 16, 4, 1.0, 1.0, (0, 2)),
    (3, 12, 4, 0.6, 1.0, (2, 1)),
    (6, 33, 8, 1.3, 1.0, (1, 4)),
    (8, 256, 32, 1.4, 0.7, (0, 3)),
    (2, 200, 16, 2.0, 1.0, (1, 0)),
]


def _cfg(gm, lm):
    return pyoracle.Cfg(1, gm, lm, 1e-6, 0.7, 0.45, 0.0, 0.0, 1)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}x{c[1]}-B{c[2]}-{c[5]}")
def test_selection_operators_vs_reference(cuda, ref, case):
    import torch
    nf, nt, bs, gm, lm, (i, j) = case
    g = rp.make_grid(nf, nt, bs)
    p = rp.RadialParams(gm, lm)
    cs = rp.candidate_set(i, j, p, g)
    cfg = _cfg(gm, lm)
    assert (cs.width, int(cs.retained), cs.pair_count()) == ref.frame_pair(nf, nt, bs, cfg, i, j)[:3]
    # static_select, several ratios and seeds (slot order of the Fisher-Yates)
    for ratio, seed in [(0.22, 7), (0.5, 12345), (1.0, 3), (1e-9, 99)]:
        got = np.asarray(rp.static_select(cs, ratio, seed), np.int64).reshape(-1, 2)
        want = ref.static_select(nf, nt, bs, cfg, i, j, ratio, seed)
        assert np.array_equal(got, want), (ratio, seed)
    # proxy_scores + normalize_scores: bit-identical
    q, k, _ = ref.random_batch(nf * nt, 2, 16, 42, with_values=False)
    s_want, z_want, st_want = ref.proxy_scores(nf, nt, bs, cfg, i, j, q, k)
    fb = rp.FeatureBatch(torch.from_numpy(q).cuda(), torch.from_numpy(k).cuda())
    s = rp.proxy_scores(fb, i, j, cs, nt)
    assert np.array_equal(s.cpu().numpy().view(np.uint32), s_want.view(np.uint32))
    st = {}
    z = rp.normalize_scores(s, st)
    assert np.array_equal(z.cpu().numpy().view(np.uint64), z_want.view(np.uint64))
    assert (st["mean"], st["stddev"]) == st_want
    # dynamic_select: thresholds that keep some, none (fallback_k 1..3)
    for tau, fk in [(-0.3, 1), (0.9, 2), (1e9, 1), (1e9, 3)]:
        got = np.asarray(rp.dynamic_select(cs, z, tau, fk), np.int64).reshape(-1, 2)
        want = ref.dynamic_select(nf, nt, bs, cfg, i, j, z_want, tau, fk)
        assert np.array_equal(got, want), (tau, fk)


def test_fallback_ties_go_to_lowest_index(cuda, ref):
    import torch
    g = rp.make_grid(3, 8, 4)
    cs = rp.candidate_set(0, 1, rp.RadialParams(), g)
    n = cs.pair_count()
    z = np.zeros(n)  # every pair ties
    z[[5, 9, 17]] = -1.0
    zt = torch.from_numpy(z).cuda()
    for fk in (1, 2, 4, n + 3):
        got = np.asarray(rp.dynamic_select(cs, zt, 5.0, fk), np.int64).reshape(-1, 2)
        want = ref.dynamic_select(3, 8, 4, _cfg(1.0, 1.0), 0, 1, z, 5.0, fk)
        assert np.array_equal(got, want), fk


def test_static_select_errors(cuda):
    g = rp.make_grid(3, 8, 4)
    cs = rp.candidate_set(0, 1, rp.RadialParams(), g)
    with pytest.raises(rp.InvalidArgument, match="ratio must be in"):
        rp.static_select(cs, 1.5, 1)
    empty = rp.CandidateSet(0, 5, 5, 8, 4, False)
    assert rp.static_select(empty, 1.5, 1) == []  # empty band returns before validating
