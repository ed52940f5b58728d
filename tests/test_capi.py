"""CPU: the C-ABI library loads, exports every symbol include/dynrad.h
declares, maps errors like the reference's exceptions, and refuses to
compute without a GPU (there is no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2604_20470_b200 import _lib
from paper_2604_20470_b200 import radialplan as rp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "dynrad.h")).read()
    return sorted(set(re.findall(r"\b(rp_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(_lib.PUBLIC_SYMBOLS) == set(syms)


def test_grid_like_reference_tests():
    # tests/test_grid.cpp:7-68
    g = rp.make_grid(4, 8, 4)
    assert (g.total_tokens, g.padded_tokens, g.blocks_per_dim) == (32, 32, 8)
    g = rp.make_grid(1, 1, 2)
    assert (g.total_tokens, g.padded_tokens, g.blocks_per_dim) == (1, 2, 1)
    g = rp.make_grid(72, 3667, 32)
    assert (g.total_tokens, g.padded_tokens, g.blocks_per_dim) == (264024, 264032, 8251)
    for bad in [(2, 4, 3), (2, 4, 1), (2, 4, 0), (2, 4, 12), (0, 4, 4), (4, 0, 4)]:
        with pytest.raises(rp.InvalidArgument):
            rp.make_grid(*bad)
    g = rp.make_grid(4, 8, 4)
    assert rp.block_of(0, g) == 0 and rp.block_of(7, g) == 1 and rp.block_of(31, g) == 7
    with pytest.raises(rp.OutOfRange):
        rp.block_of(32, g)
    assert rp.frame_of(15, g) == 1
    assert rp.frame_of(15, rp.make_grid(3, 5, 4)) == 2
    for nf in (1, 3, 7):
        for nt in (1, 5, 9, 64):
            for bs in (2, 4, 16):
                g = rp.make_grid(nf, nt, bs)
                assert 0 <= g.padded_tokens - g.total_tokens < bs
                assert g.blocks_per_dim * bs == g.padded_tokens


def test_radial_scalars_like_reference_tests():
    # tests/test_radial.cpp and SPEC.md:100-160 examples
    assert [rp.group_index(t) for t in (1, 3, 8)] == [1, 2, 4]
    assert [rp.base_span(n) for n in (8, 10, 1, 3667)] == [8, 16, 1, 4096]
    assert rp.decay_length(2, 2.0, 8) == 4.0 and rp.decay_length(4, 1.0, 8) == 1.0
    g = rp.make_grid(8, 8, 4)
    p = rp.RadialParams(decay_factor=2.0)
    assert rp.window_width(3, 3, p, g) == 8 and rp.window_width(3, 4, p, g) == 8
    assert rp.window_width(0, 2, p, g) == 4
    assert rp.window_width(0, 4, rp.RadialParams(1.0), g) == 4
    g16 = rp.make_grid(16, 8, 4)
    # test_radial.cpp:69-73 expects split_factor(2) == 2 here, but the
    # reference LIBRARY returns 1: raw = 4 / (2.0 + 1e-6) = 1.999999 truncates
    # to 1 (radial.cpp:41-49).  The shipped test never ran (doctest absent);
    # we follow the library, which is what build_mask uses.
    assert rp.split_factor(2, rp.RadialParams(1.0, 1.0), g16) == 1
    assert rp.frame_retained(3, rp.RadialParams(1.0, 1.0), g16)
    assert rp.split_factor(2, rp.RadialParams(1.0, 0.3), g16) == 6
    assert not rp.frame_retained(3, rp.RadialParams(1.0, 0.3), g16)
    cs = rp.candidate_set(0, 2, p, g)
    assert cs.width == 4 and cs.pair_count() == 52
    assert rp.candidate_set(3, 4, p, g).pair_count() == 64
    pr = rp.candidate_set(0, 2, rp.RadialParams(1.0, 0.3), g)
    assert not pr.retained and pr.pair_count() == 0
    seen = []
    c = rp.CandidateSet(0, 0, 0, 7, 2, True)
    c.visit(lambda u, v: seen.append((u, v)))
    assert len(seen) == c.pair_count() and seen == sorted(seen)
    assert all(c.pair_at(i) == seen[i] for i in range(len(seen)))
    with pytest.raises(rp.OutOfRange):
        c.pair_at(c.pair_count())


def test_scalars_match_reference_library(ref):
    cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.7, 0.35), 0.6, 0.3, 0.4, 0.2)
    from oracle.pyoracle import Cfg
    oc = Cfg(0, 1.7, 0.35, 1e-6, 0.6, 0.3, 0.4, 0.2)
    for nf, nt, bs in [(16, 64, 8), (21, 3600, 128), (61, 3600, 64), (9, 250, 32)]:
        g = rp.make_grid(nf, nt, bs)
        for j in range(nf):
            fp = rp._pair(0, j, cfg.radial, g, cfg)
            w, ret, n, tier, sf = ref.frame_pair(nf, nt, bs, oc, 0, j)
            assert (fp.width, fp.retained, fp.pair_count, fp.tier) == (w, ret, n, tier)
            if j >= 1:
                assert fp.split_factor == sf


def test_config_validation_messages():
    # selection.cpp:11-32 messages are part of the API
    bad = [
        (dict(radial=rp.RadialParams(0.0)), "decay_factor must be positive"),
        (dict(radial=rp.RadialParams(1.0, -1.0)), "long_range_factor must be positive"),
        (dict(mask_threshold=0.0), "mask_threshold must be in"),
        (dict(col_threshold=1.5), "col_threshold must be in"),
        (dict(fallback_k=0), "fallback_k must be >= 1"),
        (dict(near_param=1.5), "static retention ratios must be in"),
        (dict(mode=rp.Mode.DynamicThreshold, far_param=float("inf")),
         "dynamic thresholds must be finite"),
    ]
    for kw, msg in bad:
        with pytest.raises(rp.InvalidArgument, match=msg):
            rp.SparsityConfig(**kw).validate()
    rp.SparsityConfig().validate()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = rp.make_grid(2, 8, 4).c()
    act = C.c_int64()
    sp = C.c_double()
    rc = _lib.lib().rp_mask_sparsity(C.byref(g), None, C.byref(act), C.byref(sp), None)
    assert rc == 5  # RP_CUDA_ERROR
    assert "no CPU fallback" in _lib.lib().rp_last_error().decode()


def test_aggregate_block_spec_example():
    # 4x4 tile, 2 full columns, theta_c=.5: theta_m=.5 on, .6 off
    kept = [(r, c) for r in range(4) for c in (0, 1)]
    assert rp.aggregate_block(kept, 0.5, 0.5, 4)
    assert not rp.aggregate_block(kept, 0.5, 0.6, 4)
    assert rp.aggregate_block([(r, c) for r in range(4) for c in range(4)], 1.0, 1.0, 4)
    assert not rp.aggregate_block([], 0.1, 0.1, 4)
