"""Stages (a)-(c) parity on the B200: device build_mask vs the reference.

Bit-exact (integer/byte work): every golden mask of the compiled reference,
the Wan2.1 config-3 production mask, and a sweep of random configs checked
against the C restatement (itself pinned to the reference in test_oracle).
"""
import json

import numpy as np
import pytest
import torch

from golden_util import GOLDEN, case_id, features, mask_cases, read_drbm
from oracle import pyoracle
from oracle.pyoracle import Cfg
from paper_2604_20470_b200 import radialplan as rp

pytestmark = pytest.mark.gpu
CASES = mask_cases()


def to_cfg(c: Cfg) -> rp.SparsityConfig:
    return rp.SparsityConfig(rp.Mode(c.mode),
                             rp.RadialParams(c.decay_factor, c.long_range_factor,
                                             c.split_epsilon),
                             c.mask_threshold, c.col_threshold, c.near_param, c.far_param,
                             c.fallback_k)


def gpu_mask(nf, nt, bs, c, seed, disable_split=False, q=None, k=None, dtype=torch.float32,
             engine=0, stats=None):
    g = rp.make_grid(nf, nt, bs)
    feats = None
    if q is not None:
        feats = rp.FeatureBatch(torch.from_numpy(q).cuda().to(dtype),
                                torch.from_numpy(k).cuda().to(dtype))
    m = rp.build_mask(g, to_cfg(c), seed, rp.BuildOptions(disable_split, engine), feats,
                      stats=stats)
    return m.bits


@pytest.mark.parametrize("case", CASES, ids=[case_id(c) for c in CASES])
def test_golden_masks_bit_exact(cuda, port, case):
    q, k = features(port, case["features"])
    got = gpu_mask(case["nf"], case["nt"], case["bs"], case["cfg"], case["seed"],
                   case["disable_split"], q, k)
    assert np.array_equal(got, case["bits"]), int((got != case["bits"]).sum())


def test_wan_config3_static_bit_exact(cuda):
    _, want = read_drbm(f"{GOLDEN}/wan_cfg3.drbm")
    st = {}
    got = gpu_mask(21, 3600, 128, Cfg(0, 1.0, 0.1, 1e-6, 1.0, 0.2, 0.3, 0.3), 7, stats=st)
    assert np.array_equal(got, want)
    assert st["active_blocks"] == 67743
    assert st["sampled_pairs"] > 2e8  # 231.4M Fisher-Yates draws


@pytest.mark.parametrize("bs", [4, 8, 16, 32, 64, 128])
def test_static_random_configs_vs_oracle(cuda, port, bs):
    rng = np.random.default_rng(bs)
    for trial in range(6):
        nf = int(rng.integers(2, 9))
        nt = int(rng.integers(bs // 2 + 1, 3 * bs + 40))
        c = Cfg(0, rng.uniform(1.0, 3.0), rng.uniform(0.1, 1.0), 1e-6, rng.uniform(0.1, 1.0),
                rng.uniform(0.1, 1.0), rng.uniform(0.3, 1.0), rng.uniform(0.1, 0.8))
        seed = int(rng.integers(0, 2**62))
        want = port.build_mask(nf, nt, bs, c, seed, threads=4)
        got = gpu_mask(nf, nt, bs, c, seed)
        assert np.array_equal(got, want), (nf, nt, c, seed)


def test_spec_criterion1_sweep_gpu(cuda, port):
    """SPEC.md:783 sweep (B=4) through the GPU builder, both modes, exact engine."""
    from test_oracle import spec_sweep
    for mode in (0, 1):
        for n, (nf, nt, c, seed, fs) in enumerate(spec_sweep(mode)):
            if n % 5:  # every 5th case keeps the GPU suite short
                continue
            q = k = None
            if mode == 1:
                q, k = features(port, fs)
            want = port.build_mask(nf, nt, 4, c, seed, False, q, k)
            got = gpu_mask(nf, nt, 4, c, seed, False, q, k)
            assert np.array_equal(got, want), (mode, nf, nt, c, seed)


def test_static_mask_is_cached_per_plan(cuda):
    g = rp.make_grid(8, 256, 32)
    plan = rp.Plan(g, to_cfg(Cfg(0, 2.0, 0.3, 1e-6, 0.75, 0.2, 0.2, 0.2)), 7)
    a = plan.build_mask_device().clone()
    n0 = rp.kernel_launch_count()
    b = plan.build_mask_device()
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert rp.kernel_launch_count() == n0  # second call re-emits the cache


def test_dynamic_needs_features(cuda):
    g = rp.make_grid(4, 16, 4)
    with pytest.raises(rp.InvalidArgument, match="dynamic mode needs features"):
        rp.build_mask(g, rp.SparsityConfig(rp.Mode.DynamicThreshold), 1)


# ------------------------------------------------ tensor-core dynamic engine
FAST_CASES = [
    # nf, nt, bs, hf, d, cfg
    (8, 256, 128, 2, 64, Cfg(1, 1.4, 0.7, 1e-6, 0.7, 0.45, 0.0, 0.0)),
    (8, 256, 32, 2, 64, Cfg(1, 1.4, 0.7, 1e-6, 0.7, 0.45, -1.5, 2.0)),
    (8, 256, 64, 2, 64, Cfg(1, 1.4, 0.7, 1e-6, 0.7, 0.45, 0.05, 0.05)),
    (6, 500, 128, 2, 128, Cfg(1, 2.0, 0.5, 1e-6, 0.5, 0.3, 0.5, 1.0)),
    (6, 500, 64, 1, 128, Cfg(1, 1.0, 1.0, 1e-6, 0.3, 0.2, -0.5, 0.8)),
    (8, 512, 128, 2, 128, Cfg(1, 1.4, 0.7, 1e-6, 0.7, 0.45, -1.5, 2.0)),
]


@pytest.mark.parametrize("case", FAST_CASES, ids=lambda c: f"{c[0]}x{c[1]}-B{c[2]}-hf{c[3]}-d{c[4]}")
def test_fast_engine_matches_reference(cuda, port, case):
    """bf16 features: tensor-core scores + exact fp64 recheck near tau vs the
    reference algorithm on the same (bf16-valued) features."""
    nf, nt, bs, hf, d, c = case
    q, k, _ = port.random_batch(nf * nt, hf, d, 42, with_values=False, threads=8)
    qb = torch.from_numpy(q).to(torch.bfloat16)
    kb = torch.from_numpy(k).to(torch.bfloat16)
    want = port.build_mask(nf, nt, bs, c, 7, False, qb.float().numpy(), kb.float().numpy(),
                           threads=8)
    st = {}
    got = gpu_mask(nf, nt, bs, c, 7, False, qb.float().numpy(), kb.float().numpy(),
                   dtype=torch.bfloat16, engine=1, stats=st)
    exact = gpu_mask(nf, nt, bs, c, 7, False, qb.float().numpy(), kb.float().numpy(),
                     dtype=torch.bfloat16, engine=2)
    assert np.array_equal(exact, want)
    assert np.array_equal(got, want), int((got != want).sum())
    assert st["rechecked_pairs"] < 0.05 * max(st["scored_pairs"], 1)


@pytest.mark.parametrize("engine", [1, 2])
def test_split_scoring_shards_or_to_the_full_mask(cuda, engine):
    """BuildOptions.shard_index / shard_count (multi-GPU split of the dynamic
    scoring): the OR of every shard's mask is the unsharded mask, and the
    shards' scored pairs partition the layer's."""
    nf, nt, bs = (8, 256, 128) if engine == 1 else (5, 64, 16)
    g = rp.make_grid(nf, nt, bs)
    cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45,
                            0.05, 0.08)
    torch.manual_seed(4)
    q = torch.randn(g.total_tokens, 2, 64, device="cuda").to(torch.bfloat16)
    k = torch.randn(g.total_tokens, 2, 64, device="cuda").to(torch.bfloat16)
    st = {}
    full = rp.Plan(g, cfg, 7, rp.BuildOptions(score_engine=engine)).build_mask_device(
        q, k, 2, stats=st)
    for world in (2, 3):
        acc = torch.zeros_like(full)
        scored = 0
        for r in range(world):
            s2 = {}
            part = rp.Plan(g, cfg, 7, rp.BuildOptions(score_engine=engine, shard_index=r,
                                                      shard_count=world)).build_mask_device(
                q, k, 2, stats=s2)
            acc |= part
            scored += s2["scored_pairs"]
        assert torch.equal(acc, full), world
        assert scored == st["scored_pairs"]
    with pytest.raises(rp.InvalidArgument):
        rp.Plan(g, cfg, 7, rp.BuildOptions(shard_index=2, shard_count=2))


def _mid_cfg():
    return rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45,
                             -1.5, 2.0)


@pytest.mark.parametrize("name", ["wan", "hunyuan"])
def test_production_dynamic_mask_equals_reference_golden(cuda, name):
    """Production scale against the REFERENCE's own output (SURVEY 8d config
    4 and the Wan grid, Table-3 Mid, H_f = 2, d = 128): the golden DRBM files
    were written by the reference's build_mask (oracle/_ref, all host cores,
    tests/golden/make_golden_production.py) on bf16-rounded random_batch(S, 2,
    128, 42) features -- the same values rp.random_batch generates on the
    device here.  Both device scoring engines must reproduce it bit for bit:
    the tensor-core engine (fp32 tile scores + fp64 recheck of every pair
    within the error bound of tau) and the exact fp64 engine.  A differing
    block would have to be an exact tie; none occurs."""
    with open(f"{GOLDEN}/production_meta.json") as f:
        meta = json.load(f)[name]
    dim, want = read_drbm(f"{GOLDEN}/{name}_mid.drbm")
    g = rp.make_grid(meta["nf"], meta["nt"], meta["bs"])
    assert dim == g.blocks_per_dim
    fb = rp.random_batch(g.total_tokens, 2, 128, meta["features"]["seed"], with_values=False)
    for engine in (1, 2):
        st = {}
        got = rp.Plan(g, _mid_cfg(), meta["mask_seed"],
                      rp.BuildOptions(score_engine=engine)).build_mask_device(
            fb.queries, fb.keys, 2, stats=st).cpu().numpy()
        assert st["scored_pairs"] == meta["timings"]["scored_pairs"]
        diff = np.argwhere(np.unpackbits(got ^ want, axis=1, bitorder="little")[:, :dim])
        assert diff.size == 0, (engine, diff[:10].tolist(), len(diff))
        assert st["active_blocks"] == meta["nnz"]
        if engine == 1:
            assert st["rechecked_pairs"] > 0


def test_wan_dynamic_fast_engine_equals_exact_engine(cuda):
    """Production scale (Wan 21x3600, B=128, Table-3 Mid, 1.6 G scored pairs)
    on torch.randn features (no reference output at this size): the
    tensor-core engine against the exact fp64 engine, which reproduces the
    reference's arithmetic bit for bit (scores, sequential per-pair
    mu/sigma)."""
    g = rp.make_grid(21, 3600, 128)
    cfg = _mid_cfg()
    gen = torch.Generator(device="cuda").manual_seed(42)
    q = torch.randn((g.total_tokens, 2, 128), device="cuda", generator=gen).to(torch.bfloat16)
    k = torch.randn((g.total_tokens, 2, 128), device="cuda", generator=gen).to(torch.bfloat16)
    st_fast, st_exact = {}, {}
    fast = rp.Plan(g, cfg, 7, rp.BuildOptions(score_engine=1)).build_mask_device(
        q, k, 2, stats=st_fast)
    exact = rp.Plan(g, cfg, 7, rp.BuildOptions(score_engine=2)).build_mask_device(
        q, k, 2, stats=st_exact)
    assert st_fast["scored_pairs"] == st_exact["scored_pairs"] == 1599385652
    assert torch.equal(fast, exact)
    assert st_fast["rechecked_pairs"] > 0


_SCHEDULE_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2604_20470_b200 import radialplan as rp
g = rp.make_grid(8, 512, 64)
cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45, -1.5, 2.0)
gen = torch.Generator(device="cuda").manual_seed(5)
q = torch.randn((g.total_tokens, 4, 128), device="cuda", generator=gen).to(torch.bfloat16)
k = torch.randn((g.total_tokens, 4, 128), device="cuda", generator=gen).to(torch.bfloat16)
fast = rp.Plan(g, cfg, 7, rp.BuildOptions(score_engine=1)).build_mask_device(q, k, 2)
exact = rp.Plan(g, cfg, 7, rp.BuildOptions(score_engine=2)).build_mask_device(q, k, 2)
assert torch.equal(fast, exact)
print("OK", int(fast.sum()))
"""


@pytest.mark.parametrize("env", [{"DYNRAD_SCORE_CG": "1"}, {"DYNRAD_SCORE_CG": "2"},
                                 {"DYNRAD_SCORE_CG": "4"}, {"DYNRAD_SCORE_ORDER": "plain"},
                                 {"DYNRAD_SCORE_UCAP": "1"}],
                         ids=lambda e: "-".join(f"{k}={v}" for k, v in e.items()))
def test_fast_engine_schedules_are_exact(cuda, env):
    """Every epilogue width (warps per sub-partition) and work order of the
    tensor-core scorer, and the in-place exact decision of undecided pairs
    that overflow a CTA's list (capacity forced to 1), give the exact
    engine's mask (read once per process, so each runs in a subprocess)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _SCHEDULE_SCRIPT, root], capture_output=True,
                       text=True, timeout=300, env={**os.environ, **env})
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-2000:]
