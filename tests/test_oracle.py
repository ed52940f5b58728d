"""CPU: pin the oracle (C restatement) against the reference's own outputs.

* every golden mask (made by the compiled reference, tests/golden) is
  reproduced bit for bit by the restatement;
* SPEC acceptance criterion 1 run against the compiled
  reference: N_f in 2..6, N_t in {4, 8, 12}, B = 4, 50 random Table-5 configs
  per mode (1500 builds);
* stage (d) restatement vs the reference's masked_attention_exact golden.
"""
import numpy as np
import pytest

from golden_util import GOLDEN, case_id, features, mask_cases, read_drbm
from oracle import pyoracle
from oracle.pyoracle import Cfg

CASES = mask_cases()


@pytest.mark.parametrize("case", CASES, ids=[case_id(c) for c in CASES])
def test_port_matches_golden_masks(port, case):
    q, k = features(port, case["features"])
    bits = port.build_mask(case["nf"], case["nt"], case["bs"], case["cfg"], case["seed"],
                           case["disable_split"], q, k, threads=3)
    assert np.array_equal(bits, case["bits"])


def test_wan_config3_golden(port):
    dim, bits = read_drbm(f"{GOLDEN}/wan_cfg3.drbm")
    assert dim == 591
    assert int(np.unpackbits(bits).sum()) == 67743  # sparsity 0.8061
    got = port.build_mask(21, 3600, 128, Cfg(0, 1.0, 0.1, 1e-6, 1.0, 0.2, 0.3, 0.3), 7,
                          threads=8)
    assert np.array_equal(got, bits)


def _spec_configs(mode, rng, n=50):
    out = []
    for _ in range(n):
        g = rng.uniform(1.0, 3.0)
        lam = rng.uniform(0.1, 1.0)
        tc = rng.uniform(0.1, 1.0)
        tm = rng.uniform(0.1, 1.0)
        if mode == 0:
            a, b = rng.uniform(0.3, 1.0), rng.uniform(0.1, 0.8)
        else:
            a, b = rng.uniform(-10.0, 5.0), rng.uniform(-5.0, 8.0)
        out.append(Cfg(mode, g, lam, 1e-6, tm, tc, a, b, int(rng.integers(1, 4))))
    return out


def spec_sweep(mode, seed=2024):
    rng = np.random.default_rng(seed + mode)
    cfgs = _spec_configs(mode, rng)
    for nf in range(2, 7):
        for nt in (4, 8, 12):
            for ci, c in enumerate(cfgs):
                yield nf, nt, c, int(rng.integers(0, 2**63)), (nf * nt, 2, 8, 100 + ci)


@pytest.mark.parametrize("mode", [0, 1])
def test_spec_criterion1_port_vs_reference(ref, port, mode):
    n = 0
    for nf, nt, c, seed, fs in spec_sweep(mode):
        q = k = None
        if mode == 1:
            q, k = features(port, fs)
        a = ref.build_mask(nf, nt, 4, c, seed, False, q, k)
        b = port.build_mask(nf, nt, 4, c, seed, False, q, k)
        assert np.array_equal(a, b), (nf, nt, c, seed)
        n += 1
    assert n == 750


def test_random_batch_bit_identical(ref, port):
    a = ref.random_batch(300, 3, 16, 42)
    b = port.random_batch(300, 3, 16, 42, threads=3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_attention_restatement_vs_reference_golden(port):
    z = np.load(f"{GOLDEN}/attn_small.npz")
    nf, nt, bs = int(z["nf"]), int(z["nt"]), int(z["bs"])
    q, k, v = port.random_batch(nf * nt, 2, 32, int(z["seed"]), threads=2)
    out = port.masked_attention_exact(nf, nt, bs, z["bits"], q, k, v, threads=4)
    assert np.abs(out - z["exact"]).max() <= 1e-6
    # soft vs exact differ by ~S'*eps mass: informational bound
    assert np.abs(z["soft"] - z["exact"]).max() < 1e-6


def test_static_select_stream_matches_reference(ref):
    """static_select (selection.cpp:61-91): k = max(1, floor(n*rho)) distinct
    pairs of the band, in shuffle order, from the pair's splitmix64 stream."""
    c = Cfg(0, 2.0, 1.0)
    uv = ref.static_select(8, 8, 4, c, 0, 2, 0.25, 99)
    assert len(uv) == 13  # |P| = 52
    assert len({tuple(x) for x in uv}) == 13
    assert all(abs(u - v) <= 4 for u, v in uv)


def test_reference_library_and_oracle_disagree_on_disable_split(ref):
    """With BuildOptions::disable_split, the reference's build_mask gives
    split-pruned frame pairs an empty candidate set (candidate_set keeps
    retained=false, radial.cpp:111-121) while its own brute-force
    oracle::build scores their full band (tests/oracle.cpp:190-197).  Parity
    for disable_split is therefore pinned to the library (the GPU follows it,
    tests/test_mask_gpu.py golden '-nosplit' cases), not to oracle::build.
    (Static mode with disable_split divides by zero in the reference, SIGFPE;
    the GPU path raises InvalidArgument instead.)"""
    differ = 0
    for seed in range(5):
        cfg = pyoracle.Cfg(1, 1.0, 0.1, 1e-6, 0.3, 0.3, -0.5, -0.5, 1)
        q, k, _ = ref.random_batch(6 * 8, 2, 8, seed, with_values=False)
        lib = ref.build_mask(6, 8, 4, cfg, 7, disable_split=True, q=q, k=k)
        orc = pyoracle.pack_dense(ref.oracle_build(6, 8, 4, cfg, 7, disable_split=True, q=q, k=k))
        same_split = np.array_equal(
            ref.build_mask(6, 8, 4, cfg, 7, q=q, k=k),
            pyoracle.pack_dense(ref.oracle_build(6, 8, 4, cfg, 7, q=q, k=k)))
        assert same_split
        differ += not np.array_equal(np.asarray(lib), np.asarray(orc))
    assert differ == 5


def test_soft_attention_restatement_vs_reference_golden(port):
    """masked_attention (attention.cpp:59-81) soft mask at four epsilons."""
    z = np.load(f"{GOLDEN}/attn_small.npz")
    nf, nt, bs = int(z["nf"]), int(z["nt"]), int(z["bs"])
    q, k, v = port.random_batch(nf * nt, 2, 32, int(z["seed"]), threads=2)
    out = port.masked_attention(nf, nt, bs, z["bits"], q, k, v, eps=1e-10, threads=4)
    assert np.abs(out - z["soft"]).max() <= 1e-6
    for eps, want in zip(z["soft_eps"], z["soft_multi"]):
        out = port.masked_attention(nf, nt, bs, z["bits"], q, k, v, eps=float(eps), threads=4)
        assert np.abs(out - want).max() <= 1e-6, eps
    with pytest.raises(pyoracle.OracleError):
        port.masked_attention(nf, nt, bs, z["bits"], q, k, v, eps=0.0)


def test_objective_restatement_vs_reference_golden(port):
    """build_proxy_cache / objective (profiler.cpp:49-148): the C restatement
    reproduces the reference's golden records bit for bit."""
    z = np.load(f"{GOLDEN}/objective.npz")
    nf, nt, bs = int(z["nf"]), int(z["nt"]), int(z["bs"])
    for r, seed in enumerate(z["seeds"]):
        f = z["features"][r]
        _, rs, sq = port.proxy_cache(f, threads=2)
        assert np.array_equal(rs, z["row_sums"][r]) and sq == z["sq_norm"][r]
        for c, want in zip(z["configs"], z["trials"][r]):
            cfg = Cfg(int(c[0]), *c[1:8], int(c[8]))
            got = port.objective(nf, nt, bs, cfg, f, int(seed), threads=2)
            assert got == tuple(want), (r, c)


def test_objective_restatement_vs_reference_random(ref, port):
    """Fresh simulated batches and configs, straight against oracle/_ref."""
    rng = np.random.default_rng(3)
    for trial in range(6):
        nf, nt, bs = 5, 64, (8, 16, 32)[trial % 3]
        f = ref.simulate(nf, nt, bs, 24, 100 + trial, drift_rate=float(rng.uniform(0, 0.5)))
        mode = trial % 2
        far = float(rng.uniform(-1, 2)) if mode else float(rng.uniform(0.1, 0.8))
        cfg = Cfg(mode, float(rng.uniform(1, 3)), float(rng.uniform(0.1, 1)), 1e-6,
                  float(rng.uniform(0.1, 1)), float(rng.uniform(0.1, 1)),
                  float(rng.uniform(-1, 1)) if mode else float(rng.uniform(0.3, 1)), far, 1)
        want = ref.objective(nf, nt, bs, cfg, f, 7 + trial)
        assert port.objective(nf, nt, bs, cfg, f, 7 + trial, threads=2) == want


def test_expand_mask_port_matches_reference_golden(port):
    """The C restatement's expand_mask equals the reference's own TokenMask
    bytes (tests/golden/expand_mask.npz, made by oracle/_ref)."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "expand_mask.npz"))
    for i in range(int(g["n"])):
        nf, nt, bs = (int(x) for x in g[f"grid_{i}"])
        np.testing.assert_array_equal(port.expand_mask(nf, nt, bs, g[f"bits_{i}"]),
                                      g[f"token_{i}"])
