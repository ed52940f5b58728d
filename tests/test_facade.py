"""The C++ facade (libradialplan_b200.so, namespace radialplan): the
reference's own unit tests and brute-force oracle compiled unmodified against
it (oracle/_ref/*_on_facade, built by `make -C oracle facade` where
/root/reference exists), plus the facade's own self-test."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
SELFTEST = os.path.join(ROOT, "cpp", "tests", "facade_selftest")


def _run(path, *args, timeout=600):
    if not os.path.exists(path):
        pytest.skip(f"{os.path.relpath(path, ROOT)} not built")
    return subprocess.run([path, *args], capture_output=True, text=True, timeout=timeout)


def _have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def test_facade_selftest():
    # host checks always; without a GPU every GPU operator must throw
    r = _run(SELFTEST)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_reference_unit_tests_same_verdicts_on_facade():
    """tests/test_grid.cpp + tests/test_radial.cpp (the reference's own
    doctest files) give the identical check-by-check verdict on the facade as
    on the reference library.  Two checks of the shipped test_radial.cpp
    (:71, :73) fail on the reference itself: split_factor(2) at lambda=1 over
    8-token frames is trunc(4 / (2 + 1e-6)) = 1, not the 2 the test expects."""
    on_ref = _run(os.path.join(REF, "ref_unit_on_ref"))
    on_facade = _run(os.path.join(REF, "ref_unit_on_facade"))
    assert on_facade.stdout == on_ref.stdout
    assert on_facade.stderr == on_ref.stderr
    assert "675 checks, 2 failures" in on_facade.stdout
    failed = [ln for ln in on_facade.stderr.splitlines() if "CHECK failed" in ln]
    assert [ln.split(":")[1] for ln in failed] == ["71", "73"]


@pytest.mark.gpu
def test_facade_selftest_gpu():
    if not _have_gpu():
        pytest.skip("no CUDA device")
    r = _run(SELFTEST)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_reference_oracle_parity_on_facade():
    """oracle::build / pick_static / score_pairs / standardize / pick_dynamic
    (the reference's brute-force oracle) against the GPU facade: SPEC
    criterion-1 sweep + tiny golden shapes bit-identical, attention 1e-5."""
    if not _have_gpu():
        pytest.skip("no CUDA device")
    r = _run(os.path.join(REF, "parity_on_facade"), timeout=1200)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert "failures 0" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    # nf nt bs mode gamma lambda tm tc near far fk seed [feat_seed heads dim]
    "8 256 32 0 2.0 0.3 0.75 0.2 0.22 0.22 1 7",
    "8 256 64 0 2.0 1.0 0.75 0.2 0.22 0.22 1 7",
    "8 256 32 1 1.4 0.7 0.7 0.45 0.0 0.0 1 7 42 2 64",
    "5 12 4 1 1.1 0.4 0.3 0.3 0.8 1.5 3 99 5 2 8",
])
def test_facade_build_mask_vs_port(port, args):
    if not _have_gpu():
        pytest.skip("no CUDA device")
    from oracle import pyoracle
    a = args.split()
    r = _run(SELFTEST, "mask", *a)
    assert r.returncode == 0, r.stderr
    got = np.frombuffer(bytes.fromhex(r.stdout.strip()), np.uint8)
    nf, nt, bs, mode = (int(x) for x in a[:4])
    gm, lm, tm, tc, near, far = (float(x) for x in a[4:10])
    cfg = pyoracle.Cfg(mode, gm, lm, 1e-6, tm, tc, near, far, int(a[10]))
    q = k = None
    if len(a) > 12:
        q, k, _ = port.random_batch(nf * nt, int(a[13]), int(a[14]), int(a[12]),
                                    with_values=False)
    want = port.build_mask(nf, nt, bs, cfg, int(a[11]), q=q, k=k)
    assert np.array_equal(got, np.asarray(want, np.uint8).ravel())


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    # nf nt bs dim mode gamma lambda tm tc near far fk seed
    "6 96 16 32 0 1.5 0.5 0.6 0.3 0.5 0.3 1 11",
    "4 150 32 24 1 1.5 0.5 0.6 0.3 0.0 1.0 1 5",
])
def test_facade_objective_vs_port(port, args):
    """radialplan::objective / build_proxy_cache on the facade (with and
    without a host DenseProxyCache) against the restatement (bit-identical
    to the reference's profiler.cpp, tests/test_oracle.py)."""
    if not _have_gpu():
        pytest.skip("no CUDA device")
    from oracle import pyoracle
    a = args.split()
    r = _run(SELFTEST, "objective", *a)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.split("\n")
    nf, nt, bs, dim, mode = (int(x) for x in a[:5])
    t = np.arange(nf * nt)[:, None]
    d = np.arange(dim)[None, :]
    feats = (((t * 131 + d * 71) % 97 - 48) / 32.0).astype(np.float32)
    gm, lm, tm, tc, near, far = (float(x) for x in a[5:11])
    cfg = pyoracle.Cfg(mode, gm, lm, 1e-6, tm, tc, near, far, int(a[11]))
    want = port.objective(nf, nt, bs, cfg, feats, int(a[12]), threads=4)
    _, _, sq = port.proxy_cache(feats, threads=4)
    for line in lines[:2]:
        loss, mse, sp = (float(x) for x in line.split())
        assert sp == want[2]
        assert abs(mse - want[1]) <= 1e-9 * want[1] and abs(loss - want[0]) <= 1e-9 * want[0]
    assert abs(float(lines[2]) - sq) <= 1e-12 * sq
