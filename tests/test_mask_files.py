"""Mask file interop: the reference's DRBM / CSV / PGM formats
(mask.cpp:291-376) in the Python mirror and the C++ facade."""
import os

import numpy as np
import pytest

from golden_util import GOLDEN, read_drbm
from paper_2604_20470_b200 import radialplan as rp


def test_golden_drbm_round_trip(tmp_path):
    dim, bits = read_drbm(os.path.join(GOLDEN, "wan_cfg3.drbm"))  # the reference's mask bits
    m = rp.read_mask(os.path.join(GOLDEN, "wan_cfg3.drbm"))
    assert m.dim == dim == 591 and np.array_equal(m.bits, bits)
    assert m.active_count() == 67743
    out = tmp_path / "m.bin"
    rp.write_mask(m, rp.mask_format_for_path(str(out)), str(out))
    assert out.read_bytes() == open(os.path.join(GOLDEN, "wan_cfg3.drbm"), "rb").read()


def test_csv_and_pgm(tmp_path):
    m = rp.BlockMask(5)
    for r, c in [(0, 0), (1, 3), (4, 4), (4, 0)]:
        m.set(r, c)
    rp.write_mask(m, rp.MaskFormat.Csv, str(tmp_path / "m.csv"))
    assert (tmp_path / "m.csv").read_text() == "0,0\n1,3\n4,0\n4,4\n"
    rp.write_mask(m, rp.MaskFormat.Pgm, str(tmp_path / "m.pgm"))
    raw = (tmp_path / "m.pgm").read_bytes()
    assert raw.startswith(b"P5\n5 5\n255\n")
    img = np.frombuffer(raw[len(b"P5\n5 5\n255\n"):], np.uint8).reshape(5, 5)
    assert np.array_equal(img == 0, m.dense().astype(bool))


def test_errors(tmp_path):
    with pytest.raises(rp.InvalidArgument):
        rp.mask_format_for_path("mask.txt")
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"DRBX" + bytes(6))
    with pytest.raises(rp.RuntimeFailure, match="bad magic"):
        rp.read_mask(str(bad))
    trunc = tmp_path / "t.bin"
    trunc.write_bytes(b"DRBM" + (1).to_bytes(2, "little") + (9).to_bytes(4, "little") + bytes(3))
    with pytest.raises(rp.RuntimeFailure, match="truncated"):
        rp.read_mask(str(trunc))


@pytest.mark.parametrize("fmt", [0])
def test_files_byte_identical_to_reference_writer(tmp_path, ref, fmt):
    """Our writer and the reference's own write_mask produce identical DRBM
    files, and the reference's read_mask reads ours (oracle/_ref).  (The
    CSV / PGM writers use formatted iostream output, which crashes when the
    in-place reference build is dlopen'ed next to this interpreter's
    libstdc++; those two formats are pinned by test_csv_and_pgm.)"""
    m = rp.read_mask(os.path.join(GOLDEN, "wan_cfg3.drbm"))
    ours, theirs = tmp_path / f"o.{fmt}", tmp_path / f"r.{fmt}"
    rp.write_mask(m, rp.MaskFormat(fmt), str(ours))
    ref.write_mask(m.bits, m.dim, fmt, str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
    if fmt == 0:
        dim, bits = ref.read_mask(str(ours))
        assert dim == m.dim and np.array_equal(bits, m.bits)


def test_production_goldens_are_consistent():
    """The production-scale dynamic goldens (reference build_mask output,
    tests/golden/make_golden_production.py) parse as DRBM and carry the
    active-block counts recorded with them."""
    import json
    import os

    from golden_util import GOLDEN, read_drbm
    with open(os.path.join(GOLDEN, "production_meta.json")) as f:
        meta = json.load(f)
    for name, m in meta.items():
        dim, bits = read_drbm(os.path.join(GOLDEN, f"{name}_mid.drbm"))
        nb = (m["nf"] * m["nt"] + m["bs"] - 1) // m["bs"]
        assert dim == nb
        assert int(np.unpackbits(bits, axis=1, bitorder="little")[:, :dim].sum()) == m["nnz"]
    assert meta["hunyuan"]["nnz"] == 567038
