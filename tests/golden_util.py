"""Loading helpers for tests/golden (fixtures made by tests/golden/make_golden.py)."""
import json
import os

import numpy as np

from oracle.pyoracle import Cfg

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def mask_cases():
    with open(os.path.join(GOLDEN, "masks.json")) as f:
        cases = json.load(f)
    out = []
    for c in cases:
        nb = (c["nf"] * c["nt"] + c["bs"] - 1) // c["bs"]
        rb = (nb + 7) // 8
        bits = np.frombuffer(bytes.fromhex(c["bits"]), np.uint8).reshape(nb, rb).copy()
        out.append(dict(c, cfg=Cfg(**c["cfg"]), bits=bits, blocks=nb))
    return out


def case_id(c):
    f = c["cfg"]
    return (f"{'dyn' if f.mode else 'sta'}-{c['nf']}x{c['nt']}-B{c['bs']}-"
            f"{f.near_param:g}_{f.far_param:g}{'-nosplit' if c['disable_split'] else ''}")


def read_drbm(path):
    """DRBM reader written from the format description (mask.cpp:349-376)."""
    raw = open(path, "rb").read()
    if raw[:4] != b"DRBM":
        raise ValueError("bad magic")
    if int.from_bytes(raw[4:6], "little") != 1:
        raise ValueError("bad version")
    dim = int.from_bytes(raw[6:10], "little")
    rb = (dim + 7) // 8
    if len(raw) != 10 + dim * rb:
        raise ValueError("payload size mismatch")
    return dim, np.frombuffer(raw[10:], np.uint8).reshape(dim, rb).copy()


def features(port, spec):
    """random_batch(tokens, heads, d, seed) Q/K as float32 [S, H, d]."""
    if spec is None:
        return None, None
    tok, h, d, seed = spec
    q, k, _ = port.random_batch(tok, h, d, seed, with_values=False, threads=4)
    return q, k
