"""Golden token masks from the reference's own expand_mask (mask.cpp:52-66),
run through oracle/_ref: block masks of the reference's build_mask (static
and dynamic) plus random masks, on grids with and without padding and for
B in {4, 8, 16, 32, 64, 128}.  Writes expand_mask.npz (bits_<i>, token_<i>,
grid_<i> = (nf, nt, bs)).

    python tests/golden/make_golden_expand.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import pyoracle  # noqa: E402
from oracle.pyoracle import Cfg  # noqa: E402


def main():
    R = pyoracle.ref()
    rng = np.random.default_rng(3)
    out = {}
    cases = [((4, 300, 128), "static"), ((3, 100, 16), "static"), ((2, 64, 4), "dynamic"),
             ((5, 37, 8), "random"), ((2, 1000, 64), "random"), ((6, 50, 32), "dynamic"),
             ((1, 129, 128), "random")]
    for i, ((nf, nt, bs), kind) in enumerate(cases):
        _, _, nb, rb = pyoracle.grid_dims(nf, nt, bs)
        if kind == "static":
            bits = R.build_mask(nf, nt, bs, Cfg(0, 2.0, 0.3, 1e-6, 0.75, 0.2, 0.3, 0.3, 1), 7)
        elif kind == "dynamic":
            q, k, _ = R.random_batch(nf * nt, 2, 16, 5, with_values=False)
            bits = R.build_mask(nf, nt, bs, Cfg(1, 1.4, 0.7, 1e-6, 0.5, 0.3, 0.0, 0.3, 1), 7,
                                False, q, k)
        else:
            dense = (rng.random((nb, nb)) < 0.3).astype(np.uint8)
            bits = pyoracle.pack_dense(dense)
        out[f"grid_{i}"] = np.array([nf, nt, bs])
        out[f"bits_{i}"] = bits
        out[f"token_{i}"] = R.expand_mask(nf, nt, bs, bits)
    np.savez_compressed(os.path.join(HERE, "expand_mask.npz"), n=len(cases), **out)


if __name__ == "__main__":
    main()
