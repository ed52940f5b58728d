"""Regenerate the golden fixtures from the reference's OWN code.

Runs the reference radialplan sources compiled in place (oracle/_ref, see
oracle/Makefile; needs /root/reference in this container) and writes:

  masks.json        tiny/small block masks (bit-packed, hex) for static and
                    dynamic configs, with the exact inputs that produced them
  wan_cfg3.drbm     Wan2.1 21x3600 B=128 static config-3 mask (SURVEY §8d:
                    gamma 1.0, lambda 0.1, theta_m 1.0, theta_c 0.2,
                    rho .3/.3, seed 7), DRBM format (mask.cpp:301-347)
  attn_small.npz    masked_attention_exact and soft-mask masked_attention
                    (eps 1e-10, 1e-3, 0.25, 4) outputs on a small padded grid

Features for dynamic cases are random_batch(S, H_f=2, d, seed) (the
reference's counter-based generator, attention.cpp:182-204), which the C
restatement reproduces bit for bit, so the GPU tests rebuild them without
the reference.

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402
from oracle.pyoracle import Cfg  # noqa: E402


def cfg_dict(c: Cfg):
    return dict(mode=c.mode, decay_factor=c.decay_factor, long_range_factor=c.long_range_factor,
                split_epsilon=c.split_epsilon, mask_threshold=c.mask_threshold,
                col_threshold=c.col_threshold, near_param=c.near_param, far_param=c.far_param,
                fallback_k=c.fallback_k)


def write_drbm(path, bits, dim):
    with open(path, "wb") as f:
        f.write(b"DRBM")
        f.write((1).to_bytes(2, "little"))
        f.write(int(dim).to_bytes(4, "little"))
        f.write(np.ascontiguousarray(bits, np.uint8).tobytes())


def read_drbm(path):
    """Reader written against the format description (mask.cpp:349-376)."""
    raw = open(path, "rb").read()
    assert raw[:4] == b"DRBM", "bad magic"
    assert int.from_bytes(raw[4:6], "little") == 1, "bad version"
    dim = int.from_bytes(raw[6:10], "little")
    rb = (dim + 7) // 8
    assert len(raw) == 10 + dim * rb, "payload size mismatch"
    return dim, np.frombuffer(raw[10:], np.uint8).reshape(dim, rb).copy()


def main():
    R = pyoracle.ref()
    cases = []

    def add(nf, nt, bs, c, seed, feats=None, disable_split=False):
        q = k = None
        if feats is not None:
            tok, h, d, fseed = feats
            q, k, _ = R.random_batch(tok, h, d, fseed, with_values=False)
        bits = R.build_mask(nf, nt, bs, c, seed, disable_split, q, k)
        dense = R.oracle_build(nf, nt, bs, c, seed, disable_split, q, k)
        agree = np.array_equal(pyoracle.unpack_bits(bits, dense.shape[0]), dense)
        # With disable_split, pruned pairs keep retained=false in the library
        # (radial.cpp:111-121), so a dynamic build scores nothing for them,
        # while tests/oracle.cpp scores the band; the library (build_mask) is
        # the reference path and the golden records its output.
        assert agree or (disable_split and c.mode == 1), \
            "reference library and reference oracle disagree"
        cases.append(dict(nf=nf, nt=nt, bs=bs, cfg=cfg_dict(c), seed=seed,
                          disable_split=disable_split, features=feats,
                          bits=bits.tobytes().hex(),
                          active=int(np.unpackbits(bits).sum()), oracle_agrees=bool(agree)))

    # configs[0]: tiny static: the throughput point and
    # the RNG-sensitive windows that exercise the Fisher-Yates stream.
    for bs in (16, 32, 64, 128):
        add(8, 256, bs, Cfg(0, 2.0, 0.3, 1e-6, 0.75, 0.2, 0.2, 0.2), 7)
    add(8, 256, 32, Cfg(0, 2.0, 0.3, 1e-6, 0.75, 0.2, 0.21, 0.21), 7)
    add(8, 256, 32, Cfg(0, 2.0, 0.3, 1e-6, 0.75, 0.2, 0.22, 0.22), 7)
    add(8, 256, 64, Cfg(0, 1.0, 1.0, 1e-6, 0.75, 0.2, 0.22, 0.22), 7)
    add(8, 256, 128, Cfg(0, 1.0, 1.0, 1e-6, 0.75, 0.2, 0.22, 0.22), 7)
    add(8, 250, 32, Cfg(0, 1.0, 1.0, 1e-6, 0.75, 0.2, 0.22, 0.22), 3)  # padded grid
    # configs[1]: tiny dynamic, z-threshold window + Table-3 Mid.
    for tau in (0.0, 0.05, 0.08):
        for bs in (32, 128):
            add(8, 256, bs, Cfg(1, 1.4, 0.7, 1e-6, 0.7, 0.45, tau, tau), 7, (2048, 2, 64, 42))
    add(8, 256, 32, Cfg(1, 1.4, 0.7, 1e-6, 0.7, 0.45, -1.5, 2.0), 7, (2048, 2, 64, 42))
    # fallback exercised at B=4 (fallback_k >= ceil(theta_c * B)).
    add(6, 12, 4, Cfg(1, 1.0, 1.0, 1e-6, 0.25, 0.25, 9.0, 9.0, 2), 11, (72, 2, 16, 5))
    add(6, 12, 4, Cfg(1, 1.7, 0.4, 1e-6, 0.5, 0.25, 3.5, 6.0, 3), 12, (72, 2, 8, 6))
    # disable_split with full bands / dynamic (never the crashing static case).
    add(8, 64, 8, Cfg(0, 1.5, 0.3, 1e-6, 0.5, 0.3, 1.0, 1.0), 5, None, True)
    add(8, 64, 8, Cfg(1, 1.5, 0.3, 1e-6, 0.5, 0.3, 0.5, 1.0), 5, (512, 2, 16, 9), True)

    with open(os.path.join(HERE, "masks.json"), "w") as f:
        json.dump(cases, f, indent=0)

    # Wan2.1 config 3 (static, bit-exact target at production scale).
    wan = Cfg(0, 1.0, 0.1, 1e-6, 1.0, 0.2, 0.3, 0.3)
    bits = R.build_mask(21, 3600, 128, wan, 7)
    write_drbm(os.path.join(HERE, "wan_cfg3.drbm"), bits, bits.shape[0])

    # Small stage-(d) golden: padded grid, 2 heads, d=32, exact and soft.
    nf, nt, bs = 4, 100, 32
    q, k, v = R.random_batch(nf * nt, 2, 32, 17)
    mbits = R.build_mask(nf, nt, bs, Cfg(0, 1.0, 1.0, 1e-6, 0.5, 0.2, 0.5, 0.5), 3)
    exact = R.masked_attention(nf, nt, bs, mbits, q, k, v, exact=True)
    soft = R.masked_attention(nf, nt, bs, mbits, q, k, v, exact=False)
    # soft mask at epsilons where inactive blocks carry visible mass
    soft_eps = np.array([1e-3, 0.25, 4.0])
    soft_multi = np.stack([R.masked_attention(nf, nt, bs, mbits, q, k, v, exact=False, eps=e)
                           for e in soft_eps])
    np.savez_compressed(os.path.join(HERE, "attn_small.npz"), nf=nf, nt=nt, bs=bs, seed=17,
                        bits=mbits, exact=exact, soft=soft, soft_eps=soft_eps,
                        soft_multi=soft_multi)
    print(f"{len(cases)} mask cases; wan cfg3 active={int(np.unpackbits(bits).sum())}")


if __name__ == "__main__":
    main()
