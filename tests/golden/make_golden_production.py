"""Production-scale dynamic-mode golden masks from the reference's OWN build_mask.

BASELINE.json configs[3] (HunyuanVideo 61x45x80, B=128) and the Wan2.1
21x45x80 grid, both at Table-3 Mid (gamma 1.4, lambda 0.7, theta_m 0.7,
theta_c 0.45, tau -1.5 / 2.0), scored from H_f = 2 heads of d = 128:

  features = bf16_rne(random_batch(S, 2, 128, seed=42))  (attention.cpp:182-204)

i.e. exactly the values the bf16 GPU path sees (the reference receives the
same bf16 values widened to float).  Runs the reference sources
compiled in place (oracle/_ref) with RADIALPLAN_THREADS = all host cores and
writes

  hunyuan_mid.drbm, wan_mid.drbm   DRBM (mask.cpp:301-347)
  production_meta.json             inputs, nnz, BuildTimings, wall time,
                                   CPU model and thread count of the run

The GPU tests (tests/test_mask_gpu.py::test_production_*) regenerate the
same bf16 features on the device (rp_random_batch) and compare the tcgen05
scoring engine's mask with these files.

    python tests/golden/make_golden_production.py [hunyuan|wan|all]
"""
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402
from oracle.pyoracle import Cfg  # noqa: E402

MID = dict(mode=1, decay_factor=1.4, long_range_factor=0.7, split_epsilon=1e-6,
           mask_threshold=0.7, col_threshold=0.45, near_param=-1.5, far_param=2.0,
           fallback_k=1)
GRIDS = {"hunyuan": (61, 3600, 128), "wan": (21, 3600, 128)}
FEAT_SEED, MASK_SEED, HF, D = 42, 7, 2, 128


def bf16_rne(x):
    """Round float32 to bfloat16 (round to nearest even) and widen back."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def make(name, meta):
    R = pyoracle.ref()
    nf, nt, bs = GRIDS[name]
    S = nf * nt
    q, k, _ = R.random_batch(S, HF, D, FEAT_SEED, with_values=False)
    q, k = bf16_rne(q), bf16_rne(k)
    c = Cfg(**MID)
    threads = os.cpu_count() or 1
    os.environ["RADIALPLAN_THREADS"] = str(threads)
    tm = {}
    t0 = time.perf_counter()
    bits = R.build_mask(nf, nt, bs, c, MASK_SEED, False, q, k, timings=tm)
    wall = time.perf_counter() - t0
    blocks = bits.shape[0]
    R.write_mask(bits, blocks, 0, os.path.join(HERE, f"{name}_mid.drbm"))
    nnz = int(np.unpackbits(bits, axis=1, bitorder="little")[:, :blocks].sum())
    meta[name] = dict(nf=nf, nt=nt, bs=bs, cfg=MID, mask_seed=MASK_SEED,
                      features=dict(kind="bf16_rne(random_batch)", tokens=S, heads=HF, d=D,
                                    seed=FEAT_SEED),
                      nnz=nnz, block_sparsity=1 - nnz / float(blocks * blocks),
                      wall_s=wall, threads=threads, cpu=cpu_model(), timings=tm,
                      build="oracle/_ref (reference src/*.cpp -O3 -DNDEBUG, in place)")
    print(name, json.dumps(meta[name]), flush=True)


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    path = os.path.join(HERE, "production_meta.json")
    meta = json.load(open(path)) if os.path.exists(path) else {}
    for name in (["wan", "hunyuan"] if which == "all" else [which]):
        make(name, meta)
        with open(path, "w") as f:
            json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
