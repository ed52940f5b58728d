"""The reference's own build_mask (oracle/_ref) at FULL size on this host's
cores, for the two benched configs (Wan static config 3, Hunyuan dynamic
Table-3 Mid on bf16 random_batch scoring heads): wall time, BuildTimings,
CPU model, threads.  Writes profiles/r2_cpu_reference_build_mask.json (run on
the GPU box, whose host cores are the bench's CPU baseline).  ~5-10 min."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, FEATURE_SEED, cpu_model  # noqa: E402
from oracle import pyoracle  # noqa: E402


def bf16_rne(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def main(out_path):
    R = pyoracle.ref()
    threads = os.cpu_count() or 1
    os.environ["RADIALPLAN_THREADS"] = str(threads)
    res = {"cpu": cpu_model(), "threads": threads}
    for name in ("wan_static", "hunyuan_dynamic"):
        c = CONFIGS[name]
        gm, gl, tm, tc, a, b = c["cfg"]
        cfg = pyoracle.Cfg(c["mode"], gm, gl, 1e-6, tm, tc, a, b, 1)
        q = k = None
        if c["mode"] == 1:
            q, k, _ = pyoracle.port().random_batch(c["nf"] * c["nt"], 2, c["d"], FEATURE_SEED,
                                                   with_values=False, threads=threads)
            q, k = bf16_rne(q), bf16_rne(k)
        tmg = {}
        t0 = time.perf_counter()
        bits = R.build_mask(c["nf"], c["nt"], c["bs"], cfg, c["seed"], False, q, k, timings=tmg)
        wall = time.perf_counter() - t0
        nb = bits.shape[0]
        res[name] = {"wall_ms": wall * 1e3, "threads": threads, "cpu": res["cpu"],
                     "active_blocks": int(np.unpackbits(bits, axis=1,
                                                        bitorder="little")[:, :nb].sum()),
                     "build_timings_worker_s": tmg,
                     "note": "reference radialplan::build_mask (oracle/_ref) at full size, "
                             "measured (not extrapolated)"}
        print(name, json.dumps(res[name]), flush=True)
        with open(out_path, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out",
                                                            "r2_cpu_reference_build_mask.json"))
