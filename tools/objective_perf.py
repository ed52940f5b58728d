"""SURVEY 8f3 measurement: the profiler objective on the GPU vs the C
restatement (bit-identical to the reference's profiler.cpp) on the host.

GPU: cache build (two passes of the S x S x dim float GEMM + fp64 exp) and one
trial (mask build + block-statistics error) per config, CUDA-event timed.
CPU: the restatement's objective (its own cache, as the reference's
objective(..., cache=nullptr)) and a trial given the cache, on the same grid
where it finishes in seconds; larger grids are extrapolated by S^2 and marked.
Writes one JSON object (stdout, and to the path given as argv[1]).
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle  # noqa: E402
from oracle.pyoracle import Cfg  # noqa: E402
from bench import ClockSampler  # noqa: E402
from paper_2604_20470_b200 import radialplan as rp  # noqa: E402

GRIDS = [("cli_default_16x64_b16", 16, 64, 16, 64),
         ("wan_21x3600_b128", 21, 3600, 128, 64)]
STATIC = (0, 1.5, 0.5, 1e-6, 0.6, 0.3, 0.5, 0.3, 1)
DYNAMIC = (1, 1.5, 0.5, 1e-6, 0.6, 0.3, 0.0, 1.0, 1)


def cfg_rp(c):
    return rp.SparsityConfig(rp.Mode(int(c[0])), rp.RadialParams(c[1], c[2], c[3]), c[4], c[5],
                             c[6], c[7], int(c[8]))


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def _cpu_objective(lib, nf, nt, bs, fh, threads):
    c = Cfg(*STATIC[:8], STATIC[8])
    if lib.kind == "reference":
        return lib.objective(nf, nt, bs, c, fh, 5)
    return lib.objective(nf, nt, bs, c, fh, 5, threads=threads)


def main():
    # CPU side: the reference's own profiler objective (oracle/_ref, single
    # threaded, its own S x S cache) when built, else the C restatement
    port = pyoracle.ref() if pyoracle.have_ref() else pyoracle.port()
    kind = "reference (oracle/_ref)" if pyoracle.have_ref() else "C restatement"
    threads = 1 if pyoracle.have_ref() else (os.cpu_count() or 1)
    out = {"what": "profiler objective (SURVEY 8f3), GPU trial vs CPU objective", "cpu_threads": threads,
           "grids": []}
    for name, nf, nt, bs, dim in GRIDS:
        g = rp.make_grid(nf, nt, bs)
        n = nf * nt
        gen = torch.Generator(device="cuda").manual_seed(1)
        f = (torch.randn(n, dim, device="cuda", generator=gen) * 0.5).contiguous()
        holder = {}

        def build():
            if "c" in holder:
                holder["c"].close()
            holder["c"] = rp.ProxyCache(g, f)
        with ClockSampler(0) as clk:
            cache_ms = timed(build, 3)
            cache = holder["c"]
            st = timed(lambda: cache.objective(cfg_rp(STATIC), 5), 5)
            dy = timed(lambda: cache.objective(cfg_rp(DYNAMIC), 5, features=f), 3)
        rec = {"grid": name, "tokens": n, "feature_dim": dim, "gpu_cache_build_ms": cache_ms,
               "gpu_trial_static_ms": st, "gpu_trial_dynamic_ms": dy,
               "cache_bytes": n * ((n + bs - 1) // bs) * 16 + n * 20,
               "reference_cache_bytes": n * n * 4 + n * 8, "clocks": clk.summary(),
               "cpu_kind": kind}
        fh = f.cpu().numpy()
        if n <= 4096:
            t0 = time.time()
            _cpu_objective(port, nf, nt, bs, fh, threads)
            rec["cpu_objective_s"] = time.time() - t0
            rec["cpu_sample"] = "full objective on this grid (restatement, own cache)"
        else:
            # bounded sample: a 21 x 400 grid, scaled by S^2
            sn = 21 * 400
            t0 = time.time()
            _cpu_objective(port, 21, 400, bs, fh[:sn], threads)
            dt = time.time() - t0
            rec["cpu_objective_s"] = dt * (n / sn) ** 2
            rec["cpu_sample"] = f"21x400 grid ({sn} tokens) timed {dt:.2f} s, scaled by (S/{sn})^2"
        rec["speedup_trial_static_vs_cpu_objective"] = rec["cpu_objective_s"] * 1e3 / st
        out["grids"].append(rec)
        cache.close()
        print(json.dumps(rec), flush=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fo:
            json.dump(out, fo, indent=1)


if __name__ == "__main__":
    main()
