#!/usr/bin/env python
"""DynamicRad sparse-attention layer on B200 — the driver's benchmark contract.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--config wan_static|hunyuan_dynamic] [--gather]

A "step" is one attention layer's hot path over synthetic Q/K/V resident in
HBM.  The headline (top-level keys) is BASELINE.json configs[2]: Wan2.1-14B
720p, 21x45x80 = 75,600 tokens, 40 heads, d=128, bf16, static-ratio mask
gamma 1.0 lambda 0.1 theta_m 1.0 theta_c 0.2 rho .3/.3 seed 7 -> 80.6% block
sparsity, B=128.  In static mode the mask is built once and cached
(PAPER.md:769), so a layer is the block-sparse attention forward (stage d);
the one-time mask build is timed and reported beside it.  The same JSON line
carries a `hunyuan_dynamic` record: BASELINE.json configs[3] (HunyuanVideo
61x45x80 = 219,600 tokens, 24 heads, dynamic Table-3 Mid), whose layer
rebuilds the mask from its own Q/K every step (stages a-d).

Inputs are the reference's own synthetic batch, random_batch(S, H, 128,
seed 42) (attention.cpp:182-204), generated on the device and rounded to
bf16; so the benched Hunyuan mask IS the reference's golden mask
(tests/golden/hunyuan_mid.drbm, written by the reference's build_mask).

Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run) when
it is not already running under torchrun.  Heads are sharded across ranks
(stage d is head-independent, every rank holds the same static mask: no
data-path collective; dynamic mode splits the scoring across ranks and ORs
the bitmasks).  The timed region is bracketed by barriers and the reported
time is the max over ranks (strong scaling: the layer's work is fixed).
`--gather` also times the optional all-gather of the head-sharded outputs.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse-attn ms/layer & effective TFLOPS at Wan2.1-14B shape vs dense and CPU"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}

CONFIGS = {
    # BASELINE.json configs[2]
    "wan_static": dict(workload="Wan2.1-14B 720p 81f: 21x45x80=75600 tok, 40 heads, d=128, "
                                "bf16, static-ratio (SURVEY 8d config 3), B=128",
                       nf=21, nt=3600, bs=128, heads=40, d=128, mode=0,
                       cfg=(1.0, 0.1, 1.0, 0.2, 0.3, 0.3), seed=7, golden=None),
    # BASELINE.json configs[3]
    "hunyuan_dynamic": dict(workload="HunyuanVideo 241f: 61x45x80=219600 tok, 24 heads, d=128, "
                                     "bf16, dynamic-threshold Table-3 Mid (H_f=2), B=128",
                            nf=61, nt=3600, bs=128, heads=24, d=128, mode=1,
                            cfg=(1.4, 0.7, 0.7, 0.45, -1.5, 2.0), seed=7,
                            golden="tests/golden/hunyuan_mid.drbm"),
}
FEATURE_SEED = 42
N_SCORE_HEADS = 2


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """NVML samples of SM clock + throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------- reference arm --
def reference_sample(cfgd, threads):
    """The reference's own CPU implementation (oracle/_ref, else the C
    restatement) on a bounded sample of the layer: masked_attention_exact
    (single-threaded by design) on one frame's worth of tokens (N_f = 1)
    for `threads` heads run concurrently, one per core.  The reference is a
    dense O(S'^2) evaluator per head whatever the mask, so the layer time
    extrapolates as (S'_full / S'_sample)^2: "h_way" = ceil(H / threads)
    rounds of `threads` concurrent heads, "one_core" = H heads one after the
    other.  Dynamic mode adds the reference's build_mask (std::thread over
    frame pairs, all cores) on the first 5 frames, extrapolated by the token
    pairs it scores."""
    from oracle import pyoracle
    have_ref = pyoracle.have_ref()
    lib = pyoracle.ref() if have_ref else pyoracle.port()
    nf, nt, bs, H, d = 1, cfgd["nt"], cfgd["bs"], cfgd["heads"], cfgd["d"]
    heads = max(1, min(threads, H))
    padded = (nf * nt + bs - 1) // bs * bs
    nb = padded // bs
    bits = pyoracle.pack_dense(np.ones((nb, nb), np.uint8))  # the work is dense O(S'^2) anyway
    q, k, v = pyoracle.port().random_batch(nf * nt, heads, d, FEATURE_SEED, threads=threads)
    t0 = time.perf_counter()
    if have_ref:
        outs = [None] * heads

        def one(h):  # ctypes releases the GIL
            outs[h] = lib.masked_attention(nf, nt, bs, bits, q[:, h:h + 1].copy(),
                                           k[:, h:h + 1].copy(), v[:, h:h + 1].copy())
        ts = [threading.Thread(target=one, args=(h,)) for h in range(heads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    else:
        lib.masked_attention_exact(nf, nt, bs, bits, q, k, v, threads=threads)
    dt = time.perf_counter() - t0
    full_padded = (cfgd["nf"] * cfgd["nt"] + bs - 1) // bs * bs
    sq = (full_padded / padded) ** 2
    h_way = dt * sq * math.ceil(H / heads) * 1e3
    one_core = dt * sq * H * 1e3
    kind = "reference" if have_ref else "port"
    desc = (f"{'reference radialplan::masked_attention_exact (oracle/_ref)' if have_ref else 'C restatement (oracle port)'}"
            f" measured on N_f=1 ({padded} padded tokens) x {heads} heads concurrently "
            f"({dt:.2f} s), EXTRAPOLATED to the full layer by (S'/S'_sample)^2 = {sq:.0f}: "
            f"value = ideal {heads}-way over the host cores (x ceil(H/{heads}) rounds); "
            f"one_core_ms = the {H} heads one after the other")
    out = {"h_way_ms": h_way, "one_core_ms": one_core, "sample_s": dt}
    if cfgd["mode"] == 1:
        nf_s = 5
        gm, lm, tm, tc, a, b = cfgd["cfg"]
        cfg = pyoracle.Cfg(1, gm, lm, 1e-6, tm, tc, a, b, 1)
        qf, kf, _ = pyoracle.port().random_batch(nf_s * nt, 2, d, FEATURE_SEED, with_values=False,
                                                 threads=threads)
        os.environ["RADIALPLAN_THREADS"] = str(threads)
        tm_ = {}
        t1 = time.perf_counter()
        lib.build_mask(nf_s, nt, bs, cfg, cfgd["seed"], q=qf, k=kf, timings=tm_)
        dm = time.perf_counter() - t1
        full_pairs = scored_pairs(lib, cfgd["nf"], nt, bs, cfg)
        ratio = full_pairs / max(1, tm_.get("scored_pairs", 0))
        out["build_mask_ms"] = dm * ratio * 1e3
        out["h_way_ms"] += out["build_mask_ms"]
        out["one_core_ms"] += out["build_mask_ms"] * threads
        out["sample_s"] += dm
        desc += (f"; plus build_mask (dynamic, {threads} threads) measured on N_f={nf_s} "
                 f"({tm_.get('scored_pairs', 0)} token pairs scored, {dm:.1f} s), extrapolated "
                 f"x{ratio:.1f} to the layer's {full_pairs} scored pairs")
    out["desc"] = desc
    out["kind"] = kind
    return out


def scored_pairs(lib, nf, nt, bs, cfg):
    """Token pairs the reference scores in dynamic mode: the candidate bands
    of retained frame pairs at distance >= 2 (radial.cpp:56-62,
    selection.cpp:52-59)."""
    total = 0
    for i in range(nf):
        for j in range(nf):
            if abs(i - j) < 2:
                continue
            width, retained, count, tier, _ = lib.frame_pair(nf, nt, bs, cfg, i, j)
            if retained and tier >= 1:
                total += count
    return total


def reference_build_mask_full(cfgd, threads):
    """The reference's build_mask at FULL size (static mode: ~seconds), timed
    on the host cores: wall time, BuildTimings, CPU model, thread count."""
    from oracle import pyoracle
    if not pyoracle.have_ref():
        return None
    lib = pyoracle.ref()
    gm, lm, tm, tc, a, b = cfgd["cfg"]
    cfg = pyoracle.Cfg(cfgd["mode"], gm, lm, 1e-6, tm, tc, a, b, 1)
    os.environ["RADIALPLAN_THREADS"] = str(threads)
    timings = {}
    t0 = time.perf_counter()
    bits = lib.build_mask(cfgd["nf"], cfgd["nt"], cfgd["bs"], cfg, cfgd["seed"], timings=timings)
    wall = time.perf_counter() - t0
    nb = bits.shape[0]
    nnz = int(np.unpackbits(bits, axis=1, bitorder="little")[:, :nb].sum())
    return {"wall_ms": wall * 1e3, "threads": threads, "cpu": cpu_model(), "active_blocks": nnz,
            "build_timings_worker_s": timings, "kind": "reference (oracle/_ref)",
            "note": "measured at full size, not extrapolated"}


def run_reference(args, cfgd):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals, last = [], None
    for i in range(args.warmup + args.steps):
        last = reference_sample(cfgd, threads)
        if i >= args.warmup:
            vals.append(last["h_way_ms"])
    v = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "ms/layer",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 logits + f64 softmax (reference CPU)",
        "data": f"synthetic random_batch(S, H, {cfgd['d']}, seed {FEATURE_SEED})",
        "config": {"workload": cfgd["workload"], "parallelism": f"cpu x{threads} threads"},
        "extrapolated": True,
        "cpu_baseline": {"value": v, "unit": "ms/layer", "cores": threads, "kind": last["kind"],
                         "sample": last["desc"], "one_core_ms": float(last["one_core_ms"]),
                         "cpu": cpu_model()},
        "e2e": {"value": v, "unit": "ms/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- launch --
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_self_launch(args):
    """`--gpus N` outside torchrun: re-exec as N ranks of one node."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


# --------------------------------------------------------------- our arm --
class Ctx:
    """Per-process distributed / device context."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={self.world}")
        # validation mode: fewer GPUs than ranks (e.g. --gpus 2 on a 1-GPU
        # box, or DYNRAD_BENCH_SHARED_GPU=1): every rank on cuda:0 over gloo;
        # the N > 1 code path runs end to end but its timings mean nothing
        self.shared = (os.environ.get("DYNRAD_BENCH_SHARED_GPU") == "1"
                       or torch.cuda.device_count() < self.world)
        if self.shared:
            self.local = 0
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            if self.shared:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64,
                              device="cpu" if self.shared else self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())


def measure(args, ctx, cfgd, peaks, steps, full=True):
    """One configuration: mask build, timed layer steps, per-stage device
    times and rooflines, end-to-end host-buffer run, comparators."""
    torch = ctx.torch
    from paper_2604_20470_b200 import radialplan as rp
    from paper_2604_20470_b200.sharding import (broadcast_scoring_features, gather_heads,
                                                head_shards, or_allgather_mask)
    dev, world, rank = ctx.dev, ctx.world, ctx.rank
    H, d = cfgd["heads"], cfgd["d"]
    h0, Hl = head_shards(H, world)[rank]
    g = rp.make_grid(cfgd["nf"], cfgd["nt"], cfgd["bs"])
    gm, gl, tm, tc, a, b = cfgd["cfg"]
    cfg = rp.SparsityConfig(rp.Mode(cfgd["mode"]), rp.RadialParams(gm, gl), tm, tc, a, b)
    S = g.total_tokens
    nb = g.blocks_per_dim
    dynamic = cfgd["mode"] == 1
    stream = torch.cuda.Stream(device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    # this rank's heads of the layer's random_batch (the reference's features)
    fb = rp.random_batch(S, Hl, d, FEATURE_SEED, first_head=h0, device=dev, stream=stream)
    q, k, v = fb.queries, fb.keys, fb.values
    out = torch.empty((g.padded_tokens, Hl, d), device=dev, dtype=torch.bfloat16)
    stream.synchronize()

    plan = rp.Plan(g, cfg, cfgd["seed"],
                   rp.BuildOptions(shard_index=rank, shard_count=world) if dynamic else None)
    score_bufs = None
    if dynamic and world > 1:
        score_bufs = (torch.empty((S, N_SCORE_HEADS, d), dtype=torch.bfloat16, device=dev),
                      torch.empty((S, N_SCORE_HEADS, d), dtype=torch.bfloat16, device=dev))

    def build_dynamic(out_mask=None):
        if world == 1:
            return plan.build_mask_device(q, k, N_SCORE_HEADS, out=out_mask, stream=stream)
        qs, ks = broadcast_scoring_features(q, k, N_SCORE_HEADS, src=0, out=score_bufs)
        m = plan.build_mask_device(qs, ks, N_SCORE_HEADS, out=out_mask, stream=stream)
        return or_allgather_mask(m)

    # ---- one-time mask build (static: cached afterwards) ----------------------
    # A tiny build of the same mode first, untimed: CUDA loads kernel modules
    # lazily on their first launch, a per-process cost that is not the
    # mask build's.
    with torch.cuda.stream(stream):
        gw = rp.make_grid(2, 256, cfgd["bs"])
        pw = rp.Plan(gw, cfg, cfgd["seed"])
        if dynamic:
            fw = torch.zeros((gw.total_tokens, N_SCORE_HEADS, d), dtype=torch.bfloat16, device=dev)
            mw = pw.build_mask_device(fw, fw, N_SCORE_HEADS, stream=stream)
        else:
            mw = pw.build_mask_device(stream=stream)
        rp.mask_to_csr(gw, mw, stream=stream)
    stream.synchronize()
    # ... and one full-size build of another plan (seed + 1), timed on its
    # own: the process's stream-ordered pool grows to the build's scratch
    # here (seconds on some boxes), so mask_build_ms_one_time below is a new
    # plan's first build in a warm process and this is the first in the process.
    pf = rp.Plan(g, cfg, cfgd["seed"] + 1,
                 rp.BuildOptions(shard_index=rank, shard_count=world) if dynamic else None)
    f0, f1 = ev(), ev()
    with torch.cuda.stream(stream):
        f0.record(stream)
        mf = (pf.build_mask_device(q, k, N_SCORE_HEADS, stream=stream) if dynamic and world == 1
              else pf.build_mask_device(stream=stream) if not dynamic else None)
        f1.record(stream)
    stream.synchronize()
    first_in_process_ms = f0.elapsed_time(f1) if mf is not None else None
    del pf, mf
    e0, e1 = ev(), ev()
    build_stats = {}
    with torch.cuda.stream(stream):
        e0.record(stream)
        if dynamic:
            mask = build_dynamic()
        else:
            mask = plan.build_mask_device(stream=stream)
        row_ptr, col_idx, order = rp.mask_to_csr(g, mask, stream=stream)
        e1.record(stream)
    stream.synchronize()
    mask_build_ms = e0.elapsed_time(e1)
    nnz = int(col_idx.numel())
    sparsity = 1.0 - nnz / float(nb * nb)
    golden_equal = None
    if cfgd.get("golden") and os.path.exists(os.path.join(ROOT, cfgd["golden"])):
        raw = open(os.path.join(ROOT, cfgd["golden"]), "rb").read()
        want = np.frombuffer(raw[10:], np.uint8).reshape(nb, g.row_bytes)
        golden_equal = bool(np.array_equal(mask.cpu().numpy(), want))
    if dynamic:
        # scored pairs of this rank's share (for the scoring roofline)
        plan.build_mask_device(q if world == 1 else score_bufs[0],
                               k if world == 1 else score_bufs[1], N_SCORE_HEADS,
                               out=torch.empty_like(mask), stats=build_stats, stream=stream)

    csr_bufs = None
    if dynamic:
        csr_bufs = (torch.empty(nb + 1, dtype=torch.int32, device=dev),
                    torch.empty(nb * nb, dtype=torch.int32, device=dev),
                    torch.empty(nb, dtype=torch.int32, device=dev),
                    torch.zeros(1, dtype=torch.int64, device=dev))

    def layer(mark=None):
        nonlocal row_ptr, col_idx, order
        if dynamic:
            build_dynamic(out_mask=mask)
            row_ptr, col_idx, order = rp.mask_to_csr(g, mask, stream=stream, out=csr_bufs)
        if mark is not None:
            mark[0].record(stream)
        rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order, out=out, stream=stream)
        if mark is not None:
            mark[1].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            layer()
    stream.synchronize()
    ctx.barrier()
    torch.cuda.synchronize()
    starts = [ev() for _ in range(steps)]
    ends = [ev() for _ in range(steps)]
    marks = [(ev(), ev()) for _ in range(steps)]
    launches0 = rp.kernel_launch_count()
    rp.profile_stages(True)
    with ClockSampler(ctx.local) as clk:
        with torch.cuda.stream(stream):
            for i in range(steps):
                starts[i].record(stream)
                layer(marks[i])
                ends[i].record(stream)
        stream.synchronize()
    launches = rp.kernel_launch_count() - launches0
    torch.cuda.synchronize()
    ctx.barrier()
    stages = rp.profile_read()
    rp.profile_stages(False)
    per_step = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = starts[0].elapsed_time(ends[-1])
    ms = ctx.max_over_ranks(total_ms / steps)
    k6_ms = [x.elapsed_time(y) for x, y in marks]  # stage (d) alone, same stream
    k6_mean = float(np.mean(k6_ms))
    flops_alg = 4.0 * H * d * cfgd["bs"] ** 2 * nnz
    flops_local = 4.0 * Hl * d * cfgd["bs"] ** 2 * nnz
    flops_dense_eq = 4.0 * H * d * float(S) ** 2
    kernel_tflops = flops_local / (k6_mean * 1e-3) / 1e12
    peak = peaks["bf16_tflops"]
    kname = rp.attention_kernel(g, "bf16", d)
    # DRAM traffic per launch from the one ncu --set full capture of this
    # kernel at this config (null when none was taken)
    prof = {("wan_static", "bsfa_fwd_db_kernel<128>"): "r2_k6db_wan_ncu_summary.json",
            ("hunyuan_dynamic", "bsfa_fwd_rp_kernel<128>"): "r2_k6rp_hunyuan_ncu_summary.json"}
    key = "wan_static" if not dynamic else "hunyuan_dynamic"
    traffic = None
    pf = prof.get((key, kname))
    if pf and os.path.exists(os.path.join(ROOT, "profiles", pf)):
        with open(os.path.join(ROOT, "profiles", pf)) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    stage_ms = {name: tot / max(1, cnt) for name, (tot, cnt) in stages.items()}
    rec = {
        "value": ms, "unit": "ms/layer", "ms_per_step": ms, "steps": steps,
        "config": {"workload": cfgd["workload"], "global_heads": H, "heads_this_rank": Hl,
                   "seq_len": S, "padded_tokens": g.padded_tokens, "block_size": cfgd["bs"],
                   "mask_active_blocks": nnz, "block_sparsity": round(sparsity, 4),
                   "parallelism": f"head-sharded x{world}" + (
                       " (static mask cached on every rank: no collective)" if not dynamic
                       else " (split scoring: broadcast of the 2 scoring heads + OR "
                            "all-gather of the bitmask)" if world > 1 else ""),
                   "l2": f"inputs larger than L2 (Q/K/V {3 * S * H * d * 2 / 1e9:.1f} GB bf16 "
                         "per layer)"},
        "effective_tflops": flops_dense_eq / (ms * 1e-3) / 1e12,
        "algorithmic_tflops": flops_alg / (ms * 1e-3) / 1e12,
        "mask_build_ms_one_time": mask_build_ms,
        "mask_build_ms_first_in_process": first_in_process_ms,
        "mask_build_note": "one_time: this plan's first build (plan scratch allocated, "
                           "Fisher-Yates or scoring, row lists) in a warm process; "
                           "first_in_process: the same for another seed before it, which "
                           "also grows the stream-ordered pool (kernel modules loaded by an "
                           "untimed tiny build)",
        "roofline": {"bound": "tensor", "achieved": kernel_tflops, "peak": peak,
                     "unit": "TFLOP/s", "frac": kernel_tflops / peak, "traffic": traffic,
                     "kernel": kname + " (stage d)", "kernel_ms": k6_mean,
                     "per_launch": f"4*H*d*B^2*nnz = {flops_local / 1e12:.2f} TFLOP on the "
                                   f"{nnz} active blocks x {Hl} heads",
                     "algorithmic_bytes": 4 * S * Hl * d * 2,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)"},
        "roofline_sustained_frac": kernel_tflops / peaks.get("bf16_tflops_sustained", peak),
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "stages_ms": {"per_stage_device_ms": stage_ms,
                      "attention_stage_d": k6_mean,
                      "mask_stages_a_c_plus_csr": float(np.mean(per_step) - k6_mean)
                      if dynamic else 0.0,
                      "note": "static: mask cached per (grid, config, seed), built once "
                              "(mask_build_ms_one_time)" if not dynamic else
                              "dynamic: mask rebuilt from the layer's Q/K every step; "
                              "per_stage_device_ms from library CUDA events (rp_profile_stages)"},
        "per_step_ms": {"min": float(min(per_step)), "median": float(np.median(per_step)),
                        "max": float(max(per_step))},
    }
    if golden_equal is not None:
        rec["mask_equals_reference_golden"] = golden_equal
    if dynamic:
        # stage (b) on the tensor pipe: 2 * d * H_f flops per scored band pair
        # per pass; each pass runs over every scored pair
        sp = build_stats.get("scored_pairs", 0)
        alg = 2.0 * d * N_SCORE_HEADS * sp
        rec["scoring_roofline"] = {}
        for name in ("score_stats", "score_select"):
            t = stage_ms.get(name)
            if t:
                ach = alg / (t * 1e-3) / 1e12
                rec["scoring_roofline"][name] = {
                    "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                    "frac": ach / peak, "kernel_ms": t,
                    "per_launch": f"2*d*H_f*P_band = {alg / 1e12:.2f} TFLOP "
                                  f"({sp} scored token pairs on this rank)"}
        rec["build_stats"] = build_stats
        # stages (a) K5 and (c) on HBM: latency-bound at these
        # sizes, so the microseconds are the figure; the fraction is the
        # algorithmic bytes over the measured HBM bandwidth
        hbm = peaks["hbm_gbs"]
        nbk = g.blocks_per_dim
        mask_bytes = nbk * g.row_bytes
        stage_bytes = {
            # bitmask read; row_ptr, col_idx, row order written
            "csr": mask_bytes + 4 * (nbk + 1) + 4 * nnz + 4 * nbk,
            # per-tile column counts read, mask written, mu / sigma per frame pair
            "apply": mask_bytes + 16 * build_stats.get("retained_frame_pairs", 0),
            # Q'/K' of the scoring heads read once, per-token norms written
            "mask_prep": 2 * S * N_SCORE_HEADS * d * 2 + 2 * g.padded_tokens * 4,
        }
        rec["hbm_stage_rooflines"] = {}
        for name, b in stage_bytes.items():
            t = stage_ms.get(name)
            if t:
                rec["hbm_stage_rooflines"][name] = {
                    "bound": "hbm", "us": t * 1e3, "algorithmic_bytes": int(b),
                    "achieved": b / (t * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": b / (t * 1e-3) / 1e9 / hbm}

    # ---- optional all-gather of the head-sharded outputs ----------------------
    if args.gather and world > 1:
        torch.cuda.synchronize()
        ctx.barrier()
        t0g = time.perf_counter()
        ga, gb = ev(), ev()
        ga.record()
        for _ in range(3):
            full_out = gather_heads(out, H)
        gb.record()
        torch.cuda.synchronize()
        gather_ms = ctx.max_over_ranks(ga.elapsed_time(gb) / 3 if not ctx.shared else
                                       (time.perf_counter() - t0g) * 1e3 / 3)
        rec["gather_ms"] = gather_ms
        rec["value_with_gather"] = ms + gather_ms
        del full_out
    elif args.gather:
        rec["gather_ms"] = 0.0
        rec["value_with_gather"] = ms

    # ---- end to end from host buffers (rp_sparse_layer_host) ------------------
    if not args.no_e2e and (not dynamic or world == 1):
        qh = q.cpu().pin_memory()
        kh = k.cpu().pin_memory()
        vh = v.cpu().pin_memory()
        oh = torch.empty((g.padded_tokens, Hl, d), dtype=torch.bfloat16).pin_memory()
        nsc = N_SCORE_HEADS if dynamic else 0
        rp.sparse_layer_host(plan, qh, kh, vh, nsc, out=oh, stream=stream)
        n_e2e = max(3, min(steps, 5))
        ctx.barrier()
        a0, a1 = ev(), ev()
        a0.record(stream)
        for _ in range(n_e2e):
            rp.sparse_layer_host(plan, qh, kh, vh, nsc, out=oh, stream=stream)
        a1.record(stream)
        stream.synchronize()
        e2e_ms = ctx.max_over_ranks(a0.elapsed_time(a1) / n_e2e)
        e2e_ok = bool(torch.equal(oh[:S].to(dev), out[:S])) if world == 1 else None
        rec["e2e"] = {"value": e2e_ms, "unit": "ms/layer",
                      "h2d_bytes_per_step": int(3 * S * H * d * 2),
                      "d2h_bytes_per_step": int(g.padded_tokens * H * d * 2),
                      "path": "rp_sparse_layer_host: pinned host Q/K/V -> head-chunked H2D -> "
                              + ("mask rebuilt from the scoring heads (stages a-c) -> "
                                 if dynamic else "plan-cached static mask -> ")
                              + "row lists -> stage (d) per chunk -> D2H of O, per rank",
                      "output_equals_device_path": e2e_ok}
        del qh, kh, vh, oh

    # ---- dense references on the same GPU (rank 0) ----------------------------
    if full and not args.no_dense and rank == 0:
        full_np = np.packbits(np.ones((nb, nb), np.uint8), axis=1, bitorder="little")
        dense_mask = torch.from_numpy(full_np).to(dev)
        rpd, cid, ordd = rp.mask_to_csr(g, dense_mask, stream=stream)
        b0, b1 = ev(), ev()
        with torch.cuda.stream(stream):
            rp.sparse_attention(g, q, k, v, rpd, cid, ordd, out=out, stream=stream)
            b0.record(stream)
            for _ in range(2):
                rp.sparse_attention(g, q, k, v, rpd, cid, ordd, out=out, stream=stream)
            b1.record(stream)
        stream.synchronize()
        dense_ours = b0.elapsed_time(b1) / 2 * (H / Hl)
        qs = q.permute(1, 0, 2).unsqueeze(0)
        ks = k.permute(1, 0, 2).unsqueeze(0)
        vs = v.permute(1, 0, 2).unsqueeze(0)
        with torch.cuda.stream(stream):
            torch.nn.functional.scaled_dot_product_attention(qs, ks, vs)
            b0.record(stream)
            for _ in range(2):
                torch.nn.functional.scaled_dot_product_attention(qs, ks, vs)
            b1.record(stream)
        stream.synchronize()
        sdpa = b0.elapsed_time(b1) / 2 * (H / Hl)
        rec["dense"] = {"ours_dense_ms": dense_ours, "sdpa_dense_ms": sdpa,
                        "sdpa_dense_tflops": flops_dense_eq / (sdpa * 1e-3) / 1e12,
                        "speedup_vs_sdpa_dense": sdpa / ms, "speedup_vs_ours_dense": dense_ours / ms,
                        "note": "full layer (all heads) dense bf16 attention on this GPU; SDPA = "
                                "torch scaled_dot_product_attention (cuDNN/flash backend)"}
        del rpd, cid, ordd, dense_mask

    # ---- static mask: warm rebuild -------------------------------------------
    if not dynamic and rank == 0 and not args.no_rebuild:
        ts = []
        for _ in range(3):
            w0, w1 = ev(), ev()
            with torch.cuda.stream(stream):
                w0.record(stream)
                p2 = rp.Plan(g, cfg, cfgd["seed"])
                m2 = p2.build_mask_device(stream=stream)
                w1.record(stream)
            stream.synchronize()
            ts.append(w0.elapsed_time(w1))
            assert torch.equal(m2, mask)
            del p2, m2
        rec["static_mask_build_ms_warm"] = min(ts)

    # ---- library block-sparse kernels on the same mask ----------
    if full and not args.no_lib and rank == 0:
        rec["library_comparator"] = library_comparators(rp, g, q, k, v, mask, row_ptr, col_idx,
                                                        order, out, k6_mean, H, Hl, d, stream)

    # ---- the north star's pooled selector on the same Q/K -------
    if dynamic and rank == 0 and full:
        rec["pooled_selector_f1"] = pooled_record(rp, g, cfg, q, k, mask, peaks, stream)
    del q, k, v, out, fb
    torch.cuda.empty_cache()
    return rec


def library_comparators(rp, g, q, k, v, mask, row_ptr, col_idx, order, out, ours_ms, H, Hl, d,
                        stream):
    """FlashInfer's BSR block-sparse wrapper and FlashAttention-4's
    block-sparse sm100 kernel (tools/fa4_compare.py) on the same inputs."""
    import torch
    res = {}
    S = g.total_tokens
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    ours_layer = ours_ms * (H / Hl)
    try:
        import flashinfer
        Sp = g.padded_tokens
        pads = []
        for t in (q, k, v):  # FlashInfer needs N % C == 0: zero rows = the reference padding
            x = torch.zeros((Sp, Hl, d), dtype=torch.bfloat16, device=q.device)
            x[:S] = t
            pads.append(x)
        indptr, indices = rp.mask_to_bsr(g, mask)
        ws = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=q.device)
        wr = flashinfer.BlockSparseAttentionWrapper(ws)
        t0 = time.time()
        wr.plan(indptr, indices, Sp, Sp, g.block_size, g.block_size, Hl, Hl, d,
                q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16,
                o_data_type=torch.bfloat16)
        fo = wr.run(*pads)
        torch.cuda.synchronize()
        first = time.time() - t0
        with torch.cuda.stream(stream):
            wr.run(*pads)
            b0, b1 = ev(), ev()
            b0.record(stream)
            for _ in range(3):
                wr.run(*pads)
            b1.record(stream)
        stream.synchronize()
        fi_ms = b0.elapsed_time(b1) / 3 * (H / Hl)
        rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order, out=out, stream=stream)
        stream.synchronize()
        a, b = out[:S].float(), fo[:S].float()
        rel = float(((a - b).norm(dim=-1) / b.norm(dim=-1).clamp_min(1e-30)).max())
        res["flashinfer"] = {"library": f"flashinfer {flashinfer.__version__} "
                                        "BlockSparseAttentionWrapper (BSR, R=C=B)",
                             "library_ms": fi_ms, "ours_stage_d_ms": ours_layer,
                             "speedup_vs_library": fi_ms / ours_layer, "max_row_rel_diff": rel,
                             "library_first_call_s": first}
        del pads, ws, wr, fo
    except Exception as exc:  # noqa: BLE001 - comparator only: never fails the bench
        res["flashinfer"] = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import fa4_compare
        res["fa4"] = fa4_compare.compare(g, q, k, v, row_ptr, col_idx, order, H, Hl, d)
    except Exception as exc:  # noqa: BLE001
        res["fa4"] = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    torch.cuda.empty_cache()
    return res


def pooled_record(rp, g, cfg, q, k, mask, peaks, stream):
    import torch
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    S, d = g.total_tokens, q.shape[2]
    with torch.cuda.stream(stream):
        pm = torch.empty_like(mask)
        for _ in range(2):
            rp.pooled_select(g, cfg, q, k, 2, rp.PooledMode.Mass, 0.95, out=pm, stream=stream)
        b0, b1 = ev(), ev()
        b0.record(stream)
        for _ in range(5):
            rp.pooled_select(g, cfg, q, k, 2, rp.PooledMode.Mass, 0.95, out=pm, stream=stream)
        b1.record(stream)
    stream.synchronize()
    p_ms = b0.elapsed_time(b1) / 5
    with torch.cuda.stream(stream):
        pq = rp.block_mean_pool(g, q, 2, stream=stream)
        pk = rp.block_mean_pool(g, k, 2, stream=stream)
        b0.record(stream)
        for _ in range(5):
            rp.block_mean_pool(g, q, 2, out=pq, stream=stream)
            rp.block_mean_pool(g, k, 2, out=pk, stream=stream)
        b1.record(stream)
    stream.synchronize()
    pool_ms = b0.elapsed_time(b1) / 5
    alg = 2 * S * 2 * d * 2  # one read of the H_f = 2 heads of Q and K (bf16)
    nb = g.blocks_per_dim
    p_nnz = int(np.unpackbits(pm.cpu().numpy()).sum())
    return {"ms": p_ms, "mode": "cumulative softmax mass 0.95 over radial candidates, "
            "H_f=2 block-mean pooled Q/K (NOT reference semantics, SURVEY 8f1)",
            "stage_b_pool_ms": pool_ms, "stage_b_bytes": alg,
            "stage_b_achieved_gbs": alg / (pool_ms * 1e-3) / 1e9,
            "stage_b_hbm_frac": alg / (pool_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
            "stages_c_ms": p_ms - pool_ms,
            "block_sparsity": round(1 - p_nnz / float(nb * nb), 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="wan_static", choices=sorted(CONFIGS))
    ap.add_argument("--gather", action="store_true",
                    help="also time the all-gather of the head-sharded outputs (SURVEY 8e)")
    ap.add_argument("--no-dynamic", action="store_true",
                    help="skip the hunyuan_dynamic record of the default (wan_static) run")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-rebuild", action="store_true",
                    help="skip the warm static-mask rebuild measurement")
    ap.add_argument("--no-lib", action="store_true",
                    help="skip the FlashInfer / FA4 block-sparse comparators (SURVEY 8f2)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfgd = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfgd)
        return
    maybe_self_launch(args)
    ctx = Ctx(args)
    peaks, peaks_kind = load_peaks()
    rec = measure(args, ctx, cfgd, peaks, args.steps, full=True)
    dyn = None
    if args.config == "wan_static" and not args.no_dynamic:
        dyn = measure(args, ctx, CONFIGS["hunyuan_dynamic"], peaks, min(args.steps, 10),
                      full=True)

    cpu = None
    if not args.no_cpu and ctx.rank == 0 and ctx.world == 1:
        threads = os.cpu_count() or 1
        smp = reference_sample(cfgd, threads)
        cpu = {"value": smp["h_way_ms"], "unit": "ms/layer", "cores": threads,
               "kind": smp["kind"], "sample": smp["desc"], "sample_wall_s": smp["sample_s"],
               "one_core_ms": smp["one_core_ms"], "extrapolated": True, "cpu": cpu_model()}
        if cfgd["mode"] == 0:
            cpu["build_mask_full_size"] = reference_build_mask_full(cfgd, threads)
            cpu["build_mask_full_size_gpu_ms"] = {"one_time": rec["mask_build_ms_one_time"],
                                                  "warm": rec.get("static_mask_build_ms_warm")}
        if dyn is not None:
            ds = reference_sample(CONFIGS["hunyuan_dynamic"], threads)
            dyn["cpu_baseline"] = {"value": ds["h_way_ms"], "unit": "ms/layer", "cores": threads,
                                   "kind": ds["kind"], "sample": ds["desc"],
                                   "one_core_ms": ds["one_core_ms"], "extrapolated": True,
                                   "build_mask_ms_extrapolated": ds.get("build_mask_ms"),
                                   "cpu": cpu_model()}
            full_ref = os.path.join(ROOT, "profiles", "r2_cpu_reference_build_mask.json")
            if os.path.exists(full_ref):
                with open(full_ref) as f:
                    dyn["cpu_baseline"]["build_mask_full_size_measured"] = \
                        json.load(f).get("hunyuan_dynamic")

    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": rec["value"], "unit": "ms/layer", "n_gpus": ctx.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": rec["ms_per_step"],
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16",
            "data": f"synthetic: the reference's random_batch(S, H, 128, seed {FEATURE_SEED}) "
                    "(attention.cpp:182-204) generated on the device, rounded to bf16; each "
                    "rank takes its head slice",
        }
        if ctx.shared and ctx.world > 1:
            line["validation_only"] = ("ranks share one GPU over gloo (fewer GPUs than ranks): "
                                       "exercises the N>1 path, timings are not a measurement")
        for key in ("config", "effective_tflops", "algorithmic_tflops", "mask_build_ms_one_time",
                    "mask_build_ms_first_in_process", "mask_build_note",
                    "static_mask_build_ms_warm", "roofline", "roofline_sustained_frac", "clocks",
                    "gpu_launches", "e2e", "gather_ms", "value_with_gather", "dense",
                    "library_comparator", "stages_ms", "per_step_ms", "scoring_roofline",
                    "hbm_stage_rooflines", "build_stats", "mask_equals_reference_golden",
                    "pooled_selector_f1"):
            if key in rec:
                line[key] = rec[key]
        line["roofline"]["peak_source"] = f"{peaks_kind} bf16_tflops (burst)"
        line["cpu_baseline"] = cpu
        line["hunyuan_dynamic"] = dyn
        print(json.dumps(line), flush=True)
    if ctx.world > 1:
        ctx.dist.destroy_process_group()


if __name__ == "__main__":
    main()
