#!/usr/bin/env python
"""DynamicRad sparse-attention layer on B200 — the driver's benchmark contract.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--config wan_static|hunyuan_dynamic]

A "step" is one attention layer's hot path over synthetic Q/K/V resident in
HBM (BASELINE.json configs[2]: Wan2.1-14B 720p, 21x45x80 = 75,600 tokens,
40 heads, d=128, bf16, static-ratio mask gamma 1.0 lambda 0.1 theta_m 1.0
theta_c 0.2 rho .3/.3 seed 7 -> 80.6% block sparsity, B=128).  In static
mode the mask is built once and cached, so a layer is the
block-sparse attention forward (stage d); the one-time mask build is timed
and reported beside it.  hunyuan_dynamic (configs[3]) rebuilds the mask from
the layer's own Q/K every step (stages a-d).

Multi-GPU (torchrun, one rank per GPU): heads are sharded across ranks
(stage d is head-independent and every rank holds the same static mask), so
there is no data-path collective; the timed region is bracketed by barriers
and the reported time is the max over ranks (strong scaling: the layer's
total work is fixed).
"""
from __future__ import annotations

import argparse
import json
import math
import os
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
                       cfg=(1.0, 0.1, 1.0, 0.2, 0.3, 0.3), seed=7),
    # BASELINE.json configs[3]
    "hunyuan_dynamic": dict(workload="HunyuanVideo 241f: 61x45x80=219600 tok, 24 heads, d=128, "
                                     "bf16, dynamic-threshold Table-3 Mid (H_f=2), B=128",
                            nf=61, nt=3600, bs=128, heads=24, d=128, mode=1,
                            cfg=(1.4, 0.7, 0.7, 0.45, -1.5, 2.0), seed=7),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


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
def reference_sample(cfgd, threads, target_s=20.0):
    """The reference's own CPU implementation (oracle/_ref, else the C
    restatement) on a bounded sample of the layer: masked_attention_exact
    on one frame's worth of tokens (N_f = 1) for `threads` heads run
    concurrently (one head per core; the reference is single-threaded per
    call), extrapolated to the full layer by (S'_full / S'_sample)^2 *
    ceil(H / threads).  Returns (ms_per_layer_extrapolated, sample_s, desc)."""
    from oracle import pyoracle
    have_ref = pyoracle.have_ref()
    lib = pyoracle.ref() if have_ref else pyoracle.port()
    nf, nt, bs, H, d = 1, cfgd["nt"], cfgd["bs"], cfgd["heads"], cfgd["d"]
    heads = max(1, min(threads, H))
    padded = (nf * nt + bs - 1) // bs * bs
    nb = padded // bs
    bits = pyoracle.pack_dense(np.ones((nb, nb), np.uint8))  # work is dense O(S'^2) anyway
    q, k, v = pyoracle.port().random_batch(nf * nt, heads, d, 42, threads=threads)
    t0 = time.perf_counter()
    if have_ref:
        # one reference call per head, concurrently (ctypes releases the GIL)
        outs = [None] * heads
        def one(h):
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
    scale = (full_padded / padded) ** 2 * math.ceil(H / heads)
    desc = (f"{'reference radialplan::masked_attention_exact (oracle/_ref)' if have_ref else 'C restatement (oracle port)'}"
            f" on N_f=1 ({padded} padded tokens) x {heads} heads concurrently, "
            f"extrapolated x{scale:.0f} to the full layer by S'^2 * ceil(H/heads) "
            f"(the reference evaluates the expanded mask densely, O(S'^2))")
    ms = dt * scale * 1e3
    sample_s = dt
    if cfgd["mode"] == 1:
        # dynamic mode also rebuilds the mask every layer: the reference's
        # build_mask (std::thread over frame pairs, all host cores) on the
        # first nf_s frames with H_f = 2 scoring heads, extrapolated by the
        # ratio of token pairs scored (its own BuildTimings::scored_pairs).
        nf_s = 5
        gm, lm, tm, tc, a, b = cfgd["cfg"]
        cfg = pyoracle.Cfg(1, gm, lm, 1e-6, tm, tc, a, b, 1)
        qf, kf, _ = pyoracle.port().random_batch(nf_s * nt, 2, d, 42, with_values=False,
                                                 threads=threads)
        os.environ.setdefault("RADIALPLAN_THREADS", str(threads))
        tm_ = {}
        t1 = time.perf_counter()
        lib.build_mask(nf_s, nt, bs, cfg, cfgd["seed"], q=qf, k=kf, timings=tm_)
        dm = time.perf_counter() - t1
        full_pairs = scored_pairs(lib, cfgd["nf"], nt, bs, cfg)
        ratio = full_pairs / max(1, tm_.get("scored_pairs", 0))
        ms += dm * ratio * 1e3
        sample_s += dm
        desc += (f"; plus build_mask (dynamic, {threads} threads) on N_f={nf_s} "
                 f"({tm_.get('scored_pairs', 0)} token pairs scored, {dm:.1f} s) extrapolated "
                 f"x{ratio:.1f} to the layer's {full_pairs} scored pairs")
    return ms, sample_s, desc, ("reference" if have_ref else "port")


def scored_pairs(lib, nf, nt, bs, cfg):
    """Token pairs the reference scores in dynamic mode: the candidate bands
    of retained frame pairs at distance >= 2 (tier 0 takes the full band
    unscored), radial.cpp:56-62 / selection.cpp:52-59."""
    total = 0
    for i in range(nf):
        for j in range(nf):
            if abs(i - j) < 2:
                continue
            width, retained, count, tier, _ = lib.frame_pair(nf, nt, bs, cfg, i, j)
            if retained and tier >= 1:
                total += count
    return total


def run_reference(args, cfgd):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        ms, dt, desc, kind = reference_sample(cfgd, threads)
        if i >= args.warmup:
            vals.append(ms)
    v = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "ms/layer",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": v,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 logits + f64 softmax (reference CPU)", "data": "synthetic random_batch",
        "config": {"workload": cfgd["workload"], "parallelism": f"cpu x{threads} threads"},
        "cpu_baseline": {"value": v, "unit": "ms/layer", "cores": threads, "kind": kind,
                         "sample": desc},
        "e2e": {"value": v, "unit": "ms/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- our arm --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="wan_static", choices=sorted(CONFIGS))
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-rebuild", action="store_true",
                    help="skip the warm static-mask rebuild measurement")
    ap.add_argument("--no-lib", action="store_true",
                    help="skip the FlashInfer block-sparse comparator (SURVEY 8f2)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfgd = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfgd)
        return

    import torch
    import torch.distributed as dist

    from paper_2604_20470_b200 import radialplan as rp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DYNRAD_BENCH_SHARED_GPU=1 (validation only, never a reported number):
    # every rank on cuda:0 over gloo, so the N > 1 code path (head shards,
    # split scoring, broadcast / OR all-gather, max-over-ranks timing) can be
    # exercised on a one-GPU box.
    shared = os.environ.get("DYNRAD_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    peaks, peaks_kind = load_peaks()
    H, d = cfgd["heads"], cfgd["d"]
    from paper_2604_20470_b200.sharding import (broadcast_scoring_features, head_shards,
                                                or_allgather_mask)
    h0, Hl = head_shards(H, world)[rank]  # contiguous head shard per rank
    g = rp.make_grid(cfgd["nf"], cfgd["nt"], cfgd["bs"])
    gm, gl, tm, tc, a, b = cfgd["cfg"]
    cfg = rp.SparsityConfig(rp.Mode(cfgd["mode"]), rp.RadialParams(gm, gl), tm, tc, a, b)
    S = g.total_tokens
    stream = torch.cuda.Stream(device=dev)
    # The whole layer's Q/K/V from one seed on every rank, then this rank's
    # head slice: every N sees the same data (and so the same dynamic mask).
    gen = torch.Generator(device=dev).manual_seed(42)
    with torch.cuda.stream(stream):
        qkv = []
        for _ in range(3):
            full = torch.randn((S, H, d), device=dev, generator=gen).to(torch.bfloat16)
            qkv.append(full[:, h0:h0 + Hl].contiguous())
            del full
        q, k, v = qkv
        del qkv
        out = torch.empty((g.padded_tokens, Hl, d), device=dev, dtype=torch.bfloat16)
    stream.synchronize()

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    dynamic = cfgd["mode"] == 1
    # dynamic mode on N GPUs: split scoring (SURVEY 8e option 2) -- every rank
    # scores 1/N of the frame pairs from a broadcast copy of the H_f = 2
    # scoring heads, and the partial bitmasks are OR-combined
    plan = rp.Plan(g, cfg, cfgd["seed"],
                   rp.BuildOptions(shard_index=rank, shard_count=world) if dynamic else None)
    score_bufs = None
    if dynamic and world > 1:
        score_bufs = (torch.empty((S, 2, d), dtype=torch.bfloat16, device=dev),
                      torch.empty((S, 2, d), dtype=torch.bfloat16, device=dev))

    def build_dynamic(out=None):
        if world == 1:
            return plan.build_mask_device(q, k, 2, out=out, stream=stream)
        qs, ks = broadcast_scoring_features(q, k, 2, src=0, out=score_bufs)
        m = plan.build_mask_device(qs, ks, 2, out=out, stream=stream)
        return or_allgather_mask(m)

    # ---- one-time mask build (static: cached afterwards), timed -----------
    e0, e1 = ev(), ev()
    with torch.cuda.stream(stream):
        e0.record(stream)
        mask = build_dynamic() if dynamic else plan.build_mask_device(stream=stream)
        row_ptr, col_idx, order = rp.mask_to_csr(g, mask, stream=stream)
        e1.record(stream)
    stream.synchronize()
    mask_build_ms = e0.elapsed_time(e1)
    nnz = int(col_idx.numel())
    nb = g.blocks_per_dim
    sparsity = 1.0 - nnz / float(nb * nb)

    csr_bufs = None
    if dynamic:
        csr_bufs = (torch.empty(nb + 1, dtype=torch.int32, device=dev),
                    torch.empty(nb * nb, dtype=torch.int32, device=dev),
                    torch.empty(nb, dtype=torch.int32, device=dev),
                    torch.zeros(1, dtype=torch.int64, device=dev))

    def layer(mark=None):
        """One layer; `mark` (a pair of events) brackets the stage-(d) launch
        so its own duration feeds the roofline."""
        nonlocal row_ptr, col_idx, order
        if dynamic:
            build_dynamic(out=mask)
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
    barrier()
    torch.cuda.synchronize()
    starts = [ev() for _ in range(args.steps)]
    ends = [ev() for _ in range(args.steps)]
    marks = [(ev(), ev()) for _ in range(args.steps)]
    launches0 = rp.kernel_launch_count()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                starts[i].record(stream)
                layer(marks[i])
                ends[i].record(stream)
        stream.synchronize()
    launches = rp.kernel_launch_count() - launches0
    torch.cuda.synchronize()
    barrier()
    per_step = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = starts[0].elapsed_time(ends[-1])
    ms_local = total_ms / args.steps
    ms = max_over_ranks(ms_local)
    kern_ms = max_over_ranks(float(np.mean(per_step)))

    flops_alg = 4.0 * H * d * cfgd["bs"] ** 2 * nnz          # on active blocks (whole layer)
    flops_local = 4.0 * Hl * d * cfgd["bs"] ** 2 * nnz
    flops_dense_eq = 4.0 * H * d * float(S) ** 2             # dense-equivalent
    tflops_eff = flops_dense_eq / (ms * 1e-3) / 1e12
    tflops_alg = flops_alg / (ms * 1e-3) / 1e12
    k6_ms = [a.elapsed_time(b) for a, b in marks]  # stage (d) launch alone, same stream
    kernel_tflops = flops_local / (float(np.mean(k6_ms)) * 1e-3) / 1e12

    # ---- end to end through the host-buffer C ABI call ----------------------
    e2e = None
    if not args.no_e2e:
        import ctypes as C
        from paper_2604_20470_b200 import _lib
        qh = q.cpu().pin_memory()
        kh = k.cpu().pin_memory()
        vh = v.cpu().pin_memory()
        oh = torch.empty((g.padded_tokens, Hl, d), dtype=torch.bfloat16).pin_memory()
        mh = mask.cpu().pin_memory()
        gc = g.c()

        def e2e_call():
            _lib.check(_lib.lib().rp_masked_attention_exact_host(
                C.byref(gc), C.c_void_p(mh.data_ptr()), C.c_void_p(qh.data_ptr()),
                C.c_void_p(kh.data_ptr()), C.c_void_p(vh.data_ptr()), 1, S, Hl, d,
                C.c_void_p(oh.data_ptr()), C.c_void_p(stream.cuda_stream)))
        e2e_call()
        n_e2e = max(3, min(args.steps, 5))
        barrier()
        a0, a1 = ev(), ev()
        a0.record(stream)
        for _ in range(n_e2e):
            e2e_call()
        a1.record(stream)
        stream.synchronize()
        e2e_ms = max_over_ranks(a0.elapsed_time(a1) / n_e2e)
        e2e = {"value": e2e_ms, "unit": "ms/layer",
               "h2d_bytes_per_step": int(3 * S * H * d * 2 + mh.numel() * world),
               "d2h_bytes_per_step": int(g.padded_tokens * H * d * 2),
               "path": "rp_masked_attention_exact_host (pinned host Q/K/V/mask -> H2D -> "
                       "CSR -> tcgen05 kernel -> D2H), per rank"}

    # ---- dense references on the same GPU (rank 0) ----------------------------
    dense = {}
    if not args.no_dense and rank == 0:
        full_np = np.packbits(np.ones((nb, nb), np.uint8), axis=1, bitorder="little")
        full = torch.from_numpy(full_np).to(dev)
        rpd, cid, ordd = rp.mask_to_csr(g, full, stream=stream)
        with torch.cuda.stream(stream):
            for _ in range(2):
                rp.sparse_attention(g, q, k, v, rpd, cid, ordd, out=out, stream=stream)
            b0, b1 = ev(), ev()
            b0.record(stream)
            for _ in range(3):
                rp.sparse_attention(g, q, k, v, rpd, cid, ordd, out=out, stream=stream)
            b1.record(stream)
        stream.synchronize()
        dense_ours = b0.elapsed_time(b1) / 3 * (H / Hl)
        qs = q.permute(1, 0, 2).unsqueeze(0)
        ks = k.permute(1, 0, 2).unsqueeze(0)
        vs = v.permute(1, 0, 2).unsqueeze(0)
        with torch.cuda.stream(stream):
            for _ in range(2):
                torch.nn.functional.scaled_dot_product_attention(qs, ks, vs)
            b0.record(stream)
            for _ in range(3):
                torch.nn.functional.scaled_dot_product_attention(qs, ks, vs)
            b1.record(stream)
        stream.synchronize()
        sdpa = b0.elapsed_time(b1) / 3 * (H / Hl)
        dense = {"ours_dense_ms": dense_ours, "sdpa_dense_ms": sdpa,
                 "speedup_vs_sdpa_dense": sdpa / ms, "speedup_vs_ours_dense": dense_ours / ms,
                 "note": "full layer (all heads) dense bf16 attention on this GPU; SDPA = "
                         "torch scaled_dot_product_attention (cuDNN/flash backend)"}

    # ---- static mask: warm rebuild (the one-time figure includes first-call
    # module loading and pool growth) ------------------------------------------
    static_warm = None
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
        static_warm = min(ts)

    # ---- a library block-sparse kernel on the same BSR mask ------
    libcmp = None
    if not args.no_lib and rank == 0:
        try:
            import flashinfer
            Sp = g.padded_tokens
            pads = []
            for t in (q, k, v):  # FlashInfer needs N % C == 0: zero rows = the
                x = torch.zeros((Sp, Hl, d), dtype=torch.bfloat16, device=dev)  # reference's
                x[:S] = t                                                        # padding
                pads.append(x)
            indptr, indices = rp.mask_to_bsr(g, mask)
            ws = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
            wr = flashinfer.BlockSparseAttentionWrapper(ws)
            t0 = time.time()
            wr.plan(indptr, indices, Sp, Sp, cfgd["bs"], cfgd["bs"], Hl, Hl, d,
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
            ours_k = float(np.mean(k6_ms)) * (H / Hl)
            with torch.cuda.stream(stream):
                rp.sparse_attention(g, q, k, v, row_ptr, col_idx, order, out=out, stream=stream)
            stream.synchronize()
            a, b = out[:S].float(), fo[:S].float()
            rel = float(((a - b).norm(dim=-1) / b.norm(dim=-1).clamp_min(1e-30)).max())
            libcmp = {"library": f"flashinfer {flashinfer.__version__} BlockSparseAttentionWrapper "
                                 "(BSR, R=C=B) on the same mask and Q/K/V",
                      "library_ms": fi_ms, "ours_stage_d_ms": ours_k,
                      "speedup_vs_library": fi_ms / ours_k, "max_row_rel_diff": rel,
                      "library_first_call_s": first}
            del pads, ws, wr, fo
        except Exception as exc:  # comparator only: never fails the bench
            libcmp = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}

    # ---- the north star's pooled selector on the same Q/K -------
    pooled = None
    if dynamic and rank == 0:
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
        # stage (b) alone (the HBM-bound block-mean pooling of Q and K)
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
        p_nnz = int(np.unpackbits(pm.cpu().numpy()).sum())
        pooled = {"ms": p_ms, "mode": "cumulative softmax mass 0.95 over radial candidates, "
                  "H_f=2 block-mean pooled Q/K (NOT reference semantics, SURVEY 8f1)",
                  "stage_b_pool_ms": pool_ms, "stage_b_bytes": alg,
                  "stage_b_achieved_gbs": alg / (pool_ms * 1e-3) / 1e9,
                  "stage_b_hbm_frac": alg / (pool_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                  "stages_c_ms": p_ms - pool_ms,
                  "block_sparsity": round(1 - p_nnz / float(nb * nb), 4)}

    # ---- CPU baseline (rank 0, N=1) --------------------------------------------
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        threads = os.cpu_count() or 1
        cms, dt, desc, kind = reference_sample(cfgd, threads)
        cpu = {"value": cms, "unit": "ms/layer", "cores": threads, "kind": kind,
               "sample": desc, "sample_wall_s": dt}

    traffic = None
    # stage-(d) kernel: DYNRAD_K6 if set, else the library's auto rule (rp once
    # one head's K + V exceed 64 MiB, see capi.cu launch_attention)
    forced = os.environ.get("DYNRAD_K6")
    rpk = forced == "rp" or (forced is None and 4 * g.padded_tokens * 128 > 64 * 2**20)
    kname = "bsfa_fwd_rp_kernel<128> (row pairs)" if rpk else "bsfa_fwd_db_kernel<128>"
    # DRAM traffic per launch from the one ncu --set full capture of this
    # kernel at this config (null when none was taken)
    prof = {("wan_static", False): "k6db_ncu_summary.json",
            ("hunyuan_dynamic", True): "k6rp_hunyuan_ncu_summary.json"}.get((args.config, rpk))
    if prof and os.path.exists(os.path.join(ROOT, "profiles", prof)):
        with open(os.path.join(ROOT, "profiles", prof)) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    peak = peaks["bf16_tflops"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": ms, "unit": "ms/layer", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic N(0,1) Q/K/V of the whole layer (torch generator, seed 42; each rank takes its head slice)",
            "config": {"workload": cfgd["workload"], "global_heads": H,
                       "seq_len": S, "padded_tokens": g.padded_tokens,
                       "block_size": cfgd["bs"], "mask_active_blocks": nnz,
                       "block_sparsity": round(sparsity, 4),
                       "parallelism": f"head-sharded x{world}" + (
                           " (static mask cached on every rank: no collective)" if not dynamic
                           else " (split scoring: broadcast of the 2 scoring heads + OR "
                                "all-gather of the bitmask)" if world > 1 else ""),
                       "l2": "inputs larger than L2 (Q/K/V 2.3 GB bf16 per layer)"},
            "effective_tflops": tflops_eff,
            "algorithmic_tflops": tflops_alg,
            "mask_build_ms_one_time": mask_build_ms,
            "static_mask_build_ms_warm": static_warm,
            "roofline": {"bound": "tensor", "achieved": kernel_tflops, "peak": peak,
                         "unit": "TFLOP/s", "frac": kernel_tflops / peak,
                         "traffic": traffic,
                         "kernel": kname + " (stage d)",
                         "kernel_ms": float(np.mean(k6_ms)),
                         "per_launch": "4*H*d*B^2*nnz flop on active blocks",
                         "peak_source": f"{peaks_kind} bf16_tflops (burst)"},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "dense": dense or None,
            "library_comparator": libcmp,
            "pooled_selector_f1": pooled,
            "stages_ms": {"attention_stage_d": float(np.mean(k6_ms)),
                          "mask_stages_a_c_plus_csr": float(np.mean(per_step) - np.mean(k6_ms))
                          if dynamic else 0.0,
                          "note": "static: mask cached per (grid, config, seed), built once "
                                  "(mask_build_ms_one_time)" if not dynamic else
                                  "dynamic: mask rebuilt from the layer's Q/K every step"},
            "per_step_ms": {"min": float(min(per_step)), "median": float(np.median(per_step)),
                            "max": float(max(per_step))},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
