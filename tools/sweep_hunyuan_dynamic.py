"""Dynamic-threshold sweep at the HunyuanVideo shape (61x45x80 = 219,600
tokens, 24 heads, d=128, bf16, B=128, H_f=2 scoring heads): for each
(tau_near, tau_far) point of the reference's z-threshold rule the whole
per-layer path (stages a-c mask build from the layer's own Q/K, row lists,
stage d) and its parts, block sparsity, stage-(d) TFLOP/s on active blocks
and fraction of the measured bf16 peak.  The bench's random_batch inputs;
NVML clocks sampled over the sweep.  Writes one JSON document to stdout."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from bench import ClockSampler, FEATURE_SEED  # noqa: E402
from paper_2604_20470_b200 import radialplan as rp  # noqa: E402

POINTS = [(-3.0, 1.0), (-1.5, 1.0), (-1.5, 2.0), (-1.0, 2.0), (-0.5, 2.5), (0.0, 3.0)]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["bf16_tflops"]
    H, d, HF = 24, 128, 2
    g = rp.make_grid(61, 3600, 128)
    S, nb = g.total_tokens, g.blocks_per_dim
    fb = rp.random_batch(S, H, d, FEATURE_SEED)
    q, k, v = fb.queries, fb.keys, fb.values
    out = torch.empty((g.padded_tokens, H, d), device="cuda", dtype=torch.bfloat16)
    rows = []
    with ClockSampler(0) as clk:
        for tn, tf in POINTS:
            cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7,
                                    0.45, tn, tf)
            plan = rp.Plan(g, cfg, 7)
            mask = plan.build_mask_device(q, k, HF)
            rpt, col, order = rp.mask_to_csr(g, mask)
            nnz = int(col.numel())

            def layer():
                m = plan.build_mask_device(q, k, HF, out=mask)
                r, c, o = rp.mask_to_csr(g, m)
                rp.sparse_attention(g, q, k, v, r, c, o, out=out)

            mask_ms = timed(lambda: plan.build_mask_device(q, k, HF, out=mask))
            attn_ms = timed(lambda: rp.sparse_attention(g, q, k, v, rpt, col, order, out=out))
            layer_ms = timed(layer)
            tflops = 4.0 * H * d * 128 * 128 * nnz / (attn_ms * 1e-3) / 1e12
            rows.append({"tau_near": tn, "tau_far": tf, "block_sparsity": round(1 - nnz / nb**2, 4),
                         "nnz": nnz, "layer_ms": round(layer_ms, 2),
                         "mask_build_ms": round(mask_ms, 2), "attention_ms": round(attn_ms, 2),
                         "kernel": rp.attention_kernel(g, "bf16", d),
                         "tflops_active": round(tflops, 1),
                         "frac_of_peak": round(tflops / peak, 4)})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
            del plan
    print(json.dumps({"workload": "HunyuanVideo 61x45x80, 24 heads, d=128, bf16, B=128, "
                                  "dynamic threshold (gamma 1.4, lambda 0.7, theta_m 0.7, "
                                  "theta_c 0.45), H_f=2, random_batch(S, 24, 128, 42) inputs, "
                                  "1 GPU",
                      "peak_bf16_tflops": peak, "clocks": clk.summary(), "points": rows}))


if __name__ == "__main__":
    main()
