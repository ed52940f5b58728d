"""SURVEY 8f4 measurement: soft-mask attention (masked_attention, every key
with a log(mask + eps) offset) vs the exact block-sparse kernel and torch SDPA
dense, at the Wan2.1 shape (21 x 3600 tokens, 40 heads, d = 128, config-3
static mask).  Soft attention is dense work by definition (the reference's
semantics), so its yardstick is dense attention.  JSON to stdout / argv[1]."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402
from paper_2604_20470_b200 import radialplan as rp  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    nf, nt, H, d = 21, 3600, 40, 128
    g = rp.make_grid(nf, nt, 128)
    cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
    mask = rp.Plan(g, cfg, 7).build_mask_device()
    fb = rp.random_batch(nf * nt, H, d, 42)
    q, k, v = fb.queries, fb.keys, fb.values
    out = torch.empty((g.padded_tokens, H, d), dtype=torch.bfloat16, device="cuda")
    rpt, col, order = rp.mask_to_csr(g, mask)
    with ClockSampler(0) as clk:
        exact = timed(lambda: rp.sparse_attention(g, q, k, v, rpt, col, order, out=out))
        soft = timed(lambda: rp.soft_attention(g, q, k, v, mask, 1e-10, out=out))
        qs, ks, vs = (x.permute(1, 0, 2).unsqueeze(0) for x in (q, k, v))
        sdpa = timed(lambda: torch.nn.functional.scaled_dot_product_attention(qs, ks, vs))
    nb = g.blocks_per_dim
    flop = 4.0 * H * d * 128 * 128 * nb * nb
    rec = {"workload": "Wan2.1 21x3600, 40 heads, d=128, bf16, config-3 static mask",
           "exact_sparse_ms": exact, "soft_mask_ms": soft, "sdpa_dense_ms": sdpa,
           "soft_tflops": flop / (soft * 1e-3) / 1e12,
           "soft_vs_sdpa_dense": sdpa / soft, "clocks": clk.summary(),
           "kernel_soft": "dense row lists + per-block log-eps offset on "
                          + rp.attention_kernel(g, "bf16", d)}
    print(json.dumps(rec))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
