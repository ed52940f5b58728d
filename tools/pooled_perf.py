"""SURVEY 8f1 timing: the pooled selector's kernels at the Hunyuan / Wan
shapes (CUDA events around the whole call; run under ncu for the split)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20470_b200 import radialplan as rp  # noqa: E402

for name, nf, H in [("hunyuan", 61, 24), ("wan", 21, 40)]:
    g = rp.make_grid(nf, 3600, 128)
    cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45, -1.5, 2.0)
    gen = torch.Generator(device="cuda").manual_seed(42)
    q = torch.randn((g.total_tokens, H, 128), device="cuda", generator=gen).to(torch.bfloat16)
    k = torch.randn((g.total_tokens, H, 128), device="cuda", generator=gen).to(torch.bfloat16)
    out = torch.empty((g.blocks_per_dim, g.row_bytes), dtype=torch.uint8, device="cuda")
    for mode, param in [(rp.PooledMode.Mass, 0.95), (rp.PooledMode.TopK, 0.2)]:
        for _ in range(3):
            rp.pooled_select(g, cfg, q, k, 2, mode, param, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            rp.pooled_select(g, cfg, q, k, 2, mode, param, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        alg = 2 * g.total_tokens * 2 * 128 * 2
        print(f"{name} {mode.name}: {ms * 1e3:.1f} us/call, pooled-read {alg / ms / 1e6:.0f} GB/s")
