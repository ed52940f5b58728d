"""Dynamic-mode mask build at the Hunyuan / Wan shapes: stats + timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_20470_b200 import radialplan as rp

for name, nf, H in [("hunyuan", 61, 24), ("wan", 21, 40)]:
    g = rp.make_grid(nf, 3600, 128)
    cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45, -1.5, 2.0)
    gen = torch.Generator(device="cuda").manual_seed(42)
    q = torch.randn((g.total_tokens, H, 128), device="cuda", generator=gen).to(torch.bfloat16)
    k = torch.randn((g.total_tokens, H, 128), device="cuda", generator=gen).to(torch.bfloat16)
    plan = rp.Plan(g, cfg, 7)
    st = {}
    m = plan.build_mask_device(q, k, 2, stats=st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); plan.build_mask_device(q, k, 2, out=m); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(name, "stats", st, "build ms", [round(t, 2) for t in ts])
