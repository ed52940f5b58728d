"""Exact fp64 scoring engine at the Wan grid (f32 features, feature_dim 64,
H_f = 1, Table-3 Mid): the profiler objective's dynamic trial path."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2604_20470_b200 import radialplan as rp
g = rp.make_grid(21, 3600, 128)
cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45, -1.5, 2.0)
gen = torch.Generator(device="cuda").manual_seed(1)
f = (torch.randn(g.total_tokens, 1, 64, device="cuda", generator=gen) * 0.5).contiguous()
plan = rp.Plan(g, cfg, 7)
st = {}
m = plan.build_mask_device(f, f, 1, stats=st)
torch.cuda.synchronize()
for _ in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter(); plan.build_mask_device(f, f, 1, out=m); torch.cuda.synchronize()
    print("exact build ms", round(1e3 * (time.perf_counter() - t0), 1), st, flush=True)
