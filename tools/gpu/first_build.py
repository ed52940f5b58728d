"""First static Wan build of a fresh process (one-time cost incl. pool growth)."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2604_20470_b200 import radialplan as rp
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
g = rp.make_grid(21, 3600, 128)
cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
for i in range(3):
    t0 = time.perf_counter()
    p = rp.Plan(g, cfg, 7); m = p.build_mask_device(); torch.cuda.synchronize()
    print(f"build {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del p
