"""One static-ratio mask build at the Wan grid (the objective's STATIC config)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2604_20470_b200 import radialplan as rp
g = rp.make_grid(21, 3600, 128)
cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.5, 0.5, 1e-6), 0.6, 0.3, 0.5, 0.3, 1)
st = {}
p = rp.Plan(g, cfg, 5); d = p.build_mask_device(stats=st); torch.cuda.synchronize()
print(st)
