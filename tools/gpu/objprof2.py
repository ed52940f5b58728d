import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2604_20470_b200 import radialplan as rp
g = rp.make_grid(16, 64, 16)
cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.5, 0.5, 1e-6), 0.6, 0.3, 0.5, 0.3, 1)
torch.cuda.synchronize()
for it in range(5):
    t0 = time.perf_counter()
    p = rp.Plan(g, cfg, 5)
    t1 = time.perf_counter()
    d = p.build_mask_device(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    del p
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} build {1e3*(t2-t1):.2f} destroy {1e3*(t3-t2):.2f} ms")
f = (torch.randn(1024, 64, device="cuda") * 0.5).contiguous()
c = rp.ProxyCache(g, f)
for it in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    c.objective(cfg, 5); torch.cuda.synchronize()
    print(f"objective {1e3*(time.perf_counter()-t0):.2f} ms")
