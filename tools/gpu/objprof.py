import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2604_20470_b200 import radialplan as rp
g = rp.make_grid(21, 3600, 128)
cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.5, 0.5, 1e-6), 0.6, 0.3, 0.5, 0.3, 1)
for it in range(3):
    t0 = time.time()
    m = rp.build_mask(g, cfg, 5)
    t1 = time.time()
    p = rp.Plan(g, cfg, 5); d = p.build_mask_device(); torch.cuda.synchronize()
    t2 = time.time()
    del p
    torch.cuda.synchronize(); t3 = time.time()
    print(f"build_mask one-shot {1e3*(t1-t0):.1f} ms, plan build {1e3*(t2-t1):.1f} ms, destroy {1e3*(t3-t2):.1f} ms, active {m.active_count()}")
rp.profile_stages(True)
p = rp.Plan(g, cfg, 5); d = p.build_mask_device(); torch.cuda.synchronize()
print(rp.profile_read())
# host vs device split of one plan build
t0 = time.perf_counter(); p = rp.Plan(g, cfg, 5); t1 = time.perf_counter()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); d = p.build_mask_device(); e1.record(); t2 = time.perf_counter(); torch.cuda.synchronize(); t3 = time.perf_counter()
print(f"plan create {1e3*(t1-t0):.1f} ms, build call returns after {1e3*(t2-t1):.1f} ms, device {e0.elapsed_time(e1):.1f} ms, total {1e3*(t3-t0):.1f} ms")
