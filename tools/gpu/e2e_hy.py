"""Host-buffer layer (rp_sparse_layer_host) at the Hunyuan dynamic shape vs
the device path (CUDA events, 5 calls each)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2604_20470_b200 import radialplan as rp
g = rp.make_grid(61, 3600, 128)
H, d, S = 24, 128, g.total_tokens
fb = rp.random_batch(S, H, d, 42)
cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45, -1.5, 2.0)
plan = rp.Plan(g, cfg, 7)
qh, kh, vh = (t.cpu().pin_memory() for t in (fb.queries, fb.keys, fb.values))
oh = torch.empty((g.padded_tokens, H, d), dtype=torch.bfloat16).pin_memory()
st = torch.cuda.Stream()
def call():
    rp.sparse_layer_host(plan, qh, kh, vh, 2, out=oh, stream=st)
call()
for rep in range(2):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(st)
    for _ in range(5): call()
    e1.record(st); st.synchronize()
    print(os.environ.get("DYNRAD_LIB", "in-tree"), "layer_host ms", round(e0.elapsed_time(e1) / 5, 2), flush=True)
