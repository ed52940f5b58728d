import os, sys, torch, time
sys.path.insert(0, os.getcwd())
from paper_2604_20470_b200 import radialplan as rp, _lib
import ctypes as C
g = rp.make_grid(21, 3600, 128)
H, d, S = 40, 128, g.total_tokens
fb = rp.random_batch(S, H, d, 42)
cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
plan = rp.Plan(g, cfg, 7)
mask = plan.build_mask_device()
qh, kh, vh = (t.cpu().pin_memory() for t in (fb.queries, fb.keys, fb.values))
oh = torch.empty((g.padded_tokens, H, d), dtype=torch.bfloat16).pin_memory()
mh = mask.cpu().pin_memory()
st = torch.cuda.Stream()
for name in ("layer", "exact_host"):
    def call():
        if name == "layer":
            rp.sparse_layer_host(plan, qh, kh, vh, 0, out=oh, stream=st)
        else:
            gc = g.c()
            _lib.check(_lib.lib().rp_masked_attention_exact_host(C.byref(gc), C.c_void_p(mh.data_ptr()), C.c_void_p(qh.data_ptr()), C.c_void_p(kh.data_ptr()), C.c_void_p(vh.data_ptr()), 1, S, H, d, C.c_void_p(oh.data_ptr()), C.c_void_p(st.cuda_stream)))
    call()
    ts = []
    for rep in range(4):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(st)
        for _ in range(5): call()
        e1.record(st); st.synchronize()
        ts.append(round(e0.elapsed_time(e1) / 5, 2))
    print(os.environ.get("DYNRAD_E2E_TAPER", ""), name, ts, flush=True)
