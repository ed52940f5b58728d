"""Debug: per-step timing of the double-buffered K6 (variant built with -DRP_TRACE)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_20470_b200 import radialplan as rp, _lib
from oracle import pyoracle
g = rp.make_grid(21, 3600, 128)
H, d = 40, 128
fb = rp.random_batch(g.total_tokens, H, d, 42)   # the bench's inputs and mask
q, k, v = fb.queries, fb.keys, fb.values
cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
rowp, coli, order = rp.mask_to_csr(g, rp.Plan(g, cfg, 7).build_mask_device())
out = torch.empty((g.padded_tokens, H, d), device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    rp.sparse_attention(g, q, k, v, rowp, coli, order, out=out)
torch.cuda.synchronize()
buf = np.zeros((4, 12, 512), np.uint64)
assert _lib.lib().rp_debug_trace(C.c_void_p(buf.ctypes.data)) == 0
for cta in range(2):
    t = buf[cta].astype(np.int64)
    w0, rdy, ldd, exd, arr = t[0, 8:400], t[1, 8:400], t[10, 8:400], t[11, 8:400], t[2, 8:400]
    print(f"cta{cta}: period {np.median(np.diff(rdy)):.0f} clk; wait S {np.median(rdy - w0):.0f}; "
          f"ld {np.median(ldd - rdy):.0f}; max+exps {np.median(exd - ldd):.0f}; store+arrive "
          f"{np.median(arr - exd):.0f}; mma p-wait {np.median(t[7, 8:400] - t[6, 8:400]):.0f}")
