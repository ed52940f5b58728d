"""Per-step clock64 trace of the pp stage-(d) kernel (build with
tools/build_variant.sh trace "-DRP_TRACE", run with DYNRAD_LIB=variants/trace.so).
Wan config-3 mask, 40 heads; prints the median phase durations (cycles) of
tile 0 / tile 1 of CTA 0 and the MMA warp's waits."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20470_b200 import _lib  # noqa: E402
from paper_2604_20470_b200 import radialplan as rp  # noqa: E402

g = rp.make_grid(21, 3600, 128)
H, d, S = 40, 128, g.total_tokens
gen = torch.Generator(device="cuda").manual_seed(42)
q, k, v = (torch.randn((S, H, d), device="cuda", generator=gen).to(torch.bfloat16)
           for _ in range(3))
cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
mask = rp.Plan(g, cfg, 7).build_mask_device()
rpt, col, order = rp.mask_to_csr(g, mask)
out = torch.empty((g.padded_tokens, H, d), dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    rp.sparse_attention(g, q, k, v, rpt, col, order, out=out)
torch.cuda.synchronize()
buf = np.zeros((4, 16, 512), np.uint64)
L = _lib.lib()
L.rp_debug_trace_pp.argtypes = [C.c_void_p]
assert L.rp_debug_trace_pp(buf.ctypes.data) == 0
for cta in range(2):
    tr = buf[cta].astype(np.int64)
    n = 300
    print(f"CTA {cta}")
    for t in range(2):
        e = tr[5 * t:5 * t + 5, 20:n]
        wait = e[1] - e[0]
        ldmax = e[2] - e[1]
        exps = e[3] - e[2]
        tail = e[4] - e[3]
        period = np.diff(tr[5 * t + 1, 20:n])
        print(f"  tile {t}: s_wait {np.median(wait):.0f}  ld+max {np.median(ldmax):.0f}  "
              f"exps {np.median(exps):.0f}  tail {np.median(tail):.0f}  period {np.median(period):.0f}")
    for t in range(2):
        pw = tr[10 + t, 20:n]
        print(f"  mma tile {t}: P ready (MMA view) - softmax S ready: "
              f"{np.median(pw - tr[5 * t + 1, 20:n]):.0f}")
    print("  tile1 S ready - tile0 S ready:", np.median(tr[6, 20:n] - tr[1, 20:n]))
    for t in range(2):
        p_ok = tr[10 + t, 20:n]
        v_ok = tr[12 + t, 20:n]
        s_iss = tr[14 + t, 20:n]
        s_ready_next = tr[5 * t + 1, 21:n + 1]
        print(f"  mma tile {t}: P->V ready {np.median(v_ok - p_ok):.0f}  V ready->S issued "
              f"{np.median(s_iss - v_ok):.0f}  S issued->softmax sees S {np.median(s_ready_next - s_iss):.0f}")
