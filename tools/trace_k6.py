"""Debug: per-step event timing of the stage-(d) kernel (variant built with
-DRP_TRACE).  Prints softmax durations and wait gaps in SM clocks."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_20470_b200 import radialplan as rp, _lib
from oracle import pyoracle

g = rp.make_grid(21, 3600, 128)
H, d = 40, 128
q = torch.randn(g.total_tokens, H, d, device="cuda", dtype=torch.bfloat16)
k = torch.randn_like(q); v = torch.randn_like(q)
nb = g.blocks_per_dim
dense = (np.random.default_rng(0).random((nb, nb)) < float(os.environ.get("DENSITY", "0.194"))).astype(np.uint8)
np.fill_diagonal(dense, 1)
rowp, coli, order = rp.mask_to_csr(g, torch.from_numpy(pyoracle.pack_dense(dense)).cuda())
out = torch.empty((g.padded_tokens, H, d), device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    rp.sparse_attention(g, q, k, v, rowp, coli, order, out=out)
torch.cuda.synchronize()
buf = np.zeros((4, 12, 512), np.uint64)
assert _lib.lib().rp_debug_trace(C.c_void_p(buf.ctypes.data)) == 0
for cta in range(2):
    t = buf[cta].astype(np.int64)
    base = t[0, 0]
    for x in range(2):
        w0, rdy, arr = t[3 * x], t[3 * x + 1], t[3 * x + 2]
        n = 400
        soft = (arr[8:n] - rdy[8:n])
        wait = (rdy[9:n] - arr[8:n - 1])
        print(f"cta{cta} tile{x}: softmax ready->arrive median {np.median(soft):.0f} clk "
              f"(p10 {np.percentile(soft,10):.0f} p90 {np.percentile(soft,90):.0f}); "
              f"arrive->next S ready median {np.median(wait):.0f}; period median "
              f"{np.median(np.diff(rdy[8:n])):.0f}")
        pw0, pw1 = t[6 + 2 * x], t[7 + 2 * x]
        print(f"   mma: p_full wait median {np.median(pw1[8:n]-pw0[8:n]):.0f}; "
              f"arrive->mma sees P median {np.median(pw1[8:n]-arr[8:n]):.0f}")
    print("   first events A:", [(int(t[0, i] - base), int(t[1, i] - base), int(t[2, i] - base)) for i in range(8, 12)])
    print("   first events B:", [(int(t[3, i] - base), int(t[4, i] - base), int(t[5, i] - base)) for i in range(8, 12)])
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
ts = []
for _ in range(3):
    e0.record(); rp.sparse_attention(g, q, k, v, rowp, coli, order, out=out); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
nnz = int(dense.sum())
print(f"time best {min(ts):.3f} ms -> {4.0*H*d*128*128*nnz/min(ts)/1e9:.1f} TFLOP/s")
t = buf[0].astype(np.int64)
rdy, ld, ex, arr = t[1, 8:400], t[10, 8:400], t[11, 8:400], t[2, 8:400]
print(f"tile A phases (median clk): ready->ld done {np.median(ld-rdy):.0f}, ld->exps done "
      f"{np.median(ex-ld):.0f}, exps->arrive {np.median(arr-ex):.0f}")
