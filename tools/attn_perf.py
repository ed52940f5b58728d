"""Quick stage-(d) timing at the Wan2.1 shape (scratch; bench.py is the contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_20470_b200 import radialplan as rp
from oracle import pyoracle

def run(nf=21, nt=3600, H=40, d=128, density=0.194, iters=10):
    g = rp.make_grid(nf, nt, 128)
    S = g.total_tokens
    q = torch.randn(S, H, d, device="cuda", dtype=torch.bfloat16)
    k = torch.randn_like(q); v = torch.randn_like(q)
    rng = np.random.default_rng(0)
    nb = g.blocks_per_dim
    if density < 1.0 and os.environ.get("MASK", "radial") == "radial" and nf == 21:
        # the bench's mask: Wan config 3 (static radial, 0.8061 block sparsity)
        cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
        mdev = rp.Plan(g, cfg, 7).build_mask_device()
        dense = np.unpackbits(mdev.cpu().numpy(), axis=1, bitorder="little")[:, :nb]
    else:
        dense = (rng.random((nb, nb)) < density).astype(np.uint8); np.fill_diagonal(dense, 1)
        mdev = torch.from_numpy(pyoracle.pack_dense(dense)).cuda()
    rowp, coli, order = rp.mask_to_csr(g, mdev)
    if os.environ.get('NO_ORDER'): order = None
    nnz = int(dense.sum())
    out = torch.empty((g.padded_tokens, H, d), device="cuda", dtype=torch.bfloat16)
    for _ in range(3): rp.sparse_attention(g, q, k, v, rowp, coli, order, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(iters):
        e0.record(); rp.sparse_attention(g, q, k, v, rowp, coli, order, out=out); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    t = min(ts)
    flops = 4.0 * H * d * 128 * 128 * nnz
    print(f"nf={nf} nt={nt} H={H} d={d} nnz={nnz} density={nnz/nb/nb:.4f} best {t:.3f} ms "
          f"med {np.median(ts):.3f} -> {flops/t/1e9:.1f} TFLOP/s ({flops/t/1e9/1631.4*100:.1f}% of 1631)")
    return t

if __name__ == "__main__":
    if os.environ.get("QUICK"):
        run(density=0.194, iters=1)
        sys.exit(0)
    run(density=0.194)
    run(density=1.0, iters=3)
    # SDPA dense reference
    S = 75600; H = 40; d = 128
    q = torch.randn(1, H, S, d, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    for _ in range(2): torch.nn.functional.scaled_dot_product_attention(q, k, v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); torch.nn.functional.scaled_dot_product_attention(q, k, v); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1); print(f"SDPA dense {t:.2f} ms {4*H*d*S*S/t/1e9:.1f} TFLOP/s")
