"""A/B timing of the stage-(d) kernel at the Wan shape (config-3 mask, seed-42
inputs like bench.py): mean of 20 back-to-back launches after 5 warm-ups.
Run once per configuration (env vars are read once per process)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_20470_b200 import radialplan as rp  # noqa: E402

g = rp.make_grid(21, 3600, 128)
H, d, S = 40, 128, g.total_tokens
gen = torch.Generator(device="cuda").manual_seed(42)
if os.environ.get("DIRECT_BF16"):  # tools/attn_perf.py's inputs
    q, k, v = (torch.randn((S, H, d), device="cuda", dtype=torch.bfloat16) for _ in range(3))
else:
    q, k, v = (torch.randn((S, H, d), device="cuda", generator=gen).to(torch.bfloat16)
               for _ in range(3))
cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
mask = rp.Plan(g, cfg, 7).build_mask_device()
if os.environ.get("DENSE"):  # every block active (per-flop efficiency without sparsity)
    mask.fill_(255)
    nb = g.blocks_per_dim
    if nb % 8:
        mask[:, nb // 8] = (1 << (nb % 8)) - 1
    if mask.shape[1] > (nb + 7) // 8:
        mask[:, (nb + 7) // 8:] = 0
rpt, col, order = rp.mask_to_csr(g, mask)
out = torch.empty((g.padded_tokens, H, d), dtype=torch.bfloat16, device="cuda")
for _ in range(5):
    rp.sparse_attention(g, q, k, v, rpt, col, order, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20):
    rp.sparse_attention(g, q, k, v, rpt, col, order, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
nnz = col.numel()
print(f"{os.environ.get('TAG', '')} {ms:.3f} ms  {4.0 * H * d * 128 * 128 * nnz / ms / 1e9:.0f} TFLOP/s")
