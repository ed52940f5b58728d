"""One stage-(d) (and, for hunyuan, one dynamic mask build) at the bench's
config and inputs, for ncu captures:

    ncu --set full -k regex:bsfa -s 1 -c 1 -o prof python tools/prof_layer.py wan|hunyuan
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, FEATURE_SEED, N_SCORE_HEADS  # noqa: E402
from paper_2604_20470_b200 import radialplan as rp  # noqa: E402

name = {"wan": "wan_static", "hunyuan": "hunyuan_dynamic"}[sys.argv[1] if len(sys.argv) > 1 else "wan"]
c = CONFIGS[name]
g = rp.make_grid(c["nf"], c["nt"], c["bs"])
gm, gl, tm, tc, a, b = c["cfg"]
cfg = rp.SparsityConfig(rp.Mode(c["mode"]), rp.RadialParams(gm, gl), tm, tc, a, b)
fb = rp.random_batch(g.total_tokens, c["heads"], c["d"], FEATURE_SEED)
plan = rp.Plan(g, cfg, c["seed"])
for _ in range(2):
    mask = (plan.build_mask_device(fb.queries, fb.keys, N_SCORE_HEADS) if c["mode"]
            else plan.build_mask_device())
    rpt, col, order = rp.mask_to_csr(g, mask)
    out = rp.sparse_attention(g, fb.queries, fb.keys, fb.values, rpt, col, order)
torch.cuda.synchronize()
print(name, int(col.numel()))
