"""SURVEY 8f2 comparator: the same block-sparse attention through FlashInfer's
BSR wrapper (library code, JIT-compiled on first use) next to this repo's
tcgen05 kernel, at the Wan2.1 shape with the config-3 static mask.

Our row lists ARE a BSR matrix (radialplan.mask_to_bsr: indptr / indices,
R = C = B); FlashInfer needs N divisible by C, so Q/K/V are zero-padded to
S' rows -- exactly the reference's padding semantics (attention.cpp:43-48).
Prints one JSON object (and writes it to argv[1] if given)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_20470_b200 import radialplan as rp  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    import flashinfer
    H = int(os.environ.get("HEADS", "40"))
    nf, nt, d = 21, 3600, 128
    g = rp.make_grid(nf, nt, 128)
    cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
    mask = rp.Plan(g, cfg, 7).build_mask_device()
    S, Sp = g.total_tokens, g.padded_tokens
    gen = torch.Generator(device="cuda").manual_seed(42)
    qkv = [torch.zeros(Sp, H, d, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
    for t in qkv:
        t[:S] = torch.randn(S, H, d, device="cuda", generator=gen).to(torch.bfloat16)
    q, k, v = qkv
    indptr, indices = rp.mask_to_bsr(g, mask)
    nnz = int(indices.numel())
    rpt, col, order = rp.mask_to_csr(g, mask)
    ours_out = torch.empty((Sp, H, d), dtype=torch.bfloat16, device="cuda")
    ours = timed(lambda: rp.sparse_attention(g, q[:S], k[:S], v[:S], rpt, col, order,
                                             out=ours_out))
    ws = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    w = flashinfer.BlockSparseAttentionWrapper(ws)
    t0 = time.time()
    w.plan(indptr, indices, Sp, Sp, 128, 128, H, H, d, q_data_type=torch.bfloat16,
           kv_data_type=torch.bfloat16, o_data_type=torch.bfloat16)
    fi_out = w.run(q, k, v)
    torch.cuda.synchronize()
    first_s = time.time() - t0
    fi = timed(lambda: w.run(q, k, v))
    a = ours_out[:S].float()
    b = fi_out[:S].float()
    rel = float(((a - b).norm(dim=-1) / b.norm(dim=-1).clamp_min(1e-30)).max())
    flop = 4.0 * H * d * 128 * 128 * nnz
    rec = {"workload": f"Wan2.1 21x3600, {H} heads, d=128, bf16, config-3 static mask "
                       f"({nnz} active blocks)",
           "ours_ms": ours, "flashinfer_bsr_ms": fi,
           "ours_tflops": flop / ours / 1e9, "flashinfer_tflops": flop / fi / 1e9,
           "speedup_vs_flashinfer": fi / ours, "max_row_rel_diff": rel,
           "flashinfer_version": flashinfer.__version__,
           "flashinfer_first_call_s (JIT + plan)": first_s}
    print(json.dumps(rec))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
