"""SURVEY 8(f2) comparator: FlashAttention-4 (the CuTe-DSL sm100 kernel
shipped in this image as vllm.vllm_flash_attn.cute, nvidia-cutlass-dsl) with
block sparsity, on the SAME block mask and inputs as our stage-(d) kernel.

FA4's block-sparse layout (block_sparsity.py:17-37): per (batch, head, query
block) a count and a list of KV block indices; "full" blocks need no element
mask, "mask" blocks go through a mask_mod.  Its sm100 kernel processes 256
query rows per CTA (two 128-row tiles sharing the K/V stream) and requires
the sparse query block to be a multiple of 256 (tile_m = 64 does not
compile).  So two runs:

  exact   the config mask itself: per 256-row block (our rows 2p, 2p+1) the
          blocks both rows hold are "full", the blocks only one holds are
          "mask" blocks whose mask_mod reads our 128 x 128 bitmask;
  union   the mask with each row pair's lists unioned (what FA4 expresses
          without a mask_mod): both kernels run that same mask, so outputs
          are identical up to rounding.

The zero-padded rows [S, S') are passed explicitly so the padding-key
semantics (attention.cpp:43-48) are identical.

    python tools/fa4_compare.py [wan|hunyuan]     (prints one JSON line)
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_20470_b200 import radialplan as rp  # noqa: E402


def _lists(row_ptr, col_idx, nb):
    rp_ = row_ptr.cpu().numpy()
    ci = col_idx.cpu().numpy()
    return [set(ci[rp_[r]:rp_[r + 1]].tolist()) for r in range(nb)]


def fa4_tensors(g, rows, exact):
    """BlockSparseTensorsTorch over 256-row query blocks (our row pairs)."""
    import numpy as np
    from vllm.vllm_flash_attn.cute.block_sparsity import BlockSparseTensorsTorch
    nb = g.blocks_per_dim
    nq = (nb + 1) // 2
    full = np.zeros((nq, nb), np.int32)
    part = np.zeros((nq, nb), np.int32)
    fcnt = np.zeros(nq, np.int32)
    pcnt = np.zeros(nq, np.int32)
    for p in range(nq):
        a = rows[2 * p]
        b = rows[2 * p + 1] if 2 * p + 1 < nb else a
        if exact:
            fl, pl = sorted(a & b), sorted(a ^ b)
        else:
            fl, pl = sorted(a | b), []
        fcnt[p], pcnt[p] = len(fl), len(pl)
        full[p, :len(fl)] = fl
        part[p, :len(pl)] = pl
    dev = "cuda"
    t = lambda x: torch.from_numpy(x).to(dev)  # noqa: E731
    return BlockSparseTensorsTorch(mask_block_cnt=t(pcnt).view(1, 1, nq),
                                   mask_block_idx=t(part).view(1, 1, nq, nb),
                                   full_block_cnt=t(fcnt).view(1, 1, nq),
                                   full_block_idx=t(full).view(1, 1, nq, nb),
                                   block_size=(2 * g.block_size, g.block_size))


def bitmask_mod():
    """mask_mod(b, h, q_idx, kv_idx, seqlen_info, aux) = our block bit."""
    import cutlass
    import cutlass.cute as cute
    from vllm.vllm_flash_attn.cute import utils

    @cute.jit
    def mask_mod(b, h, q_idx, kv_idx, seqlen_info, aux_tensors):
        dense = aux_tensors[0]
        qi = utils.ssa_to_scalar(q_idx) // 128
        ki = utils.ssa_to_scalar(kv_idx) // 128
        return utils.scalar_to_ssa(dense[qi, ki] != 0, cutlass.Boolean)
    return mask_mod


def compare(g, q, k, v, row_ptr, col_idx, order, H, Hl, d, reps=3):
    """FA4 vs our stage-(d) kernel on the given device inputs [S, Hl, d] bf16
    and row lists; times are scaled to the full layer (x H / Hl)."""
    import numpy as np
    from vllm.vllm_flash_attn.cute.interface import _flash_attn_fwd
    S, Sp, nb = g.total_tokens, g.padded_tokens, g.blocks_per_dim
    pads = []
    for t in (q, k, v):
        x = torch.zeros((1, Sp, Hl, d), dtype=torch.bfloat16, device=q.device)
        x[0, :S] = t
        pads.append(x)
    nnz = int(row_ptr[-1].item())  # col_idx may be an untrimmed buffer (dynamic layers)
    col_idx = col_idx[:nnz]
    rows = _lists(row_ptr, col_idx, nb)
    flops_of = lambda n: 4.0 * H * d * g.block_size ** 2 * n  # noqa: E731
    scale = H / Hl
    recs = {}
    for kind in ("exact", "union"):
        rec = {"library": "FlashAttention-4 CuTe-DSL sm100 forward (vllm.vllm_flash_attn.cute) "
                          "with block_sparse_tensors, 256-row query blocks",
               "mask": kind}
        try:
            if kind == "union":
                dense = np.zeros((nb, nb), np.uint8)
                for p in range(0, nb, 2):
                    u = rows[p] | (rows[p + 1] if p + 1 < nb else set())
                    for r in (p, p + 1):
                        if r < nb:
                            dense[r, sorted(u)] = 1
                bits = np.packbits(dense, axis=1, bitorder="little")
                m2 = torch.from_numpy(bits).to(q.device)
                rpt2, col2, ord2 = rp.mask_to_csr(g, m2)
                bst = fa4_tensors(g, _lists(rpt2, col2, nb), exact=False)
                kw = {}
                n_act = int(col2.numel())
                rec["note"] = ("each row pair's lists unioned: the mask FA4 expresses without a "
                               "mask_mod; both kernels run it")
            else:
                rpt2, col2, ord2 = row_ptr, col_idx, order
                bst = fa4_tensors(g, rows, exact=True)
                dense_t = torch.zeros((nb, nb), dtype=torch.int32, device=q.device)
                rr = torch.repeat_interleave(torch.arange(nb, device=q.device),
                                             (row_ptr[1:] - row_ptr[:-1]).long())
                dense_t[rr, col_idx.long()] = 1
                kw = {"mask_mod": bitmask_mod(), "aux_tensors": [dense_t]}
                n_act = nnz
                rec["note"] = ("the config's own mask: blocks both rows of a pair hold are full "
                               "blocks, the others go through a mask_mod reading our bitmask")
            t0 = time.time()
            out, _ = _flash_attn_fwd(*pads, softmax_scale=1.0 / d ** 0.5,
                                     block_sparse_tensors=bst, **kw)
            torch.cuda.synchronize()
            first = time.time() - t0
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(reps):
                _flash_attn_fwd(*pads, softmax_scale=1.0 / d ** 0.5, block_sparse_tensors=bst,
                                out=out, **kw)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps * scale
            ours = rp.sparse_attention(g, q, k, v, rpt2, col2, ord2)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                rp.sparse_attention(g, q, k, v, rpt2, col2, ord2, out=ours)
            e1.record()
            torch.cuda.synchronize()
            ours_ms = e0.elapsed_time(e1) / reps * scale
            a, b = ours[:S].float(), out[0, :S].float()
            rel = float(((a - b).norm(dim=-1) / b.norm(dim=-1).clamp_min(1e-30)).max())
            rec.update(active_blocks=n_act, library_ms=ms,
                       library_tflops_on_active=flops_of(n_act) / ms / 1e9,
                       ours_ms=ours_ms, ours_tflops=flops_of(n_act) / ours_ms / 1e9,
                       speedup_vs_library=ms / ours_ms, max_row_rel_diff=rel,
                       library_first_call_s=first)
            del out, ours
        except Exception as exc:  # noqa: BLE001 - comparator only
            rec["unavailable"] = f"{type(exc).__name__}: {exc}"[:400]
        recs[kind] = rec
    del pads
    return recs


def run(config="wan"):
    if config == "wan":
        g = rp.make_grid(21, 3600, 128)
        H, d = 40, 128
        cfg = rp.SparsityConfig(rp.Mode.StaticRatio, rp.RadialParams(1.0, 0.1), 1.0, 0.2, 0.3, 0.3)
    else:
        g = rp.make_grid(61, 3600, 128)
        H, d = 24, 128
        cfg = rp.SparsityConfig(rp.Mode.DynamicThreshold, rp.RadialParams(1.4, 0.7), 0.7, 0.45,
                                -1.5, 2.0)
    fb = rp.random_batch(g.total_tokens, H, d, 42)
    q, k, v = fb.queries, fb.keys, fb.values
    plan = rp.Plan(g, cfg, 7)
    mask = plan.build_mask_device(q, k, 2) if config != "wan" else plan.build_mask_device()
    row_ptr, col_idx, order = rp.mask_to_csr(g, mask)
    res = compare(g, q, k, v, row_ptr, col_idx, order, H, H, d)
    res["config"] = config
    return res


if __name__ == "__main__":
    print(json.dumps(run(sys.argv[1] if len(sys.argv) > 1 else "wan")), flush=True)
