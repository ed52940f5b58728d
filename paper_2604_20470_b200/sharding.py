"""Head sharding of the attention layer across the GPUs of one node.

Stage (d) is independent per head and every head uses the same block mask,
so the layer shards by head with no data-path collective:

* static mode: every rank builds (or loads) the identical cached mask from
  (grid, config, seed) -- no communication at all;
* dynamic mode: the mask is scored from the first H_f heads (the paper's
  fused proxy heads), which live on the rank holding head
  0.  Two exchange schemes:
    - broadcast_mask: that rank builds the mask and broadcasts the
      S_b x ceil(S_b/8) bitmask (Wan 43.7 KB, Hunyuan 369 KB);
    - split scoring: the H_f-head Q/K slices are broadcast
      (broadcast_scoring_features, Hunyuan 225 MB over NVLink), every rank
      scores 1/world of the frame pairs (BuildOptions.shard_index /
      shard_count) and or_allgather_mask ORs the partial bitmasks, so the
      scoring time also divides by the number of GPUs;
* optionally the head-sharded outputs are all-gathered into [S', H, d].

The helpers take a torch.distributed process group, so the same code runs
over NCCL on the GPUs and over gloo in the CPU tests.
"""
from __future__ import annotations

from typing import List, Tuple


def head_shards(heads: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous (first_head, count) per rank; counts differ by at most one.

    Contiguous shards keep each rank's heads adjacent in the [S, H, d]
    layout (one strided view per rank) and keep head pairs together for the
    kernel's two-tile ping-pong."""
    if heads < 1 or world < 1:
        raise ValueError("head_shards: heads and world must be >= 1")
    if world > heads:
        raise ValueError(f"head_shards: {world} ranks for {heads} heads")
    base, extra = divmod(heads, world)
    out, h = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((h, n))
        h += n
    return out


def score_rank(heads: int, world: int, n_score_heads: int) -> int:
    """Rank that owns all of the H_f scoring heads (heads 0 .. H_f-1)."""
    first, n = head_shards(heads, world)[0]
    if n_score_heads > n:
        raise ValueError("score heads must live on one rank (H_f <= heads per rank)")
    return 0


def broadcast_mask(mask, src: int = 0, group=None):
    """Broadcast the bit-packed block mask (uint8 tensor) from `src` in place."""
    import torch.distributed as dist
    dist.broadcast(mask, src=src, group=group)
    return mask


def gather_heads(out_local, heads: int, group=None):
    """All-gather head-sharded outputs [S', H_r, d] into [S', H, d]."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    shards = head_shards(heads, world)
    width = max(n for _, n in shards)
    S, hr, d = out_local.shape
    buf = torch.zeros((S, width, d), dtype=out_local.dtype, device=out_local.device)
    buf[:, :hr] = out_local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf.contiguous(), group=group)
    return torch.cat([p[:, :n] for p, (_, n) in zip(parts, shards)], dim=1)


def broadcast_scoring_features(q, k, n_score_heads: int, src: int = 0, group=None, out=None):
    """Copy of the first `n_score_heads` heads of Q/K on every rank
    ([S, n, d] contiguous each), broadcast from `src` (which holds them)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    if out is None:
        shape = (q.shape[0], n_score_heads, q.shape[2])
        out = (torch.empty(shape, dtype=q.dtype, device=q.device),
               torch.empty(shape, dtype=k.dtype, device=k.device))
    qs, ks = out
    if rank == src:
        qs.copy_(q[:, :n_score_heads])
        ks.copy_(k[:, :n_score_heads])
    dist.broadcast(qs, src=src, group=group)
    dist.broadcast(ks, src=src, group=group)
    return qs, ks


def or_allgather_mask(mask, group=None):
    """Bitwise OR of every rank's bit-packed block mask, in place (all-gather
    of the packed bytes, then a local OR: NCCL has no bitwise reduction)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return mask
    parts = [torch.empty_like(mask) for _ in range(world)]
    dist.all_gather(parts, mask.contiguous(), group=group)
    acc = parts[0].clone()
    for r in range(1, world):
        acc.bitwise_or_(parts[r])
    mask.copy_(acc)
    return mask
