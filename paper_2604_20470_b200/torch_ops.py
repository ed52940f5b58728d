"""PyTorch integration of the B200 path for video-DiT attention layers
(the torch custom-op wrapper).

* ``torch.ops.dynrad.sparse_attention`` -- the stage-(d) kernel as a
  registered custom op (with a fake implementation for shape propagation), on
  bf16 ``[tokens, heads, head_dim]`` CUDA tensors and a block-sparse row list.
* :class:`RadialSparseAttention` -- a drop-in attention core for a
  Wan / HunyuanVideo layer: it owns a mask plan for the layer's latent grid,
  builds (static, cached) or rebuilds (dynamic, from the layer's own Q/K) the
  DynamicRad block mask and runs the sparse attention on the current stream.

Every call goes to libdynrad.so; there is no fallback.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import radialplan as rp


@torch.library.custom_op("dynrad::sparse_attention", mutates_args=())
def sparse_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, row_ptr: torch.Tensor,
                     col_idx: torch.Tensor, row_order: torch.Tensor, n_frames: int,
                     tokens_per_frame: int, block_size: int,
                     softmax_scale: float = 0.0) -> torch.Tensor:
    """O[S', H, d] = block-sparse softmax(Q K^T * scale) V (exact-mask
    semantics of masked_attention_exact, attention.cpp:50-121)."""
    g = rp.make_grid(n_frames, tokens_per_frame, block_size)
    return rp.sparse_attention(g, q, k, v, row_ptr, col_idx, row_order,
                               softmax_scale=softmax_scale)


@sparse_attention.register_fake
def _(q, k, v, row_ptr, col_idx, row_order, n_frames, tokens_per_frame, block_size,
      softmax_scale=0.0):
    padded = (n_frames * tokens_per_frame + block_size - 1) // block_size * block_size
    return q.new_empty((padded, q.shape[1], q.shape[2]))


@torch.library.custom_op("dynrad::soft_attention", mutates_args=())
def soft_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, mask_bits: torch.Tensor,
                   epsilon: float, n_frames: int, tokens_per_frame: int, block_size: int,
                   softmax_scale: float = 0.0) -> torch.Tensor:
    """Soft-mask attention (masked_attention, attention.cpp:59-81): every key,
    logits + log1p(eps) on active blocks and + log(eps) elsewhere."""
    g = rp.make_grid(n_frames, tokens_per_frame, block_size)
    return rp.soft_attention(g, q, k, v, mask_bits, epsilon, softmax_scale=softmax_scale)


@soft_attention.register_fake
def _(q, k, v, mask_bits, epsilon, n_frames, tokens_per_frame, block_size, softmax_scale=0.0):
    padded = (n_frames * tokens_per_frame + block_size - 1) // block_size * block_size
    return q.new_empty((padded, q.shape[1], q.shape[2]))


class RadialSparseAttention(torch.nn.Module):
    """Attention core of one DiT layer over an (N_f, h*w) latent grid.

    forward(q, k, v) with q/k/v bf16 [tokens, heads, head_dim] returns
    [tokens, heads, head_dim] (the padded rows are dropped).  Static mode
    builds the mask once per (grid, config, seed) and reuses it; dynamic mode
    rebuilds it every call from the first ``n_score_heads`` heads.  With
    ``soft_epsilon`` set, the layer runs the reference's default soft-mask
    semantics (masked_attention) instead of the exact block-sparse kernel.
    """

    def __init__(self, n_frames: int, tokens_per_frame: int, config: rp.SparsityConfig,
                 seed: int = 7, block_size: int = 128, n_score_heads: int = 2,
                 softmax_scale: float = 0.0, soft_epsilon: Optional[float] = None):
        super().__init__()
        if soft_epsilon is not None and not soft_epsilon > 0:
            raise rp.InvalidArgument("masked attention: epsilon must be positive")
        self.soft_epsilon = soft_epsilon
        self._mask = None
        self.grid = rp.make_grid(n_frames, tokens_per_frame, block_size)
        self.config = config
        self.plan = rp.Plan(self.grid, config, seed)
        self.n_score_heads = n_score_heads
        self.softmax_scale = softmax_scale
        self._lists: Optional[tuple] = None
        self._bufs: Optional[tuple] = None  # dynamic mode: mask + row-list buffers, per device

    @property
    def dynamic(self) -> bool:
        return self.config.mode == rp.Mode.DynamicThreshold

    def block_lists(self, q: Optional[torch.Tensor] = None, k: Optional[torch.Tensor] = None):
        if self.dynamic:
            # no host sync per layer: module-owned buffers, untrimmed lists
            # (row_ptr delimits them), so the layer can be graph-captured
            g = self.grid
            nb = g.blocks_per_dim
            if self._bufs is None or self._bufs[0].device != q.device:
                self._bufs = (torch.empty((nb, g.row_bytes), dtype=torch.uint8, device=q.device),
                              (torch.empty(nb + 1, dtype=torch.int32, device=q.device),
                               torch.empty(nb * nb, dtype=torch.int32, device=q.device),
                               torch.empty(nb, dtype=torch.int32, device=q.device),
                               torch.zeros(1, dtype=torch.int64, device=q.device)))
            mask = self.plan.build_mask_device(q, k, self.n_score_heads, out=self._bufs[0])
            return rp.mask_to_csr(self.grid, mask, out=self._bufs[1])
        if self._lists is None:
            self._lists = rp.mask_to_csr(self.grid, self.plan.build_mask_device())
        return self._lists

    def mask(self, q: Optional[torch.Tensor] = None, k: Optional[torch.Tensor] = None):
        if self.dynamic:
            return self.plan.build_mask_device(q, k, self.n_score_heads)
        if self._mask is None:
            self._mask = self.plan.build_mask_device()
        return self._mask

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
        g = self.grid
        if self.soft_epsilon is not None:
            out = torch.ops.dynrad.soft_attention(q, k, v, self.mask(q, k), self.soft_epsilon,
                                                  g.n_frames, g.tokens_per_frame, g.block_size,
                                                  self.softmax_scale)
            return out[: g.total_tokens]
        row_ptr, col_idx, order = self.block_lists(q, k)
        out = torch.ops.dynrad.sparse_attention(q, k, v, row_ptr, col_idx, order, g.n_frames,
                                                g.tokens_per_frame, g.block_size,
                                                self.softmax_scale)
        return out[: g.total_tokens]
