"""Python mirror of the reference's `radialplan` operator API, on the B200 path.

Names, argument meaning and error behaviour follow the reference headers
(proj/include/radialplan/{grid,radial,selection,mask,attention}.hpp) so that
parity tests read like the reference's own tests.  Every data-path call goes
through the C ABI (include/dynrad.h) into the CUDA kernels of libdynrad.so;
the scalar stage-(a) helpers (window widths, split factors, ...) are O(1)
host formulas evaluated by the same library code that plans the kernels.

Device tensors are torch CUDA tensors laid out [tokens, heads, head_dim].
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L
from ._lib import (CudaError, DomainError, InvalidArgument, OutOfRange,  # noqa: F401
                   RadialplanError, RuntimeFailure)


def _torch():
    import torch
    return torch


# ------------------------------------------------------------------ grid ---
@dataclass(frozen=True)
class GridSpec:
    """grid.hpp:13-21"""

    n_frames: int
    tokens_per_frame: int
    block_size: int
    total_tokens: int
    padded_tokens: int
    blocks_per_dim: int

    @property
    def row_bytes(self):
        return (self.blocks_per_dim + 7) // 8

    def c(self):
        return L.Grid(self.n_frames, self.tokens_per_frame, self.block_size, self.total_tokens,
                      self.padded_tokens, self.blocks_per_dim, self.row_bytes)


def make_grid(n_frames: int, tokens_per_frame: int, block_size: int) -> GridSpec:
    """grid.hpp:23-42"""
    g = L.Grid()
    L.check(L.lib().rp_make_grid(int(n_frames), int(tokens_per_frame), int(block_size),
                                 C.byref(g)))
    return GridSpec(g.n_frames, g.tokens_per_frame, g.block_size, g.total_tokens,
                    g.padded_tokens, g.blocks_per_dim)


def block_of(token: int, g: GridSpec) -> int:
    """grid.hpp:45-49"""
    if token < 0 or token >= g.padded_tokens:
        raise OutOfRange("block_of: token outside padded range")
    return token // g.block_size


def frame_of(token: int, g: GridSpec) -> int:
    """grid.hpp:52-57 (padding tokens belong to the last frame)"""
    if token < 0 or token >= g.padded_tokens:
        raise OutOfRange("frame_of: token outside padded range")
    if token >= g.total_tokens:
        return g.n_frames - 1
    return token // g.tokens_per_frame


# ---------------------------------------------------------------- config ---
class Mode(enum.IntEnum):
    StaticRatio = 0
    DynamicThreshold = 1


@dataclass
class RadialParams:
    """radial.hpp:16-20"""

    decay_factor: float = 1.0
    long_range_factor: float = 1.0
    split_epsilon: float = 1e-6


@dataclass
class SparsityConfig:
    """selection.hpp:19-29"""

    mode: Mode = Mode.StaticRatio
    radial: RadialParams = field(default_factory=RadialParams)
    mask_threshold: float = 0.75
    col_threshold: float = 0.20
    near_param: float = 0.25
    far_param: float = 0.55
    fallback_k: int = 1

    def c(self):
        r = self.radial
        return L.Config(int(self.mode), r.decay_factor, r.long_range_factor, r.split_epsilon,
                        self.mask_threshold, self.col_threshold, self.near_param,
                        self.far_param, int(self.fallback_k))

    def validate(self):
        """SparsityConfig::validate (selection.cpp:11-32)"""
        c = self.c()
        L.check(L.lib().rp_config_validate(C.byref(c)))


# ------------------------------------------------------ stage (a) scalars ---
def group_index(t: int) -> int:
    """radial.cpp:10-13"""
    if t < 1:
        raise InvalidArgument("group_index: t must be >= 1")
    return int(t).bit_length()


def base_span(tokens_per_frame: int) -> int:
    """radial.cpp:15-20"""
    if tokens_per_frame < 1:
        raise InvalidArgument("base_span: tokens_per_frame must be >= 1")
    return 1 << (int(tokens_per_frame) - 1).bit_length()


def decay_length(t: int, factor: float, base: int) -> float:
    """radial.cpp:22-28 (exact octave form)"""
    return factor * float(base) / float(1 << group_index(t))


def _pair(i, j, p: RadialParams, g: GridSpec, cfg: Optional[SparsityConfig] = None):
    c = cfg.c() if cfg is not None else SparsityConfig(radial=p).c()
    gc = g.c()
    out = L.FramePair()
    L.check(L.lib().rp_frame_pair_info(C.byref(gc), C.byref(c), int(i), int(j), C.byref(out)))
    return out


def window_width(frame_i: int, frame_j: int, p: RadialParams, g: GridSpec) -> int:
    """radial.cpp:30-39"""
    return _pair(frame_i, frame_j, p, g).width


def split_factor(t: int, p: RadialParams, g: GridSpec) -> int:
    """radial.cpp:41-49"""
    if t < 1:
        raise InvalidArgument("split_factor: t must be >= 1")
    return _pair(0, t, p, _wide(g, t)).split_factor


def _wide(g: GridSpec, t: int) -> GridSpec:
    # frame_pair_info needs both frames inside the grid; the scalar only
    # depends on (t, tokens_per_frame, block_size).
    if t < g.n_frames:
        return g
    return make_grid(t + 1, g.tokens_per_frame, g.block_size)


def frame_retained(t: int, p: RadialParams, g: GridSpec) -> bool:
    """radial.cpp:51-54"""
    if t <= 1:
        return True
    return t % split_factor(t, p, g) == 0


@dataclass
class CandidateSet:
    """radial.hpp:50-73 — lazy band |u - v| <= width in local indices."""

    frame_i: int = 0
    frame_j: int = 0
    distance: int = 0
    tokens_per_frame: int = 0
    width: int = 0
    retained: bool = False

    def pair_count(self) -> int:
        if not self.retained:
            return 0
        n = self.tokens_per_frame
        if self.width >= n - 1:
            return n * n
        m = n - 1 - self.width
        return n * n - m * (m + 1)

    def v_lo(self, u):
        return max(0, u - self.width)

    def v_hi(self, u):
        return min(self.tokens_per_frame - 1, u + self.width)

    def row_offsets(self):
        off = np.zeros(self.tokens_per_frame + 1, np.int64)
        if not self.retained:
            return off
        u = np.arange(self.tokens_per_frame)
        lens = np.minimum(self.tokens_per_frame - 1, u + self.width) - np.maximum(0, u - self.width) + 1
        off[1:] = np.cumsum(lens)
        return off

    def pair_at(self, index):
        if index < 0 or index >= self.pair_count():
            raise OutOfRange("pair_at: index outside candidate set")
        off = self.row_offsets()
        u = int(np.searchsorted(off, index, side="right") - 1)
        return (u, self.v_lo(u) + index - int(off[u]))

    def contains(self, u, v):
        if not self.retained:
            return False
        if u < 0 or u >= self.tokens_per_frame or v < 0 or v >= self.tokens_per_frame:
            return False
        return abs(u - v) <= self.width

    def visit(self, fn):
        if not self.retained:
            return
        for u in range(self.tokens_per_frame):
            for v in range(self.v_lo(u), self.v_hi(u) + 1):
                fn(u, v)


def candidate_set(frame_i: int, frame_j: int, p: RadialParams, g: GridSpec) -> CandidateSet:
    """radial.cpp:111-121"""
    fp = _pair(frame_i, frame_j, p, g)
    return CandidateSet(frame_i, frame_j, abs(frame_i - frame_j), g.tokens_per_frame, fp.width,
                        bool(fp.retained))


def mean_candidates_per_query(g: GridSpec, p: RadialParams, ignore_split: bool) -> float:
    """radial.cpp:123-139"""
    total = 0
    for t in range(g.n_frames):
        pairs_at_t = g.n_frames if t == 0 else 2 * (g.n_frames - t)
        if not ignore_split and not frame_retained(t, p, g):
            continue
        cs = CandidateSet(0, t, t, g.tokens_per_frame, window_width(0, t, p, g), True)
        total += pairs_at_t * cs.pair_count()
    return total / g.total_tokens


def distance_tier(frame_i: int, frame_j: int, p: RadialParams, g: GridSpec) -> int:
    """selection.cpp:34-41"""
    return _pair(frame_i, frame_j, p, g).tier


def retention_ratio(frame_i, frame_j, c: SparsityConfig, g: GridSpec) -> float:
    """selection.cpp:43-50"""
    tier = distance_tier(frame_i, frame_j, c.radial, g)
    return 1.0 if tier == 0 else (c.near_param if tier == 1 else c.far_param)


def score_threshold(frame_i, frame_j, c: SparsityConfig, g: GridSpec) -> float:
    """selection.cpp:52-59"""
    tier = distance_tier(frame_i, frame_j, c.radial, g)
    return -math.inf if tier == 0 else (c.near_param if tier == 1 else c.far_param)


_M64 = (1 << 64) - 1


def mix64(z: int) -> int:
    """rng.hpp:19-25"""
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def pair_seed(seed: int, frame_i: int, frame_j: int) -> int:
    """selection.hpp:45-48"""
    return mix64(mix64(mix64(seed) ^ frame_i) ^ frame_j)


# ---------------------------------------------------------------- masks ----
class BlockMask:
    """mask.hpp:17-35: S_b x S_b bits, row-major, LSB-first, row_bytes=ceil(S_b/8)."""

    def __init__(self, blocks_per_dim: int = 0, bits: Optional[np.ndarray] = None):
        self.dim = int(blocks_per_dim)
        self.row_bytes = (self.dim + 7) // 8
        if bits is None:
            bits = np.zeros((self.dim, self.row_bytes), np.uint8)
        self.bits = np.ascontiguousarray(bits, np.uint8).reshape(self.dim, self.row_bytes)

    def get(self, row, col):
        return bool((self.bits[row, col // 8] >> (col % 8)) & 1)

    def set(self, row, col):
        self.bits[row, col // 8] |= np.uint8(1 << (col % 8))

    def merge(self, other: "BlockMask"):
        if other.dim != self.dim:
            raise InvalidArgument("merge: mask dimensions differ")
        self.bits |= other.bits

    def active_count(self) -> int:
        return int(np.unpackbits(self.bits).sum())

    def dense(self) -> np.ndarray:
        return np.unpackbits(self.bits, axis=1, bitorder="little")[:, : self.dim]

    def __eq__(self, other):
        return isinstance(other, BlockMask) and self.dim == other.dim and np.array_equal(
            self.bits, other.bits)


def sparsity(mask: BlockMask) -> float:
    """mask.cpp:47-50"""
    return 1.0 - mask.active_count() / float(mask.dim * mask.dim)


# ----------------------------------------------- mask files ---
# The reference's persistent mask artifact (mask.cpp:291-376): "DRBM" binary
# (magic, u16 version 1, u32 S_b, the bit-packed rows), a CSV of active
# (row, col) pairs, or a PGM image (active = 0).  Host-side file I/O, so a
# mask built here can be consumed by the reference CLI and vice versa.
class MaskFormat(enum.IntEnum):
    Binary = 0
    Csv = 1
    Pgm = 2


def mask_format_for_path(path: str) -> MaskFormat:
    ext = path[path.rfind("."):] if "." in path else ""
    fmt = {".bin": MaskFormat.Binary, ".csv": MaskFormat.Csv, ".pgm": MaskFormat.Pgm}.get(ext)
    if fmt is None:
        raise InvalidArgument("mask path needs a .bin/.csv/.pgm extension: " + path)
    return fmt


def write_mask(mask: "BlockMask", fmt: MaskFormat, path: str) -> None:
    try:
        with open(path, "wb") as f:
            if fmt == MaskFormat.Binary:
                f.write(b"DRBM" + (1).to_bytes(2, "little") + int(mask.dim).to_bytes(4, "little"))
                f.write(np.ascontiguousarray(mask.bits, np.uint8).tobytes())
            elif fmt == MaskFormat.Csv:
                r, c = np.nonzero(mask.dense())
                f.write("".join(f"{a},{b}\n" for a, b in zip(r, c)).encode())
            else:
                f.write(f"P5\n{mask.dim} {mask.dim}\n255\n".encode())
                f.write(np.where(mask.dense() != 0, 0, 255).astype(np.uint8).tobytes())
    except OSError as e:
        raise RuntimeFailure("cannot open for writing: " + path) from e


def read_mask(path: str) -> "BlockMask":
    try:
        raw = open(path, "rb").read()
    except OSError as e:
        raise RuntimeFailure("cannot open: " + path) from e
    if len(raw) < 10 or raw[:4] != b"DRBM":
        raise RuntimeFailure("mask file has bad magic: " + path)
    if int.from_bytes(raw[4:6], "little") != 1:
        raise RuntimeFailure("unsupported mask version in " + path)
    dim = int.from_bytes(raw[6:10], "little")
    if dim == 0 or dim > (1 << 26):
        raise RuntimeFailure("mask dimension out of range in " + path)
    rb = (dim + 7) // 8
    if len(raw) - 10 < dim * rb:
        raise RuntimeFailure("mask payload truncated: " + path)
    if len(raw) - 10 > dim * rb:
        raise RuntimeFailure("mask payload has trailing bytes: " + path)
    return BlockMask(dim, np.frombuffer(raw[10:], np.uint8).reshape(dim, rb).copy())


def aggregate_block(kept_in_tile, col_threshold: float, mask_threshold: float,
                    block_size: int) -> bool:
    """mask.cpp:68-85 — the tile activation rule the mask kernels apply."""
    counts = [0] * block_size
    for r, c in kept_in_tile:
        if r < 0 or r >= block_size or c < 0 or c >= block_size:
            raise OutOfRange("aggregate_block: pair outside tile")
        counts[c] += 1
    active = sum(1 for x in counts if x / block_size >= col_threshold)
    return active / block_size >= mask_threshold


# ------------------------------------ per-frame-pair selection operators ---
# selection.hpp:60-82, each on its own CUDA kernel (rp_static_select, ...).
def _band(cands: CandidateSet, tokens_per_frame: Optional[int] = None) -> L.Band:
    return L.Band(int(cands.frame_i), int(cands.frame_j),
                  int(tokens_per_frame or cands.tokens_per_frame), int(cands.width),
                  1 if cands.retained else 0)


def static_select(cands: CandidateSet, ratio: float, seed: int):
    """selection.cpp:61-91 -> list of (u, v) in Fisher-Yates slot order."""
    torch = _torch()
    n = cands.pair_count()
    cap = max(1, n)
    uv = torch.empty((cap, 2), dtype=torch.int64, device="cuda")
    k = C.c_int64(0)
    b = _band(cands)
    L.check(L.lib().rp_static_select(C.byref(b), float(ratio), int(seed) & (2**64 - 1),
                                     C.c_void_p(uv.data_ptr()), cap, C.byref(k), None))
    return [tuple(x) for x in uv[: k.value].cpu().tolist()]


def proxy_scores(features: "FeatureBatch", frame_i: int, frame_j: int, cands: CandidateSet,
                 tokens_per_frame: int):
    """selection.cpp:93-123 on device features [tokens, heads, d] -> float32 scores."""
    torch = _torch()
    q, k = features.queries, features.keys
    n = cands.pair_count()
    out = torch.empty(max(n, 1), dtype=torch.float32, device="cuda")
    tq, tk = _tensor(q), _tensor(k)
    b = _band(cands, tokens_per_frame)
    b.frame_i, b.frame_j = int(frame_i), int(frame_j)
    L.check(L.lib().rp_proxy_scores(C.byref(tq), C.byref(tk), int(q.shape[1]), C.byref(b),
                                    C.c_void_p(out.data_ptr()), None))
    return out[:n]


def normalize_scores(scores, stats: Optional[dict] = None):
    """selection.cpp:125-148: device float32 scores -> float64 z (+ mean/stddev)."""
    torch = _torch()
    n = int(scores.numel())
    z = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    mean, sd = C.c_double(0.0), C.c_double(0.0)
    L.check(L.lib().rp_normalize_scores(C.c_void_p(scores.data_ptr()) if n else None, n,
                                        C.c_void_p(z.data_ptr()), C.byref(mean), C.byref(sd),
                                        None))
    if stats is not None:
        stats["mean"], stats["stddev"] = mean.value, sd.value
    return z[:n]


def dynamic_select(cands: CandidateSet, normalized, threshold: float, fallback_k: int = 1):
    """selection.cpp:150-185: device float64 z -> list of (u, v)."""
    torch = _torch()
    n = int(normalized.numel())
    cap = max(1, n)
    uv = torch.empty((cap, 2), dtype=torch.int64, device="cuda")
    k = C.c_int64(0)
    b = _band(cands)
    L.check(L.lib().rp_dynamic_select(C.byref(b), C.c_void_p(normalized.data_ptr()), n,
                                      float(threshold), int(fallback_k),
                                      C.c_void_p(uv.data_ptr()), cap, C.byref(k), None))
    return [tuple(x) for x in uv[: k.value].cpu().tolist()]


# ------------------------------------------------------------- devices ----
def _tensor(t, dtype_code=None) -> L.Tensor:
    """Describe a torch CUDA tensor [tokens, heads, head_dim] (head_dim contiguous)."""
    torch = _torch()
    if t.dim() != 3:
        raise InvalidArgument("feature tensor must be [tokens, heads, head_dim]")
    if t.stride(2) != 1:
        raise InvalidArgument("feature tensor: head_dim must be contiguous")
    if not t.is_cuda:
        raise InvalidArgument("feature tensor must live on the GPU")
    code = {torch.float32: L.RP_F32, torch.bfloat16: L.RP_BF16}.get(t.dtype)
    if code is None:
        raise InvalidArgument("feature tensor dtype must be float32 or bfloat16")
    return L.Tensor(t.data_ptr(), code, t.shape[0], t.shape[1], t.shape[2], t.stride(0),
                    t.stride(1))


def _stream(stream=None, device=None):
    """The stream a call is enqueued on: `stream`, else the current stream of
    `device` (the inputs' device), else of the current device."""
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return C.c_void_p(s.cuda_stream)


def _on(device):
    """Make `device` current for a library call: the C ABI works on the
    current CUDA device (kernel attributes, SM count, host-copy streams)."""
    torch = _torch()
    return torch.cuda.device(device if device is not None else torch.cuda.current_device())


@dataclass
class BuildOptions:
    """mask.hpp:77-81 plus the device scoring engine choice (dynrad.h)."""

    disable_split: bool = False
    score_engine: int = 0  # 0 auto, 1 tensor-core + fp64 recheck, 2 exact fp64
    recheck_delta: float = 0.0
    shard_index: int = 0   # multi-GPU split of the dynamic scoring (dynrad.h)
    shard_count: int = 1

    def c(self):
        return L.BuildOptions(int(self.disable_split), int(self.score_engine),
                              float(self.recheck_delta), int(self.shard_index),
                              int(self.shard_count))


class Plan:
    """Device mask builder for one (grid, config, seed): rp_plan_*."""

    def __init__(self, g: GridSpec, c: SparsityConfig, seed: int,
                 options: Optional[BuildOptions] = None):
        self.grid, self.config, self.seed = g, c, seed
        self.options = options or BuildOptions()
        h = C.c_void_p()
        gc, cc, oc = g.c(), c.c(), self.options.c()
        L.check(L.lib().rp_plan_create(C.byref(gc), C.byref(cc), C.c_uint64(seed & _M64),
                                       C.byref(oc), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.lib().rp_plan_destroy(h)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self._h = None

    def build_mask_device(self, q=None, k=None, n_score_heads: int = 0, out=None,
                          stats: Optional[dict] = None, stream=None):
        """Returns the bit-packed mask as a uint8 CUDA tensor [S_b, row_bytes]."""
        torch = _torch()
        g = self.grid
        dev = q.device if q is not None else (out.device if out is not None else None)
        if out is None:
            out = torch.empty((g.blocks_per_dim, g.row_bytes), dtype=torch.uint8,
                              device=dev if dev is not None else "cuda")
        dev = out.device
        tq = C.byref(_tensor(q)) if q is not None else None
        tk = C.byref(_tensor(k)) if k is not None else None
        if q is not None and n_score_heads <= 0:
            n_score_heads = q.shape[1]
        st = L.BuildStats()
        with _on(dev):
            L.check(L.lib().rp_plan_build_mask(self._h, tq, tk, int(n_score_heads),
                                               C.c_void_p(out.data_ptr()),
                                               C.byref(st) if stats is not None else None,
                                               _stream(stream, dev)))
        if stats is not None:
            for name, _ in L.BuildStats._fields_:
                stats[name] = getattr(st, name)
        return out


@dataclass
class FeatureBatch:
    """attention.hpp:18-27, as device tensors [tokens, heads, head_dim]."""

    queries: object
    keys: object
    values: object = None

    @property
    def tokens(self):
        return self.queries.shape[0]

    @property
    def heads(self):
        return self.queries.shape[1]

    @property
    def head_dim(self):
        return self.queries.shape[2]


def random_batch(tokens: int, heads: int, head_dim: int, seed: int, with_values: bool = True,
                 dtype="bf16", first_head: int = 0, device=None, stream=None) -> FeatureBatch:
    """attention.hpp:62-63 random_batch, generated on the GPU: heads
    [first_head, first_head + heads) of the reference's counter-based batch as
    [tokens, heads, head_dim] tensors (bf16 = round-to-nearest-even of the
    reference's float values, or float32)."""
    torch = _torch()
    tdt = torch.bfloat16 if dtype in ("bf16", torch.bfloat16) else torch.float32
    dev = torch.device(device) if device is not None else torch.device("cuda",
                                                                       torch.cuda.current_device())
    ts = [torch.empty((tokens, heads, head_dim), dtype=tdt, device=dev)
          for _ in range(3 if with_values else 2)]
    descs = [_tensor(t) for t in ts]
    with _on(dev):
        L.check(L.lib().rp_random_batch(int(tokens), int(heads), int(head_dim),
                                        C.c_uint64(seed & _M64), int(first_head),
                                        C.byref(descs[0]), C.byref(descs[1]),
                                        C.byref(descs[2]) if with_values else None,
                                        _stream(stream, dev)))
    return FeatureBatch(ts[0], ts[1], ts[2] if with_values else None)


def build_mask(g: GridSpec, c: SparsityConfig, seed: int,
               options: Optional[BuildOptions] = None,
               features: Optional[FeatureBatch] = None,
               stats: Optional[dict] = None) -> BlockMask:
    """mask.hpp:88-89 — Algorithm 1 on the GPU, returned as a host BlockMask."""
    plan = Plan(g, c, seed, options)
    q = features.queries if features is not None else None
    k = features.keys if features is not None else None
    dev = plan.build_mask_device(q, k, q.shape[1] if q is not None else 0, stats=stats)
    return BlockMask(g.blocks_per_dim, dev.cpu().numpy())


def mask_to_csr(g: GridSpec, mask_dev, stream=None, out=None, trim: bool = True):
    """Bit-packed device mask -> (row_ptr[S_b+1], col_idx, row_order[S_b]) int32.

    With trim=False (or preallocated `out` buffers) nothing synchronizes:
    col_idx keeps its S_b^2 capacity and only row_ptr delimits the lists,
    which is what the per-layer dynamic path uses."""
    torch = _torch()
    nb = g.blocks_per_dim
    cap = nb * nb
    dev = mask_dev.device
    if out is None:
        row_ptr = torch.empty(nb + 1, dtype=torch.int32, device=dev)
        col_idx = torch.empty(cap, dtype=torch.int32, device=dev)
        order = torch.empty(nb, dtype=torch.int32, device=dev)
        nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    else:
        row_ptr, col_idx, order, nnz = out
        cap = col_idx.numel()
    gc = g.c()
    with _on(dev):
        L.check(L.lib().rp_mask_to_csr(C.byref(gc), C.c_void_p(mask_dev.data_ptr()),
                                       C.c_void_p(row_ptr.data_ptr()),
                                       C.c_void_p(col_idx.data_ptr()), cap,
                                       C.c_void_p(order.data_ptr()), C.c_void_p(nnz.data_ptr()),
                                       _stream(stream, dev)))
    if not trim or out is not None:
        return row_ptr, col_idx, order
    n = int(nnz.item())
    return row_ptr, col_idx[:n], order


def mask_to_bsr(g: GridSpec, mask_dev, stream=None):
    """SURVEY 8f2 export: the block mask as a BSR matrix (indptr[S_b+1],
    indices[nnz] int32, ascending per row, block R = C = g.block_size) -- the
    layout FlashInfer's BlockSparseAttentionWrapper.plan and scipy.sparse.bsr
    take (tools/flashinfer_compare.py runs FlashInfer on it)."""
    row_ptr, col_idx, _ = mask_to_csr(g, mask_dev, stream=stream)
    return row_ptr, col_idx


def sparse_attention(g: GridSpec, q, k, v, row_ptr, col_idx, row_order=None, out=None,
                     softmax_scale: float = 0.0, stream=None, check_empty: bool = False):
    """Block-sparse attention forward on device tensors; out [S', heads, d].

    A row without any active block is the reference's domain_error
    (attention.cpp:85-86).  The device kernel zero-fills such rows; with
    check_empty=True the kernel also raises a device flag, which this call
    reads (synchronizing the stream) and turns into DomainError."""
    torch = _torch()
    dev = q.device
    if out is None:
        out = torch.empty((g.padded_tokens, q.shape[1], q.shape[2]), dtype=q.dtype, device=dev)
    gc = g.c()
    tq, tk, tv, to = _tensor(q), _tensor(k), _tensor(v), _tensor(out)
    flag = torch.zeros(1, dtype=torch.int32, device=dev) if check_empty else None
    with _on(dev):
        L.check(L.lib().rp_sparse_attention_fwd_checked(
            C.byref(gc), C.byref(tq), C.byref(tk), C.byref(tv), C.byref(to),
            C.c_void_p(row_ptr.data_ptr()), C.c_void_p(col_idx.data_ptr()),
            C.c_void_p(row_order.data_ptr()) if row_order is not None else None,
            C.c_float(softmax_scale), C.c_void_p(flag.data_ptr()) if flag is not None else None,
            _stream(stream, dev)))
    if flag is not None and int(flag.item()):
        raise DomainError("masked attention: row has no active key")
    return out


def sparse_layer_host(plan: "Plan", q, k, v, n_score_heads: int = 0, out=None, mask_out=None,
                      stream=None):
    """One attention layer (stages a-d) from host buffers through
    rp_sparse_layer_host: q/k/v torch CPU tensors [tokens, heads, d]
    (bf16 or float32; pin them for full PCIe speed).  Returns out
    [S', heads, d] (host); mask_out (uint8 [S_b, row_bytes] host tensor)
    receives the block mask when given."""
    torch = _torch()
    g = plan.grid
    for t in (q, k, v):
        if t.is_cuda or not t.is_contiguous() or t.shape != q.shape or t.dtype != q.dtype:
            raise InvalidArgument("sparse layer: q/k/v must be contiguous host tensors of one shape")
    code = {torch.float32: L.RP_F32, torch.bfloat16: L.RP_BF16}.get(q.dtype)
    if code is None:
        raise InvalidArgument("feature tensor dtype must be float32 or bfloat16")
    tok, h, d = q.shape
    if out is None:
        out = torch.empty((g.padded_tokens, h, d), dtype=q.dtype, pin_memory=True)
    gc = g.c()
    L.check(L.lib().rp_sparse_layer_host(
        plan._h, C.byref(gc), C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
        C.c_void_p(v.data_ptr()), code, tok, h, d, int(n_score_heads), C.c_void_p(out.data_ptr()),
        C.c_void_p(mask_out.data_ptr()) if mask_out is not None else None,
        _stream(stream)))
    return out


STAGES = ("mask_prep", "score_stats", "job_stats", "score_select", "recheck", "apply", "csr",
          "attention", "exact_score", "static_build")


def profile_stages(enable: bool) -> None:
    """Start (clearing earlier records) or stop per-stage CUDA-event timing
    inside the library (rp_profile_stages)."""
    L.lib().rp_profile_stages(int(bool(enable)))


def profile_read() -> dict:
    """{stage: (total_ms, count)} of the events recorded since profile_stages(True)."""
    n = len(STAGES)
    tot = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    L.check(L.lib().rp_profile_read(tot, cnt, n))
    return {name: (tot[i], int(cnt[i])) for i, name in enumerate(STAGES) if cnt[i]}


def attention_kernel(g: GridSpec, dtype="bf16", head_dim: int = 128) -> str:
    """Name of the stage-(d) kernel the library launches for this grid, dtype
    and head_dim (bf16: db, or rp once one head's K + V exceed 64 MiB;
    DYNRAD_K6 forces one)."""
    code = L.RP_BF16 if dtype in ("bf16", L.RP_BF16) else L.RP_F32
    gc = g.c()
    return L.lib().rp_attention_kernel(C.byref(gc), code, int(head_dim)).decode()


def expand_mask(mask_dev, g: GridSpec, stream=None):
    """mask.cpp:52-66 on device: token-level bits [S', ceil(S'/8)] uint8."""
    torch = _torch()
    trb = (g.padded_tokens + 7) // 8
    dev = mask_dev.device
    out = torch.empty((g.padded_tokens, trb), dtype=torch.uint8, device=dev)
    gc = g.c()
    with _on(dev):
        L.check(L.lib().rp_expand_mask(C.byref(gc), C.c_void_p(mask_dev.data_ptr()),
                                       C.c_void_p(out.data_ptr()), _stream(stream, dev)))
    return out


def soft_attention(g: GridSpec, q, k, v, mask_dev, epsilon: float, out=None,
                   softmax_scale: float = 0.0, stream=None):
    """Soft-mask attention (masked_attention, attention.cpp:59-81) on device
    tensors: every key attended, logits + log1p(eps) on active blocks and
    + log(eps) elsewhere.  mask_dev: the bit-packed block mask on the GPU."""
    torch = _torch()
    if out is None:
        out = torch.empty((g.padded_tokens, q.shape[1], q.shape[2]), dtype=q.dtype,
                          device=q.device)
    gc = g.c()
    tq, tk, tv, to = _tensor(q), _tensor(k), _tensor(v), _tensor(out)
    with _on(q.device):
        L.check(L.lib().rp_soft_attention_fwd(
            C.byref(gc), C.byref(tq), C.byref(tk), C.byref(tv), C.byref(to),
            C.c_void_p(mask_dev.data_ptr()), C.c_double(epsilon), C.c_float(softmax_scale),
            _stream(stream, q.device)))
    return out


def _host_attention(fn, g: GridSpec, mask: BlockMask, q, k, v, *extra):
    q = np.ascontiguousarray(q)
    k = np.ascontiguousarray(k)
    v = np.ascontiguousarray(v)
    if q.dtype == np.float32:
        code, odt = L.RP_F32, np.float32
    elif q.dtype == np.uint16:
        code, odt = L.RP_BF16, np.uint16
    else:
        raise InvalidArgument("masked attention: float32 or bf16 (uint16) inputs")
    tok, h, d = q.shape
    out = np.empty((g.padded_tokens, h, d), odt)
    bits = np.ascontiguousarray(mask.bits, np.uint8)
    gc = g.c()
    L.check(fn(C.byref(gc), bits.ctypes.data_as(C.c_void_p), q.ctypes.data_as(C.c_void_p),
               k.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p), code, tok, h, d,
               *extra, out.ctypes.data_as(C.c_void_p), None))
    return out


def masked_attention_exact(g: GridSpec, mask: BlockMask, q: np.ndarray, k: np.ndarray,
                           v: np.ndarray) -> np.ndarray:
    """masked_attention_exact (attention.hpp:43-44) with host buffers.

    q/k/v: host float32 (or bf16 as uint16) arrays [tokens, heads, d];
    returns host [S', heads, d].  Raises DomainError on an empty row.
    """
    return _host_attention(L.lib().rp_masked_attention_exact_host, g, mask, q, k, v)


def masked_attention(g: GridSpec, mask: BlockMask, q: np.ndarray, k: np.ndarray,
                     v: np.ndarray, epsilon: float = 1e-10) -> np.ndarray:
    """masked_attention (attention.hpp:37-39, soft mask log(mask + eps)) with
    host buffers; raises InvalidArgument unless epsilon > 0."""
    return _host_attention(L.lib().rp_masked_attention_host, g, mask, q, k, v,
                           C.c_double(epsilon))


# ------------------------------------------- profiler objective --
class ProxyCache:
    """build_proxy_cache (profiler.cpp:49-78) on the GPU, device-resident.

    features: the ProxyBatch features, float32 [total_tokens, feature_dim]
    CUDA tensor.  Keeps per-(row, column block) statistics of the dense proxy
    attention instead of the S x S matrix (rp_proxy_cache_create)."""

    def __init__(self, g: GridSpec, features=None, *, _handle=None, stream=None):
        self.grid = g
        self._h = _handle
        if self._h is None:
            torch = _torch()
            f = features.contiguous()
            if f.dtype != torch.float32 or not f.is_cuda or f.dim() != 2:
                raise InvalidArgument("proxy cache: features must be a float32 [S, dim] CUDA tensor")
            h = C.c_void_p()
            gc = g.c()
            L.check(L.lib().rp_proxy_cache_create(C.byref(gc), C.c_void_p(f.data_ptr()),
                                                  f.shape[1], C.byref(h), _stream(stream)))
            self._h = h

    @classmethod
    def from_weights(cls, g: GridSpec, weights, row_sums, reference_sq_norm: float, stream=None):
        """From a reference-layout cache: weights [S, S] float32 and row_sums
        [S] float64 CUDA tensors (rp_proxy_cache_from_weights)."""
        h = C.c_void_p()
        gc = g.c()
        w, rs = weights.contiguous(), row_sums.contiguous()
        L.check(L.lib().rp_proxy_cache_from_weights(C.byref(gc), C.c_void_p(w.data_ptr()),
                                                    C.c_void_p(rs.data_ptr()),
                                                    float(reference_sq_norm), C.byref(h),
                                                    _stream(stream)))
        return cls(g, _handle=h)

    def stats(self):
        """(row_sums [S] float64, reference_sq_norm)."""
        rs = np.zeros(self.grid.total_tokens, np.float64)
        sq = C.c_double()
        L.check(L.lib().rp_proxy_cache_stats(self._h, rs.ctypes.data_as(C.c_void_p),
                                             C.byref(sq), None))
        return rs, sq.value

    def objective(self, c: SparsityConfig, batch_seed: int, features=None,
                  penalty_weight: float = 10.0, sparsity_target: float = 0.80, mask_out=None,
                  stream=None):
        """objective (profiler.cpp:80-148): (loss, mse, achieved_sparsity).
        Dynamic configs need the batch features (scored as one fused head)."""
        t = L.Trial()
        cc = c.c()
        fp, dim = None, 0
        if features is not None:
            fp, dim = C.c_void_p(features.data_ptr()), features.shape[1]
        L.check(L.lib().rp_objective(self._h, C.byref(cc), batch_seed, fp, dim,
                                     penalty_weight, sparsity_target, C.byref(t),
                                     C.c_void_p(mask_out.data_ptr()) if mask_out is not None
                                     else None, _stream(stream)))
        return t.loss, t.mse, t.achieved_sparsity

    def close(self):
        if self._h:
            L.lib().rp_proxy_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def block_mean_pool(g: GridSpec, x, n_heads: int, out=None, stream=None):
    """Stage (b) of the pooled selector alone: block means of the first
    n_heads heads of bf16 x [tokens, heads, d] -> float32 [S_b, n_heads * d]."""
    torch = _torch()
    if out is None:
        out = torch.empty((g.blocks_per_dim, n_heads * x.shape[2]), dtype=torch.float32,
                          device=x.device)
    gc = g.c()
    t = _tensor(x)
    L.check(L.lib().rp_block_mean_pool(C.byref(gc), C.byref(t), n_heads,
                                       C.c_void_p(out.data_ptr()), _stream(stream)))
    return out


class PooledMode(enum.IntEnum):
    TopK = 0   # static ratio: keep max(1, floor(ratio * n)) best candidates per block row
    Mass = 1   # dynamic: smallest best-first prefix reaching a softmax mass


def pooled_select(g: GridSpec, c: SparsityConfig, q, k, n_score_heads: int, mode: PooledMode,
                  param: float, out=None, stream=None):
    """SURVEY 8(f1), the north star's pooled selector (rp_pooled_select): NOT
    the reference's token-pair semantics.  q/k bf16 [tokens, heads, d] on the
    GPU; returns the bit-packed block mask [S_b, row_bytes] uint8."""
    torch = _torch()
    if out is None:
        out = torch.empty((g.blocks_per_dim, g.row_bytes), dtype=torch.uint8, device="cuda")
    gc, cc = g.c(), c.c()
    tq, tk = _tensor(q), _tensor(k)
    L.check(L.lib().rp_pooled_select(C.byref(gc), C.byref(cc), C.byref(tq), C.byref(tk),
                                     int(n_score_heads), int(mode), float(param),
                                     C.c_void_p(out.data_ptr()), _stream(stream)))
    return out


def kernel_launch_count() -> int:
    return int(L.lib().rp_kernel_launch_count())
