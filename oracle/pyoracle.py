"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

* ``ref``  : oracle/_ref/libradialplan_ref.so, the reference's own
             radialplan sources compiled in place (oracle/Makefile).
* ``port`` : oracle/liboracle.so, our plain-C restatement
             (oracle/radialplan_oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  The product path (paper_2604_20470_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libradialplan_ref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class _Cfg(C.Structure):
    _fields_ = [
        ("mode", C.c_int),
        ("decay_factor", C.c_double),
        ("long_range_factor", C.c_double),
        ("split_epsilon", C.c_double),
        ("mask_threshold", C.c_double),
        ("col_threshold", C.c_double),
        ("near_param", C.c_double),
        ("far_param", C.c_double),
        ("fallback_k", C.c_int),
    ]


class _Grid(C.Structure):
    _fields_ = [
        ("n_frames", C.c_int),
        ("tokens_per_frame", C.c_int),
        ("block_size", C.c_int),
        ("total_tokens", C.c_int64),
        ("padded_tokens", C.c_int64),
        ("blocks_per_dim", C.c_int64),
        ("row_bytes", C.c_int64),
    ]


@dataclass
class Cfg:
    """Mirror of radialplan::SparsityConfig (selection.hpp:19-29)."""

    mode: int = 0  # 0 static ratio, 1 dynamic threshold
    decay_factor: float = 1.0
    long_range_factor: float = 1.0
    split_epsilon: float = 1e-6
    mask_threshold: float = 0.75
    col_threshold: float = 0.20
    near_param: float = 0.25
    far_param: float = 0.55
    fallback_k: int = 1

    def c(self):
        return _Cfg(self.mode, self.decay_factor, self.long_range_factor,
                    self.split_epsilon, self.mask_threshold, self.col_threshold,
                    self.near_param, self.far_param, self.fallback_k)


def grid_dims(nf, nt, bs):
    total = nf * nt
    padded = (total + bs - 1) // bs * bs
    blocks = padded // bs
    return total, padded, blocks, (blocks + 7) // 8


_P = C.POINTER
_f32p = _P(C.c_float)
_u8p = _P(C.c_uint8)


def _fp(a):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_f32p)


class _Lib:
    def __init__(self, path, kind):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.kind = kind
        self.lib = C.CDLL(path)


_ref = None
_port = None


def have_ref():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        _ref = _RefLib(REF_SO, "reference")
    return _ref


def port():
    global _port
    if _port is None:
        _port = _PortLib(PORT_SO, "port")
    return _port


def _feat(q, k):
    if q is None:
        return None, None, 0, 0, 0
    assert q.shape == k.shape and q.ndim == 3
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    return q, k, q.shape[0], q.shape[1], q.shape[2]


class _RefLib(_Lib):
    def __init__(self, path, kind):
        super().__init__(path, kind)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_mask.argtypes = [C.c_int, C.c_int, C.c_int, _P(_Cfg), C.c_uint64, C.c_int,
                                     _f32p, _f32p, C.c_int64, C.c_int, C.c_int, _u8p,
                                     _P(C.c_double)]
        L.ref_oracle_build.argtypes = [C.c_int, C.c_int, C.c_int, _P(_Cfg), C.c_uint64, C.c_int,
                                       _f32p, _f32p, C.c_int64, C.c_int, C.c_int, _u8p]
        L.ref_masked_attention.argtypes = [C.c_int, C.c_int, C.c_int, _u8p, _f32p, _f32p, _f32p,
                                           C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double,
                                           _f32p]
        L.ref_expand_mask.argtypes = [C.c_int, C.c_int, C.c_int, _u8p, _u8p]
        L.ref_random_batch.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_uint64, _f32p, _f32p,
                                       _f32p]
        L.ref_frame_pair.argtypes = [C.c_int, C.c_int, C.c_int, _P(_Cfg), C.c_int, C.c_int,
                                     _P(C.c_int64)]
        L.ref_static_select.argtypes = [C.c_int, C.c_int, C.c_int, _P(_Cfg), C.c_int, C.c_int,
                                        C.c_double, C.c_uint64, _P(C.c_int64), C.c_int64,
                                        _P(C.c_int64)]
        L.ref_proxy_scores.argtypes = [C.c_int, C.c_int, C.c_int, _P(_Cfg), C.c_int, C.c_int,
                                       _f32p, _f32p, C.c_int64, C.c_int, C.c_int, _f32p,
                                       _P(C.c_double), _P(C.c_double)]
        L.ref_write_mask.argtypes = [_u8p, C.c_int64, C.c_int, C.c_char_p]
        L.ref_simulate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double,
                                   C.c_uint64, _f32p]
        L.ref_proxy_cache.argtypes = [C.c_int, C.c_int, C.c_int, _f32p, C.c_int, _f32p,
                                      _P(C.c_double), _P(C.c_double)]
        L.ref_objective.argtypes = [C.c_int, C.c_int, C.c_int, _P(_Cfg), _f32p, C.c_int,
                                    C.c_uint64, C.c_double, C.c_double, _P(C.c_double)]
        L.ref_read_mask.argtypes = [C.c_char_p, _u8p, C.c_int64, _P(C.c_int64)]
        L.ref_dynamic_select.argtypes = [C.c_int, C.c_int, C.c_int, _P(_Cfg), C.c_int, C.c_int,
                                         _P(C.c_double), C.c_int64, C.c_double, C.c_int,
                                         _P(C.c_int64), C.c_int64, _P(C.c_int64)]

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def build_mask(self, nf, nt, bs, cfg: Cfg, seed, disable_split=False, q=None, k=None,
                   timings=None):
        _, _, blocks, rb = grid_dims(nf, nt, bs)
        out = np.zeros((blocks, rb), np.uint8)
        q, k, tok, h, d = _feat(q, k)
        t = (C.c_double * 5)()
        c = cfg.c()
        self._chk(self.lib.ref_build_mask(nf, nt, bs, C.byref(c), seed, int(disable_split),
                                          _fp(q), _fp(k), tok, h, d,
                                          out.ctypes.data_as(_u8p), t))
        if timings is not None:
            timings.update(candidates_s=t[0], selection_s=t[1], aggregation_s=t[2],
                           retained_frame_pairs=int(t[3]), scored_pairs=int(t[4]))
        return out

    def oracle_build(self, nf, nt, bs, cfg: Cfg, seed, disable_split=False, q=None, k=None):
        _, _, blocks, _ = grid_dims(nf, nt, bs)
        out = np.zeros((blocks, blocks), np.uint8)
        q, k, tok, h, d = _feat(q, k)
        c = cfg.c()
        self._chk(self.lib.ref_oracle_build(nf, nt, bs, C.byref(c), seed, int(disable_split),
                                            _fp(q), _fp(k), tok, h, d,
                                            out.ctypes.data_as(_u8p)))
        return out

    def masked_attention(self, nf, nt, bs, bits, q, k, v, exact=True, eps=1e-10):
        _, padded, _, _ = grid_dims(nf, nt, bs)
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        tok, h, d = q.shape
        out = np.zeros((padded, h, d), np.float32)
        bits = np.ascontiguousarray(bits, np.uint8)
        self._chk(self.lib.ref_masked_attention(nf, nt, bs, bits.ctypes.data_as(_u8p), _fp(q),
                                                _fp(k), _fp(v), tok, h, d, int(exact), eps,
                                                _fp(out)))
        return out

    def expand_mask(self, nf, nt, bs, bits):
        _, padded, _, _ = grid_dims(nf, nt, bs)
        out = np.zeros((padded, (padded + 7) // 8), np.uint8)
        bits = np.ascontiguousarray(bits, np.uint8)
        self._chk(self.lib.ref_expand_mask(nf, nt, bs, bits.ctypes.data_as(_u8p),
                                           out.ctypes.data_as(_u8p)))
        return out

    def random_batch(self, tokens, heads, d, seed, with_values=True):
        q = np.zeros((tokens, heads, d), np.float32)
        k = np.zeros_like(q)
        v = np.zeros_like(q) if with_values else None
        self._chk(self.lib.ref_random_batch(tokens, heads, d, seed, _fp(q), _fp(k), _fp(v)))
        return q, k, v

    def frame_pair(self, nf, nt, bs, cfg: Cfg, i, j):
        out = (C.c_int64 * 5)()
        c = cfg.c()
        self._chk(self.lib.ref_frame_pair(nf, nt, bs, C.byref(c), i, j, out))
        return tuple(out)

    # ---- the profiler's objective (profiler.cpp:49-148) ----
    def simulate(self, nf, nt, bs, feature_dim, seed, drift_rate=None, regime=None,
                 spatial_scale=-1.0):
        """proxy.cpp simulate: by drift rate, or by regime (0 Low, 1 Mid, 2 High)."""
        n = nf * nt
        out = np.zeros((n, feature_dim), np.float32)
        dr = -(regime + 1.0) if regime is not None else float(drift_rate)
        self._chk(self.lib.ref_simulate(nf, nt, bs, dr, feature_dim, spatial_scale, seed,
                                        _fp(out)))
        return out

    def proxy_cache(self, nf, nt, bs, features, with_weights=False):
        f = np.ascontiguousarray(features, np.float32)
        n = f.shape[0]
        w = np.zeros((n, n), np.float32) if with_weights else None
        rs = np.zeros(n, np.float64)
        sq = C.c_double()
        self._chk(self.lib.ref_proxy_cache(nf, nt, bs, _fp(f), f.shape[1],
                                           _fp(w) if w is not None else None,
                                           rs.ctypes.data_as(_P(C.c_double)), C.byref(sq)))
        return w, rs, sq.value

    def objective(self, nf, nt, bs, cfg: Cfg, features, batch_seed, penalty_weight=10.0,
                  sparsity_target=0.8):
        """objective(c, batch, ...) -> (loss, mse, achieved_sparsity)."""
        f = np.ascontiguousarray(features, np.float32)
        out = (C.c_double * 3)()
        c = cfg.c()
        self._chk(self.lib.ref_objective(nf, nt, bs, C.byref(c), _fp(f), f.shape[1], batch_seed,
                                         penalty_weight, sparsity_target, out))
        return tuple(out)

    def static_select(self, nf, nt, bs, cfg: Cfg, i, j, ratio, seed):
        n = self.frame_pair(nf, nt, bs, cfg, i, j)[2]
        cap = max(1, n)
        out = np.zeros((cap, 2), np.int64)
        kk = C.c_int64()
        c = cfg.c()
        self._chk(self.lib.ref_static_select(nf, nt, bs, C.byref(c), i, j, ratio, seed,
                                             out.ctypes.data_as(_P(C.c_int64)), cap,
                                             C.byref(kk)))
        return out[: kk.value]

    def proxy_scores(self, nf, nt, bs, cfg: Cfg, i, j, q, k):
        n = self.frame_pair(nf, nt, bs, cfg, i, j)[2]
        q, k, tok, h, d = _feat(q, k)
        s = np.zeros(max(n, 1), np.float32)
        z = np.zeros(max(n, 1), np.float64)
        st = (C.c_double * 2)()
        c = cfg.c()
        self._chk(self.lib.ref_proxy_scores(nf, nt, bs, C.byref(c), i, j, _fp(q), _fp(k), tok,
                                            h, d, _fp(s), z.ctypes.data_as(_P(C.c_double)),
                                            st))
        return s[:n], z[:n], (st[0], st[1])

    def write_mask(self, bits, dim, fmt, path):
        bits = np.ascontiguousarray(bits, np.uint8)
        self._chk(self.lib.ref_write_mask(bits.ctypes.data_as(_u8p), dim, fmt, path.encode()))

    def read_mask(self, path, cap=1 << 26):
        buf = np.zeros(cap, np.uint8)
        dim = C.c_int64()
        self._chk(self.lib.ref_read_mask(path.encode(), buf.ctypes.data_as(_u8p), cap,
                                         C.byref(dim)))
        rb = (dim.value + 7) // 8
        return dim.value, buf[: dim.value * rb].reshape(dim.value, rb).copy()

    def dynamic_select(self, nf, nt, bs, cfg: Cfg, i, j, z, tau, fallback_k):
        z = np.ascontiguousarray(z, np.float64)
        n = z.size
        cap = max(1, n)
        out = np.zeros((cap, 2), np.int64)
        kk = C.c_int64()
        c = cfg.c()
        self._chk(self.lib.ref_dynamic_select(nf, nt, bs, C.byref(c), i, j,
                                              z.ctypes.data_as(_P(C.c_double)), n, tau,
                                              fallback_k, out.ctypes.data_as(_P(C.c_int64)),
                                              cap, C.byref(kk)))
        return out[: kk.value]


class _PortLib(_Lib):
    def __init__(self, path, kind):
        super().__init__(path, kind)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_make_grid.argtypes = [C.c_int, C.c_int, C.c_int, _P(_Grid)]
        L.orc_frame_pair.argtypes = [_P(_Grid), _P(_Cfg), C.c_int, C.c_int, _P(C.c_int64)]
        L.orc_build_mask.argtypes = [_P(_Grid), _P(_Cfg), C.c_uint64, C.c_int, _f32p, _f32p,
                                     C.c_int64, C.c_int, C.c_int, _u8p, C.c_int,
                                     _P(C.c_int64)]
        L.orc_masked_attention_exact.argtypes = [_P(_Grid), _u8p, _f32p, _f32p, _f32p,
                                                 C.c_int64, C.c_int, C.c_int, C.c_int64,
                                                 C.c_int64, _f32p, C.c_int]
        L.orc_masked_attention.argtypes = [_P(_Grid), _u8p, _f32p, _f32p, _f32p, C.c_int64,
                                           C.c_int, C.c_int, C.c_double, C.c_int64,
                                           C.c_int64, _f32p, C.c_int]
        L.orc_proxy_cache.argtypes = [C.c_int64, C.c_int, _f32p, _f32p, _P(C.c_double),
                                      _P(C.c_double), C.c_int]
        L.orc_objective.argtypes = [_P(_Grid), _P(_Cfg), _f32p, C.c_int, C.c_uint64, C.c_double,
                                    C.c_double, _P(C.c_double), C.c_int]
        L.orc_expand_mask.argtypes = [_P(_Grid), _u8p, _u8p]
        L.orc_expand_mask.restype = None
        L.orc_random_batch.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_uint64, _f32p, _f32p,
                                       _f32p, C.c_int]
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_mix64.restype = C.c_uint64

    def _grid(self, nf, nt, bs):
        g = _Grid()
        rc = self.lib.orc_make_grid(nf, nt, bs, C.byref(g))
        if rc:
            raise OracleError(rc, self.lib.orc_last_error().decode())
        return g

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    def frame_pair(self, nf, nt, bs, cfg: Cfg, i, j):
        g = self._grid(nf, nt, bs)
        out = (C.c_int64 * 5)()
        c = cfg.c()
        self.lib.orc_frame_pair(C.byref(g), C.byref(c), i, j, out)
        return tuple(out)

    def build_mask(self, nf, nt, bs, cfg: Cfg, seed, disable_split=False, q=None, k=None,
                   threads=1, stats=None):
        g = self._grid(nf, nt, bs)
        out = np.zeros((g.blocks_per_dim, g.row_bytes), np.uint8)
        q, k, tok, h, d = _feat(q, k)
        st = (C.c_int64 * 2)()
        c = cfg.c()
        self._chk(self.lib.orc_build_mask(C.byref(g), C.byref(c), seed, int(disable_split),
                                          _fp(q), _fp(k), tok, h, d,
                                          out.ctypes.data_as(_u8p), threads, st))
        if stats is not None:
            stats.update(retained_frame_pairs=st[0], scored_pairs=st[1])
        return out

    def masked_attention_exact(self, nf, nt, bs, bits, q, k, v, row_begin=0, row_end=None,
                               threads=1, eps=None):
        """eps None: masked_attention_exact; eps > 0: soft-mask masked_attention."""
        g = self._grid(nf, nt, bs)
        if row_end is None:
            row_end = g.padded_tokens
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        tok, h, d = q.shape
        out = np.zeros((row_end - row_begin, h, d), np.float32)
        bits = np.ascontiguousarray(bits, np.uint8)
        if eps is None:
            rc = self.lib.orc_masked_attention_exact(C.byref(g), bits.ctypes.data_as(_u8p),
                                                     _fp(q), _fp(k), _fp(v), tok, h, d,
                                                     row_begin, row_end, _fp(out), threads)
        else:
            rc = self.lib.orc_masked_attention(C.byref(g), bits.ctypes.data_as(_u8p), _fp(q),
                                               _fp(k), _fp(v), tok, h, d, float(eps),
                                               row_begin, row_end, _fp(out), threads)
        self._chk(rc)
        return out

    def masked_attention(self, nf, nt, bs, bits, q, k, v, eps=1e-10, **kw):
        return self.masked_attention_exact(nf, nt, bs, bits, q, k, v, eps=eps, **kw)

    def proxy_cache(self, features, with_weights=False, threads=1):
        f = np.ascontiguousarray(features, np.float32)
        n = f.shape[0]
        w = np.zeros((n, n), np.float32) if with_weights else None
        rs = np.zeros(n, np.float64)
        sq = C.c_double()
        self._chk(self.lib.orc_proxy_cache(n, f.shape[1], _fp(f), _fp(w) if w is not None else None,
                                           rs.ctypes.data_as(_P(C.c_double)), C.byref(sq),
                                           threads))
        return w, rs, sq.value

    def objective(self, nf, nt, bs, cfg: Cfg, features, batch_seed, penalty_weight=10.0,
                  sparsity_target=0.8, threads=1):
        g = self._grid(nf, nt, bs)
        f = np.ascontiguousarray(features, np.float32)
        out = (C.c_double * 3)()
        c = cfg.c()
        self._chk(self.lib.orc_objective(C.byref(g), C.byref(c), _fp(f), f.shape[1], batch_seed,
                                         penalty_weight, sparsity_target, out, threads))
        return tuple(out)

    def expand_mask(self, nf, nt, bs, bits):
        g = self._grid(nf, nt, bs)
        out = np.zeros((g.padded_tokens, (g.padded_tokens + 7) // 8), np.uint8)
        bits = np.ascontiguousarray(bits, np.uint8)
        self.lib.orc_expand_mask(C.byref(g), bits.ctypes.data_as(_u8p), out.ctypes.data_as(_u8p))
        return out

    def random_batch(self, tokens, heads, d, seed, with_values=True, threads=1):
        q = np.zeros((tokens, heads, d), np.float32)
        k = np.zeros_like(q)
        v = np.zeros_like(q) if with_values else None
        self.lib.orc_random_batch(tokens, heads, d, seed, _fp(q), _fp(k), _fp(v), threads)
        return q, k, v

    def mix64(self, z):
        return self.lib.orc_mix64(z)


# ---------------------------------------------------------------------------
# Small pure-numpy helpers shared by tests (bit layout of BlockMask,
# mask.hpp:17-35: row-major, LSB-first, row_bytes = ceil(S_b / 8)).

def unpack_bits(bits, blocks):
    return np.unpackbits(bits, axis=1, bitorder="little")[:, :blocks]


def pack_dense(dense):
    return np.packbits(dense.astype(np.uint8), axis=1, bitorder="little")
