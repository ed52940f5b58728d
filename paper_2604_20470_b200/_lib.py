"""ctypes binding of the C ABI in include/dynrad.h (libdynrad.so, in-tree).

The shared library is the product: every compute call goes to its CUDA
kernels.  There is no Python or CPU fallback; if the library is missing or
no GPU is present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DYNRAD_LIB") or os.path.join(HERE, "libdynrad.so")


# --- exceptions mirroring the reference's exception types -----------------
class RadialplanError(Exception):
    """Base class; `status` is the rp_status code."""

    status = -1


class InvalidArgument(RadialplanError, ValueError):  # std::invalid_argument
    status = 1


class OutOfRange(RadialplanError, IndexError):  # std::out_of_range
    status = 2


class DomainError(RadialplanError, ArithmeticError):  # std::domain_error
    status = 3


class RuntimeFailure(RadialplanError, RuntimeError):  # std::runtime_error
    status = 4


class CudaError(RadialplanError, RuntimeError):  # CUDA failure / no device
    status = 5


_EXC = {1: InvalidArgument, 2: OutOfRange, 3: DomainError, 4: RuntimeFailure, 5: CudaError}


class Grid(C.Structure):
    _fields_ = [
        ("n_frames", C.c_int),
        ("tokens_per_frame", C.c_int),
        ("block_size", C.c_int),
        ("total_tokens", C.c_int64),
        ("padded_tokens", C.c_int64),
        ("blocks_per_dim", C.c_int64),
        ("row_bytes", C.c_int64),
    ]


class Config(C.Structure):
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


class FramePair(C.Structure):
    _fields_ = [
        ("width", C.c_int64),
        ("retained", C.c_int),
        ("pair_count", C.c_int64),
        ("tier", C.c_int),
        ("split_factor", C.c_int64),
        ("retention_or_threshold", C.c_double),
    ]


class Tensor(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("dtype", C.c_int),
        ("tokens", C.c_int64),
        ("heads", C.c_int),
        ("head_dim", C.c_int),
        ("token_stride", C.c_int64),
        ("head_stride", C.c_int64),
    ]


class BuildOptions(C.Structure):
    _fields_ = [
        ("disable_split", C.c_int),
        ("score_engine", C.c_int),
        ("recheck_delta", C.c_double),
        ("shard_index", C.c_int),
        ("shard_count", C.c_int),
    ]


class Trial(C.Structure):
    _fields_ = [("loss", C.c_double), ("mse", C.c_double), ("achieved_sparsity", C.c_double)]


class BuildStats(C.Structure):
    _fields_ = [
        ("retained_frame_pairs", C.c_int64),
        ("scored_pairs", C.c_int64),
        ("sampled_pairs", C.c_int64),
        ("rechecked_pairs", C.c_int64),
        ("fallback_frame_pairs", C.c_int64),
        ("active_blocks", C.c_int64),
    ]


class Band(C.Structure):
    _fields_ = [
        ("frame_i", C.c_int),
        ("frame_j", C.c_int),
        ("tokens_per_frame", C.c_int64),
        ("width", C.c_int64),
        ("retained", C.c_int),
    ]


RP_F32, RP_BF16 = 0, 1

_lib = None

_P = C.POINTER
_v = C.c_void_p
_SIGS = {
    "rp_last_error": ([], C.c_char_p),
    "rp_version": ([], C.c_char_p),
    "rp_kernel_launch_count": ([], C.c_int64),
    "rp_make_grid": ([C.c_int, C.c_int, C.c_int, _P(Grid)], C.c_int),
    "rp_config_defaults": ([_P(Config)], None),
    "rp_config_validate": ([_P(Config)], C.c_int),
    "rp_frame_pair_info": ([_P(Grid), _P(Config), C.c_int, C.c_int, _P(FramePair)], C.c_int),
    "rp_build_options_defaults": ([_P(BuildOptions)], None),
    "rp_plan_create": ([_P(Grid), _P(Config), C.c_uint64, _P(BuildOptions), _P(_v)], C.c_int),
    "rp_plan_destroy": ([_v], None),
    "rp_plan_build_mask": ([_v, _P(Tensor), _P(Tensor), C.c_int, _v, _P(BuildStats), _v],
                           C.c_int),
    "rp_build_mask": ([_P(Grid), _P(Config), C.c_uint64, _P(BuildOptions), _P(Tensor),
                       _P(Tensor), C.c_int, _v, _P(BuildStats), _v], C.c_int),
    "rp_mask_to_csr": ([_P(Grid), _v, _v, _v, C.c_int64, _v, _v, _v], C.c_int),
    "rp_expand_mask": ([_P(Grid), _v, _v, _v], C.c_int),
    "rp_mask_sparsity": ([_P(Grid), _v, _P(C.c_int64), _P(C.c_double), _v], C.c_int),
    "rp_sparse_attention_fwd": ([_P(Grid), _P(Tensor), _P(Tensor), _P(Tensor), _P(Tensor), _v,
                                 _v, _v, C.c_float, _v], C.c_int),
    "rp_sparse_attention_fwd_checked": ([_P(Grid), _P(Tensor), _P(Tensor), _P(Tensor),
                                         _P(Tensor), _v, _v, _v, C.c_float, _v, _v], C.c_int),
    "rp_sparse_layer_host": ([_v, _P(Grid), _v, _v, _v, C.c_int, C.c_int64, C.c_int, C.c_int,
                              C.c_int, _v, _v, _v], C.c_int),
    "rp_profile_stages": ([C.c_int], None),
    "rp_profile_read": ([_v, _v, C.c_int], C.c_int),
    "rp_attention_kernel": ([_P(Grid), C.c_int, C.c_int], C.c_char_p),
    "rp_random_batch": ([C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_int, _P(Tensor),
                         _P(Tensor), _P(Tensor), _v], C.c_int),
    "rp_masked_attention_exact_host": ([_P(Grid), _v, _v, _v, _v, C.c_int, C.c_int64, C.c_int,
                                        C.c_int, _v, _v], C.c_int),
    "rp_soft_attention_fwd": ([_P(Grid), _P(Tensor), _P(Tensor), _P(Tensor), _P(Tensor), _v,
                               C.c_double, C.c_float, _v], C.c_int),
    "rp_masked_attention_host": ([_P(Grid), _v, _v, _v, _v, C.c_int, C.c_int64, C.c_int,
                                  C.c_int, C.c_double, _v, _v], C.c_int),
    "rp_proxy_cache_create": ([_P(Grid), _v, C.c_int, _P(_v), _v], C.c_int),
    "rp_proxy_cache_from_weights": ([_P(Grid), _v, _v, C.c_double, _P(_v), _v], C.c_int),
    "rp_proxy_cache_destroy": ([_v], None),
    "rp_proxy_weights": ([_P(Grid), _v, C.c_int, _v, _v, _P(C.c_double), _v], C.c_int),
    "rp_proxy_cache_stats": ([_v, _v, _P(C.c_double), _v], C.c_int),
    "rp_objective": ([_v, _P(Config), C.c_uint64, _v, C.c_int, C.c_double, C.c_double,
                      _P(Trial), _v, _v], C.c_int),
    "rp_static_select": ([_P(Band), C.c_double, C.c_uint64, _v, C.c_int64, _P(C.c_int64), _v],
                         C.c_int),
    "rp_proxy_scores": ([_P(Tensor), _P(Tensor), C.c_int, _P(Band), _v, _v], C.c_int),
    "rp_normalize_scores": ([_v, C.c_int64, _v, _P(C.c_double), _P(C.c_double), _v], C.c_int),
    "rp_dynamic_select": ([_P(Band), _v, C.c_int64, C.c_double, C.c_int, _v, C.c_int64,
                           _P(C.c_int64), _v], C.c_int),
    "rp_token_mask_to_blocks": ([_v, C.c_int64, C.c_int, _v, _P(C.c_int), _v], C.c_int),
    "rp_pooled_select": ([_P(Grid), _P(Config), _P(Tensor), _P(Tensor), C.c_int, C.c_int,
                          C.c_double, _v, _v], C.c_int),
    "rp_block_mean_pool": ([_P(Grid), _P(Tensor), C.c_int, _v, _v], C.c_int),
}

# Every symbol include/dynrad.h declares (the CPU tests check the exports).
PUBLIC_SYMBOLS = [s for s in _SIGS if not s.startswith("rp_debug")]


def lib():
    """Load libdynrad.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no fallback implementation)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc):
    if rc != 0:
        msg = lib().rp_last_error().decode()
        raise _EXC.get(rc, RadialplanError)(msg)
