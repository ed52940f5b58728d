"""B200-native DynamicRad sparse-attention hot path (sm_100a).

The product is libdynrad.so (CUDA kernels behind the C ABI in
include/dynrad.h); `radialplan` mirrors the reference's operator API on top.
"""
from . import radialplan  # noqa: F401

__all__ = ["radialplan"]
