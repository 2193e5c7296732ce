"""B200-native (sm_100a) mini-batch hot path of Heta (arXiv 2408.09697).

The product is the in-tree native library libhetgpu.so (C-ABI in
include/hetgpu.h); `hetsim` mirrors the reference's interface over it.
"""
from . import hetsim  # noqa: F401

__all__ = ["hetsim"]
