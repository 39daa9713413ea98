"""B200-native FP64 matrix-free p-multigrid hot path (arXiv 2204.01722).

The compute path is the in-tree CUDA library ``libhexmg_b200.so`` (sm_100a),
reached through its C-ABI (``include/hexmg_b200.h``).  There is no CPU
fallback: importing :mod:`paper_2204_01722_b200.capi` raises if the library
is missing, and every operation runs on the GPU.
"""
from .capi import HxgError, lib, library_path  # noqa: F401

__all__ = ["HxgError", "lib", "library_path"]
