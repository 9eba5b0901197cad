"""paper_1501_01809_b200 -- B200-native PyOP2 par_loop hot path (arXiv 1501.01809).

The product is libloam_gpu.so (hand-written sm_100a CUDA behind the C ABI in
include/loam_gpu.h).  `capi` is the ctypes binding, `loam` mirrors the
reference operator surface, `configs` builds the BASELINE input sets.
"""
from . import capi  # noqa: F401

__all__ = ["capi", "loam", "configs"]
