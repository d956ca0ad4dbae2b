"""B200-native (sm_100a) hot path of QTNH (arXiv 2505.06119): sharded complex128
tensors in HBM, index permutation / local<->distributed swaps, pairwise
contraction on the FP64 tensor cores, in-place gate application.

The compute lives in libqtnh_b200.so (C ABI: include/qtnh_b200.h); this package
is the host-side mirror of the reference's C++ operator API (qtnh.py).
"""
from ._lib import LIB_PATH, kernel_launches, lib  # noqa: F401  (raises if the .so is missing)
from . import qtnh  # noqa: F401

__all__ = ["qtnh", "lib", "LIB_PATH", "kernel_launches"]
