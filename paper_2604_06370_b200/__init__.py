"""paper_2604_06370_b200 — B200-native ForkKV ResidualAttention hot path.

The product: ``libforkkv.so`` (C-ABI, include/forkkv.h; C++ control plane +
sm_100a CUDA kernels) and this thin ctypes binding. Importing the package does
not load the library; ``api.ForkKV`` does, and raises if it is missing.
"""
from ._lib import FkvError  # noqa: F401

__all__ = ["api", "FkvError"]
