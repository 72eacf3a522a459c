"""B200-native GP-surrogate + Expected-Improvement hot path of arXiv 2403.08131.

The product is the C-ABI library libgpbo.so (include/gpbo.h; CUDA sources in csrc/).  This
package holds its build script and the thin ctypes binding (gpbo.py).  There is no CPU
fallback: gpbo.load() raises if the library has not been built.
"""
from . import gpbo  # noqa: F401

__all__ = ["gpbo"]
