"""B200-native assembly of RT0 / NE0 edge-element mass and stiffness matrices
(Anjam & Valdman, arXiv:1409.4618).  The hot path is libefem.so (CUDA,
sm_100a) behind the C-ABI in include/efem.h; this package is its thin Python
binding.  Importing the API requires the built library (no fallback)."""

from ._lib import EfemError, declared_symbols  # noqa: F401

__all__ = ["EfemError", "declared_symbols"]
