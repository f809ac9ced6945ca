"""B200-native (sm_100a) TGV primal-dual solver -- the hot path of
"Out-of-Core Surface Reconstruction via Global TGV Minimization" (arXiv 2107.14790).

The product is libtgv.so (C ABI, include/tgv.h); ``tgv`` is its thin ctypes
binding.  Importing this package raises if the library is not built: there is
no CPU fallback.
"""
from . import tgv  # noqa: F401  (loads lib/libtgv.so or raises)
from .tgv import Group, Solver, TgvError  # noqa: F401

__all__ = ["tgv", "Solver", "Group", "TgvError"]
