"""B200-native GPU side of the arXiv 2303.11811 coupled LBM/PSM/DEM solver.

The product is ``liblbg.so`` (CUDA for sm_100a, C-ABI in ``include/lbg.h``); this package
holds its ctypes binding (``lbg``), the host mirror of the reference operator API
(``lbdem``) and the fluid-step driver (``driver``).
"""
from . import lbg  # noqa: F401

__all__ = ["lbg"]
