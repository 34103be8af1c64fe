"""B200-native mixed-precision SLDG translate-and-project step (arXiv:1603.07008).

The compute path is libsldg.so (hand-written sm_100a CUDA behind the C ABI in
include/sldg.h); ``sldg`` is its thin ctypes binding.  No CPU fallback exists.
"""
from . import sldg  # noqa: F401
from .sldg import Grid, SldgError, VlasovPoisson  # noqa: F401

__all__ = ["sldg", "Grid", "SldgError", "VlasovPoisson"]
