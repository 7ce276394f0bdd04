"""B200-native fast DVM collision operator (Mouhot, Pareschi & Rey, arXiv 1201.3986).

The operator runs in libdvm.so (hand-written sm_100a CUDA behind the C ABI of
include/dvm.h); this package is the thin binding plus the multi-GPU plumbing.
"""
from .dvm import (DVM_HARD_SPHERES_3D, DVM_MAXWELL_2D, DvmError, Plan, load)  # noqa: F401
from . import parallel  # noqa: F401

__all__ = ["Plan", "DvmError", "load", "DVM_MAXWELL_2D", "DVM_HARD_SPHERES_3D", "parallel"]
