"""B200-native thread-safe lattice Boltzmann (arXiv 2304.06437) hot path.

The compute path is libtslb_cuda.so (hand-written sm_100a CUDA behind the
C-ABI in include/tslb_cuda.h). This package holds the kernels (csrc/), the
in-tree build (build.py), the ctypes binding (_lib.py) and a Python mirror of
the reference's solver interface (tslb.py).
"""
from . import _lib  # noqa: F401
from .tslb import *  # noqa: F401,F403

__all__ = [n for n in dir() if not n.startswith("_")]
