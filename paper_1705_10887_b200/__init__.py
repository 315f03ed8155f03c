"""B200-native sparse biharmonic MDS (sBMDS) hot path — arXiv 1705.10887.

The operator -1/2 J S D_ll S^T J and the block subspace eigensolver run in
hand-written sm_100a CUDA kernels behind the C ABI in include/sbmds.h
(libsbmds.so); this package is the thin Python binding over it.
"""
from .sbmds import Sbmds, SbmdsError, from_problem, launch_count  # noqa: F401

__all__ = ["Sbmds", "SbmdsError", "from_problem", "launch_count"]
