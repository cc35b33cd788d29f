"""B200-native shared-LHS interleaved batch tri/pentadiagonal solvers.

The product is the C-ABI library libbandsolve_b200.so (include/bandsolve.h),
built from csrc/ for sm_100a. This package only locates it and offers a
ctypes binding (bandsolve.py) for tests, the bench and Python callers.
"""
from .bandsolve import (  # noqa: F401
    Batch,
    BandsolveError,
    Library,
    PentFactor,
    TriFactor,
    UniformPentFactor,
    diffusion_bands,
    hyper_bands,
    load,
)

__all__ = [
    "Batch",
    "BandsolveError",
    "Library",
    "PentFactor",
    "TriFactor",
    "UniformPentFactor",
    "diffusion_bands",
    "hyper_bands",
    "load",
]
