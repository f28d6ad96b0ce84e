"""B200-native AIFMM (Gujjula & Ambikasaran, arXiv 2301.12704): factorization hot path.

`aifmm` (the ctypes binding of libaifmm.so, include/aifmm.h) is the product path; it fails
loudly when the CUDA library is missing.  `workloads` holds the seeded input generators.
"""
from . import workloads  # noqa: F401
