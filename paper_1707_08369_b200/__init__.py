"""B200-native (sm_100a) rank-1 SVD update — Gandhi & Rajgor, arXiv 1707.08369.

Hot path: secular-equation root solve + Cauchy-structured eigenvector apply
(direct DMMA kernel or 1-D Chebyshev FMM) behind the C ABI in include/svd1.h
(libsvd1.so, built in-tree).  This package is the thin Python binding.
"""
from ._lib import (EMULATE_RANKS, FORCE_DIRECT, FORCE_FMM, FORCE_NCCL, FUSED_SIDE, LIB_PATH, SECULAR_DIRECT,  # noqa: F401
                   SECULAR_FMM, THIN_V, nccl_unique_id, version)
from .api import Plan, SVD1Error, update  # noqa: F401
