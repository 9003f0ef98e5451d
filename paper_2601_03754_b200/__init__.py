"""B200-native (sm_100a) nested-dissection Cholesky for SPD block-tridiagonal systems.

Implements the multi-stage permuted factorization P Psi P^T = L^ L^^T and the level
solve of arXiv 2601.03754 (Algorithms 4 and 6) as hand-written CUDA kernels behind the
C ABI of include/btd.h; this package is the thin Python binding over it.
"""
from .btd import (BtdError, HostWorkspace, Plan, factor, factor_solve, factor_solve_host, lib,  # noqa: F401
                  permutation, solve)
from . import ext, partition  # noqa: F401,E402  (§8(f) extensions: mixed, arrow, banded; partition)

__all__ = ["Plan", "factor", "solve", "factor_solve", "factor_solve_host", "HostWorkspace", "permutation",
           "lib", "BtdError"]
