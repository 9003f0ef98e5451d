"""Mixed-precision iterative refinement ("mixed-precision
strategies") -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper names mixed precision as future work and gives no algorithm, so this follows the
textbook one (classical iterative refinement, Wilkinson 1963 / Moler 1967; Higham, "Accuracy
and Stability of Numerical Algorithms", Alg. 12.1 with a low-precision factorization), in this
order (reading R8):

    1. factor Psi once in binary32:        P Psi32 P^T = L32 L32^T     (Psi32 = fl32(Psi))
    2. x_0 = solve32(fl32(b)), upcast to binary64
    3. for k = 1 .. iters:
         r_k = b - Psi x_{k-1}           (binary64, Psi in binary64)
         d_k = solve32(fl32(r_k))        (the binary32 factor of step 1)
         x_k = x_{k-1} + d_k             (binary64)

Step 1 and the binary32 solves use O3 (``oracle.ndchol``, the generic block-sparse
right-looking Cholesky in the order P_inf) fed with float32 arrays, so every operation of the
factor and of the solves rounds to binary32 as numpy's float32 kernels do. ``psi_matvec`` is
the plain definition of the block-tridiagonal product (lower triangle of D
authoritative). Pinned in tests/test_oracle_ext.py: convergence to the dense
binary64 solution within the classical bound, iters = 0 equal to the binary32 solve, a
contraction factor of order kappa * u32 per step, and psi_matvec against the dense assembly.
"""
from __future__ import annotations

import numpy as np

from . import ndchol


def psi_matvec(D: np.ndarray, E: np.ndarray, x: np.ndarray) -> np.ndarray:
    """y = Psi x for one system: y_i = D_i x_i + E_{i-1} x_{i-1} + E_i^T x_{i+1} (binary64)."""
    D, E, x = (np.asarray(a, dtype=np.float64) for a in (D, E, x))
    N = D.shape[0]
    y = np.zeros_like(x)
    for i in range(N):
        Dl = np.tril(D[i])
        y[i] = (Dl + np.tril(Dl, -1).T) @ x[i]
        if i > 0:
            y[i] += E[i - 1] @ x[i - 1]
        if i < N - 1:
            y[i] += E[i].T @ x[i + 1]
    return y


def refine(D: np.ndarray, E: np.ndarray, b: np.ndarray, iters: int, history: list | None = None):
    """x after ``iters`` refinement steps on a binary32 factorization (module docstring).

    ``history`` (optional) receives x_0, x_1, ..., x_iters.
    Returns (x, Dhat32, C32): the binary64 solution and the binary32 factor in the C-ABI layout.
    """
    D, E, b = (np.asarray(a, dtype=np.float64) for a in (D, E, b))
    D32, E32 = D.astype(np.float32), E.astype(np.float32)
    L, order = ndchol.factor_blocks(D32, E32)                                   # step 1
    x = ndchol.solve_with_blocks(L, order, b.astype(np.float32)).astype(np.float64)  # step 2
    if history is not None:
        history.append(x.copy())
    for _ in range(iters):                                                      # step 3
        r = b - psi_matvec(D, E, x)
        d = ndchol.solve_with_blocks(L, order, r.astype(np.float32)).astype(np.float64)
        x = x + d
        if history is not None:
            history.append(x.copy())
    from . import layout
    N, n, _ = D.shape
    Dhat, C = layout.pack(N, n, lambda r_, c_: L.get((r_, c_)))
    return x, Dhat, C
