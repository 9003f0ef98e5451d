"""O2: dense brute-force oracle (test infrastructure only).

* ``assemble``        -- the dense Psi of PAPER.md:124-130 from D (lower triangle
                         authoritative) and E.
* ``permuted``        -- Phi = P Psi P^T with perm[new] = original (A19).
* ``factor``          -- L^ = chol(P Psi P^T), the unique lower-triangular factor with
                         positive diagonal, via numpy's dense Cholesky,
                         repacked to the C-ABI layout by ``oracle.layout.pack``.
* ``solve``           -- x = Psi^{-1} b by a dense solve.

Intended for N*n <= ~2048.
"""
from __future__ import annotations

import numpy as np

from . import layout
from .perm import perm


def assemble(D: np.ndarray, E: np.ndarray) -> np.ndarray:
    N, n, _ = D.shape
    A = np.zeros((N * n, N * n))
    for i in range(N):
        Dl = np.tril(D[i])
        A[i * n:(i + 1) * n, i * n:(i + 1) * n] = Dl + np.tril(Dl, -1).T
    for i in range(N - 1):
        A[(i + 1) * n:(i + 2) * n, i * n:(i + 1) * n] = E[i]
        A[i * n:(i + 1) * n, (i + 1) * n:(i + 2) * n] = E[i].T
    return A


def perm_matrix(N: int, n: int) -> np.ndarray:
    """Block permutation matrix P with (P Psi P^T)[new, new'] = Psi[perm[new], perm[new']]."""
    P = np.zeros((N * n, N * n))
    for new, orig in enumerate(perm(N)):
        P[new * n:(new + 1) * n, (orig - 1) * n:orig * n] = np.eye(n)
    return P


def permuted(D, E) -> np.ndarray:
    N, n, _ = D.shape
    P = perm_matrix(N, n)
    return P @ assemble(D, E) @ P.T


def factor_dense(D, E) -> np.ndarray:
    """Dense L^ with P Psi P^T = L^ L^^T (raises numpy LinAlgError if not SPD)."""
    return np.linalg.cholesky(permuted(D, E))


def factor(D, E) -> tuple[np.ndarray, np.ndarray]:
    """(Dhat, C) in the C-ABI layout, from the dense factor of P Psi P^T."""
    N, n, _ = D.shape
    L = factor_dense(D, E)
    pos = {orig: new for new, orig in enumerate(perm(N))}

    def Lblock(r, c):
        pr, pc = pos[r], pos[c]
        if pr < pc:
            return None
        return L[pr * n:(pr + 1) * n, pc * n:(pc + 1) * n]

    return layout.pack(N, n, Lblock)


def solve(D, E, b) -> np.ndarray:
    """x = Psi^{-1} b, b and x shaped [N, n, m]."""
    N, n, m = b.shape
    x = np.linalg.solve(assemble(D, E), b.reshape(N * n, m))
    return x.reshape(N, n, m)
