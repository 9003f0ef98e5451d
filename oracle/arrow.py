"""Block-tridiagonal-arrow (arrowhead) systems -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

PAPER.md:532: the permuted-Cholesky view "enables natural extensions to arrow structures"
(SURVEY.md §8(f) f4). The arrow matrix adds a dense border of size n_a coupled to every block:

    K = [[Psi, G^T],      Psi block tridiagonal (D, E) as in PAPER.md:124-130,
         [G,   Z  ]]      G = [G_1 ... G_N], G_i in R^{n_a x n}; Z in R^{n_a x n_a} SPD
                          (lower triangle authoritative, like D).

The border is the root separator of the nested dissection: it is eliminated last, so the
ordering is P_a = diag(P_inf, I) and the factor of P_a K P_a^T is

    [[L^, 0  ],     L^ the factor of P Psi P^T (Algorithm 4),
     [W,  L_Z]]     W = G P^T L^^{-T},  L_Z = chol(Z - W W^T) = chol(Z - G Psi^{-1} G^T).

Plain definitions, by dense numpy linear algebra (brute force, N*n + n_a <= ~2048):

* ``assemble``  -- dense K.
* ``factor``    -- (Dhat, C, V, L_Z): L^ in the C-ABI layout and L_Z, both read off the dense
                   Cholesky factor of P_a K P_a^T; V = Psi^{-1} G^T by a dense solve (the
                   quantity the C ABI returns in place of W, reading R9).
* ``solve``     -- [x; x_a] = K^{-1} [b; b_a] by a dense solve.

Pinned in tests/test_oracle_ext.py: a hand-worked scalar instance, G = 0 (decoupled: L_Z =
chol(Z), x_a = Z^{-1} b_a), the Schur-complement identity L_Z L_Z^T = Z - G V, and a known
solution.
"""
from __future__ import annotations

import numpy as np

from . import dense, layout
from .perm import perm


def assemble(D, E, G, Z) -> np.ndarray:
    D, E, G, Z = (np.asarray(a, dtype=np.float64) for a in (D, E, G, Z))
    N, n, _ = D.shape
    na = Z.shape[0]
    K = np.zeros((N * n + na, N * n + na))
    K[:N * n, :N * n] = dense.assemble(D, E)
    for i in range(N):
        K[N * n:, i * n:(i + 1) * n] = G[i]
        K[i * n:(i + 1) * n, N * n:] = G[i].T
    Zl = np.tril(Z)
    K[N * n:, N * n:] = Zl + np.tril(Zl, -1).T
    return K


def factor(D, E, G, Z):
    """(Dhat, C, V, L_Z) for one system (module docstring)."""
    D, E, G, Z = (np.asarray(a, dtype=np.float64) for a in (D, E, G, Z))
    N, n, _ = D.shape
    na = Z.shape[0]
    Pa = np.zeros((N * n + na, N * n + na))
    Pa[:N * n, :N * n] = dense.perm_matrix(N, n)
    Pa[N * n:, N * n:] = np.eye(na)
    Lf = np.linalg.cholesky(Pa @ assemble(D, E, G, Z) @ Pa.T)
    pos = {orig: new for new, orig in enumerate(perm(N))}

    def Lblock(r, c):
        pr, pc = pos[r], pos[c]
        if pr < pc:
            return None
        return Lf[pr * n:(pr + 1) * n, pc * n:(pc + 1) * n]

    Dhat, C = layout.pack(N, n, Lblock)
    LZ = Lf[N * n:, N * n:].copy()
    Gt = np.concatenate([G[i].T for i in range(N)], axis=0)  # [N n, n_a]
    V = np.linalg.solve(dense.assemble(D, E), Gt).reshape(N, n, na)
    return Dhat, C, V, LZ


def solve(D, E, G, Z, b, ba):
    """(x [N, n, m], x_a [n_a, m]) = K^{-1} [b; b_a]."""
    D = np.asarray(D, dtype=np.float64)
    N, n, _ = D.shape
    b, ba = np.asarray(b, dtype=np.float64), np.asarray(ba, dtype=np.float64)
    m = b.shape[2]
    rhs = np.concatenate([b.reshape(N * n, m), ba], axis=0)
    sol = np.linalg.solve(assemble(D, E, G, Z), rhs)
    return sol[:N * n].reshape(N, n, m), sol[N * n:]
