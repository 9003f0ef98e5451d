"""Error measures of SURVEY.md §8(c) A16 (test infrastructure only).

Normwise per system:
  err_L = max_abs(L^ - L^_o) / max_abs(L^_o)   over Dhat and every coupling block
  err_x = ||x - x_o||_inf / ||x_o||_inf
  resid = ||Psi x - b||_2 / ||b||_2            evaluated in fp64
"""
from __future__ import annotations

import numpy as np


def err_L(Dhat, C, Dhat_o, C_o) -> float:
    Dhat, C, Dhat_o, C_o = (np.asarray(a, dtype=np.float64) for a in (Dhat, C, Dhat_o, C_o))
    num = max(np.max(np.abs(Dhat - Dhat_o)), np.max(np.abs(C - C_o)) if C.size else 0.0)
    den = max(np.max(np.abs(Dhat_o)), np.max(np.abs(C_o)) if C_o.size else 0.0)
    return float(num / den)


def err_x(x, x_o) -> float:
    x, x_o = np.asarray(x, dtype=np.float64), np.asarray(x_o, dtype=np.float64)
    return float(np.max(np.abs(x - x_o)) / np.max(np.abs(x_o)))


def residual(D, E, x, b) -> float:
    """||Psi x - b||_2 / ||b||_2 with Psi = tridiag(E, D, E^T) (D lower-authoritative)."""
    D, E, x, b = (np.asarray(a, dtype=np.float64) for a in (D, E, x, b))
    Dl = np.tril(D)
    Ds = Dl + np.swapaxes(np.tril(D, -1), -1, -2)
    r = Ds @ x
    if D.shape[0] > 1:
        r[1:] += E @ x[:-1]
        r[:-1] += np.swapaxes(E, -1, -2) @ x[1:]
    r -= b
    return float(np.linalg.norm(r) / np.linalg.norm(b))


def reconstruction(D, E, Dhat, C) -> float:
    """||P Psi P^T - L^ L^^T||_F / ||Psi||_F, evaluated block-sparsely from the C-ABI layout.

    Uses only the layout definition (include/btd.h): Dhat[i-1] is L^'s diagonal
    block of original block i; slot (l, k) holds block ((k+1)s, ks) of M + M^T.
    Which side is the L^ column is decided by the elimination order P_inf.
    """
    from .perm import coupling_slots, position

    D, E, Dhat, C = (np.asarray(a, dtype=np.float64) for a in (D, E, Dhat, C))
    N, n, _ = D.shape
    pos = position(N)
    # L^ as blocks (row, col) in original indices
    L = {(i, i): np.tril(Dhat[i - 1]) for i in range(1, N + 1)}
    for q, (_l, _k, a, b) in enumerate(coupling_slots(N)):
        if pos[a] < pos[b]:
            L[(b, a)] = C[q]
        else:
            L[(a, b)] = C[q].T
    cols: dict[int, list[int]] = {}
    for (r, c) in L:
        cols.setdefault(c, []).append(r)
    # (L L^T)[r, q] = sum_c L[r, c] L[q, c]^T
    prod: dict[tuple[int, int], np.ndarray] = {}
    for c, rows in cols.items():
        for r in rows:
            for q in rows:
                prod[(r, q)] = prod.get((r, q), 0.0) + L[(r, c)] @ L[(q, c)].T
    ref: dict[tuple[int, int], np.ndarray] = {}
    for i in range(1, N + 1):
        Dl = np.tril(D[i - 1])
        ref[(i, i)] = Dl + np.tril(Dl, -1).T
    for i in range(1, N):
        ref[(i + 1, i)] = E[i - 1]
        ref[(i, i + 1)] = E[i - 1].T
    keys = set(prod) | set(ref)
    num = sum(float(np.sum((prod.get(k, 0.0) - ref.get(k, 0.0)) ** 2)) for k in keys)
    den = sum(float(np.sum(v ** 2)) for v in ref.values())
    return float(np.sqrt(num / den))
