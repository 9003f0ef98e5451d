"""O3: generic block-sparse right-looking Cholesky in the order P_inf (test infrastructure only).

SURVEY.md §8(c) O3. The matrix is held as a map of nonzero n x n blocks keyed by
original block indices. Columns are eliminated one at a time in the order
``perm(N)`` with the textbook submatrix (right-looking)
Cholesky step of PAPER.md:38-41 / Fig. 1 ("Submatrix-Cholesky"):

    L_cc = chol(A_cc)
    L_rc = A_rc L_cc^{-T}                     for every live neighbour r of c
    A_rq = A_rq - L_rc L_qc^T                 for every pair of live neighbours r, q
                                              (creating a fill block when absent)

Fill is discovered symbolically; the routine knows nothing about levels,
strides or the paper's E^ subscripts, so it checks the GPU path's index
arithmetic independently. The result is the unique Cholesky factor of
P Psi P^T, repacked with ``oracle.layout.pack``.

The solve applies the same block-sparse L^: y = L^{-1} (P b), x = P^T L^{-T} y.
Library primitives used as steps: numpy.linalg.cholesky on one n x n block and
scipy.linalg.solve_triangular.
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular

from . import layout
from .perm import perm


class NotPositiveDefinite(Exception):
    def __init__(self, block: int):
        super().__init__(f"pivot block {block} not positive definite")
        self.block = block


def factor_blocks(D: np.ndarray, E: np.ndarray):
    """Return (L, order) where L maps (row, col) original 1-based indices -> L^ block."""
    N, n, _ = D.shape
    order = perm(N)
    pos = {orig: p for p, orig in enumerate(order)}
    A: dict[tuple[int, int], np.ndarray] = {}
    below: dict[int, set[int]] = {i: set() for i in range(1, N + 1)}  # live rows r of column c

    def put(r, c, blk):  # store in the lower orientation of the permuted matrix
        if pos[r] < pos[c]:
            r, c, blk = c, r, blk.T
        A[(r, c)] = blk.copy()
        below[c].add(r)

    for i in range(1, N + 1):
        Dl = np.tril(D[i - 1])
        A[(i, i)] = Dl + np.tril(Dl, -1).T
    for i in range(1, N):
        put(i + 1, i, E[i - 1])

    L: dict[tuple[int, int], np.ndarray] = {}
    for c in order:
        try:
            Lcc = np.linalg.cholesky(A.pop((c, c)))
        except np.linalg.LinAlgError:
            raise NotPositiveDefinite(c) from None
        L[(c, c)] = Lcc
        nbrs = sorted(below.pop(c), key=lambda r: pos[r])
        for r in nbrs:
            # L_rc = A_rc Lcc^{-T}  <=>  Lcc L_rc^T = A_rc^T
            L[(r, c)] = solve_triangular(Lcc, A.pop((r, c)).T, lower=True).T
        for qi, q in enumerate(nbrs):
            for r in nbrs[qi:]:
                upd = L[(r, c)] @ L[(q, c)].T
                key = (r, q)  # pos[r] >= pos[q]
                if key in A:
                    A[key] = A[key] - upd
                else:
                    A[key] = -upd
                    below[q].add(r)
    return L, order


def factor(D, E) -> tuple[np.ndarray, np.ndarray]:
    """(Dhat, C) in the C-ABI layout; also checks there is no fill outside the slots."""
    N, n, _ = D.shape
    L, _order = factor_blocks(D, E)
    layout.check_no_extra_fill(N, {k for k in L if k[0] != k[1]})
    return layout.pack(N, n, lambda r, c: L.get((r, c)))


def solve_with_blocks(L, order, b: np.ndarray) -> np.ndarray:
    """x = Psi^{-1} b using the block-sparse L^ (b, x shaped [N, n, m])."""
    N = len(order)
    pos = {orig: p for p, orig in enumerate(order)}
    cols: dict[int, list[int]] = {c: [] for c in order}
    for (r, c) in L:
        if r != c:
            cols[c].append(r)
    y = {i: b[i - 1].copy() for i in range(1, N + 1)}
    for c in order:  # forward: L^ y = P b
        y[c] = solve_triangular(L[(c, c)], y[c], lower=True)
        for r in cols[c]:
            y[r] = y[r] - L[(r, c)] @ y[c]
    x = dict(y)
    for c in reversed(order):  # backward: L^^T (P x) = y
        rhs = x[c]
        for r in cols[c]:
            rhs = rhs - L[(r, c)].T @ x[r]
        x[c] = solve_triangular(L[(c, c)], rhs, lower=True, trans='T')
    assert all(pos[r] > pos[c] for (r, c) in L if r != c)
    return np.stack([x[i] for i in range(1, N + 1)])


def factor_solve(D, E, b):
    """(Dhat, C, x) for one system."""
    N, n, _ = D.shape
    L, order = factor_blocks(D, E)
    layout.check_no_extra_fill(N, {k for k in L if k[0] != k[1]})
    Dhat, C = layout.pack(N, n, lambda r, c: L.get((r, c)))
    return Dhat, C, solve_with_blocks(L, order, b)
