"""Partition permutation and Algorithm 2 -- TEST INFRASTRUCTURE ONLY
(oracle/__init__.py). SURVEY.md §8(f) f3.

p - 1 pivot blocks split the N blocks of Psi into p chunks of N_1..N_p consecutive blocks
(N = sum N_k + p - 1); in original order: chunk 1, pivot A_2, chunk 2, pivot A_3, ..., chunk p
(PAPER.md:197-214). Couplings (readings, R10):

    E_ik  = Psi[D_{i+1,k}, D_ik]        inside chunk k
    B_k   = Psi[D_1k, A_k]              (k > 1; the block under A_k in PAPER.md:207)
    F_k   = Psi[A_{k+1}, D_{N_k k}]     (k < p; the block left of A_{k+1})

P_p moves the pivots to the end. Functions:

* ``chunk_sizes_prop1`` -- Proposition 1 with the paper's rounding strategy
  (round N_k* down and up, N_1 from the block count, keep the lower maximum cost of the
  table at). The text writes N_1* = N - (p-1) N_k*; the proof's constraint
  N - (p-1) = N_1 + (p-1) N_k is used (reading R10).
* ``split``        -- original block indices of chunks and pivots.
* ``algorithm2``   -- Algorithm 2 line by line: parallel phase per chunk
  (natural-order block Cholesky of the chunk, border fill B^, F^, H^), then the sequential
  phase on the pivots. Returns every L_p block and the reduced pivot system S (Schur
  complement of the chunks, the matrix the sequential phase factors) before the phase runs.
  The loop bound "N_p - 1" of l.4 is read as N_k - 1 (typo).
* ``factor_dense`` -- L_p = chol(P_p Psi P_p^T) by numpy (plain definition, brute force).

Pinned in tests/test_oracle_ext.py against factor_dense (every block of L_p), Prop. 1's
closed form and the 19/7 ratio, and S against the dense Schur complement.
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular

from . import dense


def chunk_sizes_prop1(N: int, p: int) -> list[int]:
    """[N_1, N_2, ..., N_p] by Proposition 1 and the rounding strategy of PAPER.md:336."""
    assert p >= 1 and N >= 2 * p - 1
    if p == 1:
        return [N]
    best = None
    nk_star = (7 * N - 7 * p + 7) / (7 * p + 12)
    for nk in {int(np.floor(nk_star)), int(np.ceil(nk_star))}:
        n1 = N - (p - 1) - (p - 1) * nk
        if nk < 1 or n1 < 1:
            continue
        cost = max(7 / 3 * n1 - 1, 19 / 3 * nk - 1)  # PAPER.md:315-321 (units of n^3)
        if best is None or cost < best[0]:
            best = (cost, [n1] + [nk] * (p - 1))
    assert best is not None
    return best[1]


def split(sizes: list[int]):
    """(chunks, pivots): chunks[k] = list of 1-based original indices of chunk k+1; pivots[k] =
    original index of A_{k+2} (the pivot after chunk k+1)."""
    chunks, pivots, i = [], [], 1
    for k, Nk in enumerate(sizes):
        chunks.append(list(range(i, i + Nk)))
        i += Nk
        if k < len(sizes) - 1:
            pivots.append(i)
            i += 1
    return chunks, pivots


def perm_p(sizes: list[int]) -> list[int]:
    """P_p as perm[new] = original (1-based): chunk blocks in order, then the pivots."""
    chunks, pivots = split(sizes)
    return [i for c in chunks for i in c] + pivots


def _blk(D, E, r, c):
    """Block (r, c) of Psi (1-based original indices), lower triangle of D authoritative."""
    if r == c:
        Dl = np.tril(D[r - 1])
        return Dl + np.tril(Dl, -1).T
    if r == c + 1:
        return E[c - 1].copy()
    if c == r + 1:
        return E[r - 1].T.copy()
    return np.zeros_like(D[0])


def algorithm2(D, E, sizes: list[int]):
    """Algorithm 2. Returns a dict with the L_p blocks keyed by original
    (row, col) indices (lower orientation of P_p Psi P_p^T) and ``S_diag`` / ``S_off``: the
    pivot system after the parallel phase, S_diag[k-2] = A^_k - F^_{k-1} F^_{k-1}^T (k = 2..p)
    and S_off[k-2] = H^_k (coupling A_{k+1}, A_k; k = 2..p-1)."""
    D, E = np.asarray(D, dtype=np.float64), np.asarray(E, dtype=np.float64)
    p = len(sizes)
    chunks, pivots = split(sizes)
    piv = {k: pivots[k - 2] for k in range(2, p + 1)}  # A_k -> original index
    L: dict = {}
    Ahat, Fhat, Hhat = {}, {}, {}
    # ---------------- parallel phase (independent per k)
    for k in range(1, p + 1):
        c = chunks[k - 1]
        Nk = len(c)
        Dw = {i: _blk(D, E, c[i - 1], c[i - 1]) for i in range(1, Nk + 1)}  # working D_ik
        if k > 1:
            Ahat[k] = _blk(D, E, piv[k], piv[k])                            # l.2
            Bt = _blk(D, E, c[0], piv[k]).T                                 # l.3: B^_1k^T = B_k^T
        for i in range(1, Nk):                                              # l.4 (N_k - 1)
            Dh = np.linalg.cholesky(Dw[i])                                  # l.5
            L[(c[i - 1], c[i - 1])] = Dh
            Eh = solve_triangular(Dh, _blk(D, E, c[i], c[i - 1]).T, lower=True).T  # l.6
            L[(c[i], c[i - 1])] = Eh
            Dw[i + 1] = Dw[i + 1] - Eh @ Eh.T                               # l.7
            if k > 1:
                Bt = solve_triangular(Dh, Bt.T, lower=True).T               # l.9
                L[(piv[k], c[i - 1])] = Bt
                Ahat[k] = Ahat[k] - Bt @ Bt.T                               # l.10
                Bt = -Bt @ Eh.T                                             # l.11
        Dh = np.linalg.cholesky(Dw[Nk])                                     # l.13
        L[(c[-1], c[-1])] = Dh
        if k > 1:
            Bt = solve_triangular(Dh, Bt.T, lower=True).T                   # l.15
            L[(piv[k], c[-1])] = Bt
            Ahat[k] = Ahat[k] - Bt @ Bt.T                                   # l.16
        if k < p:
            Fhat[k] = solve_triangular(Dh, _blk(D, E, piv[k + 1], c[-1]).T, lower=True).T  # l.18
            L[(piv[k + 1], c[-1])] = Fhat[k]
        if 1 < k < p:
            Hhat[k] = -Fhat[k] @ Bt.T                                       # l.19: -F^_k B^_{N_k k}
    # pivot system handed to the sequential phase (deferred F^ update of l.22 applied)
    S_diag = [Ahat[k] - Fhat[k - 1] @ Fhat[k - 1].T for k in range(2, p + 1)]
    S_off = [Hhat[k].copy() for k in range(2, p)]
    # ---------------- sequential phase
    for k in range(2, p):
        Ahat[k] = Ahat[k] - Fhat[k - 1] @ Fhat[k - 1].T                     # l.22
        Ahat[k] = np.linalg.cholesky(Ahat[k])                               # l.23
        L[(piv[k], piv[k])] = Ahat[k]
        Hhat[k] = solve_triangular(Ahat[k], Hhat[k].T, lower=True).T        # l.24
        L[(piv[k + 1], piv[k])] = Hhat[k]
        Ahat[k + 1] = Ahat[k + 1] - Hhat[k] @ Hhat[k].T                     # l.25
    if p > 1:
        Ahat[p] = Ahat[p] - Fhat[p - 1] @ Fhat[p - 1].T                     # l.27
        Ahat[p] = np.linalg.cholesky(Ahat[p])                               # l.28
        L[(piv[p], piv[p])] = Ahat[p]
    return dict(L=L, S_diag=S_diag, S_off=S_off, chunks=chunks, pivots=pivots)


def factor_dense(D, E, sizes: list[int]) -> np.ndarray:
    """Dense L_p = chol(P_p Psi P_p^T) (plain definition)."""
    D = np.asarray(D, dtype=np.float64)
    N, n, _ = D.shape
    order = perm_p(sizes)
    Pm = np.zeros((N * n, N * n))
    for new, orig in enumerate(order):
        Pm[new * n:(new + 1) * n, (orig - 1) * n:orig * n] = np.eye(n)
    return np.linalg.cholesky(Pm @ dense.assemble(D, E) @ Pm.T)
