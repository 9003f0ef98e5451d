"""Block-banded SPD systems of block bandwidth w -- TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

PAPER.md:821 names "extension to block banded matrices with larger bandwidth" as future work
(SPEC.md:182). The matrix has N diagonal blocks D_i (n x n, lower triangle
authoritative) and, for k = 1..w, sub-diagonal blocks A_k[i] = block (i+k, i), i = 1..N-k:

    Psi_w[i, i] = D_i,   Psi_w[i+k, i] = A_k[i],   Psi_w[i, i+k] = A_k[i]^T.

A block-banded matrix of bandwidth w IS block tridiagonal in super-blocks of w consecutive
blocks (size w*n): super-block I holds the original blocks (I-1)w+1 .. Iw, and every nonzero
block (r, c) has |r - c| <= w, so it lies in super-blocks I = J or |I - J| = 1. When w does
not divide N, the last super-block is padded with identity diagonal blocks (unknowns that
solve to zero with a zero right-hand side); this changes no value of the solution.

Plain definitions:

* ``assemble`` -- the dense Psi_w.
* ``reblock``  -- (D', E') of the super-block tridiagonal matrix, sliced out of the dense
                  padded Psi_w (no index arithmetic shared with the CUDA packing kernel).
* ``factor``   -- (Dhat', C') of the reblocked system by O3 (``oracle.ndchol``).
* ``solve``    -- x = Psi_w^{-1} b by a dense solve.

Pinned in tests/test_oracle_ext.py: w = 1 reproduces (D, E) exactly, the dense assembly of
the reblocked matrix equals the padded Psi_w, blocks farther than w from the diagonal never
appear in E', and a known solution.
"""
from __future__ import annotations

import numpy as np

from . import dense, ndchol


def assemble(D, A) -> np.ndarray:
    """Dense Psi_w; D [N, n, n], A [w, N, n, n] with A[k-1][i-1] = block (i+k, i)."""
    D, A = np.asarray(D, dtype=np.float64), np.asarray(A, dtype=np.float64)
    N, n, _ = D.shape
    w = A.shape[0]
    M = np.zeros((N * n, N * n))
    for i in range(N):
        Dl = np.tril(D[i])
        M[i * n:(i + 1) * n, i * n:(i + 1) * n] = Dl + np.tril(Dl, -1).T
    for k in range(1, w + 1):
        for i in range(N - k):
            r = i + k
            M[r * n:(r + 1) * n, i * n:(i + 1) * n] = A[k - 1][i]
            M[i * n:(i + 1) * n, r * n:(r + 1) * n] = A[k - 1][i].T
    return M


def padded(D, A) -> np.ndarray:
    """Psi_w padded with identity rows/columns to N' w blocks, N' = ceil(N / w)."""
    N, n, _ = np.asarray(D).shape
    w = np.asarray(A).shape[0]
    Np = -(-N // w)
    M = np.eye(Np * w * n)
    M[:N * n, :N * n] = assemble(D, A)
    return M


def reblock(D, A):
    """(D' [N', w n, w n], E' [N'-1, w n, w n]) sliced from the padded dense matrix."""
    N, n, _ = np.asarray(D).shape
    w = np.asarray(A).shape[0]
    Np = -(-N // w)
    M = padded(D, A)
    s = w * n
    Dp = np.stack([M[I * s:(I + 1) * s, I * s:(I + 1) * s] for I in range(Np)])
    Ep = np.stack([M[(I + 1) * s:(I + 2) * s, I * s:(I + 1) * s] for I in range(Np - 1)]) if Np > 1 \
        else np.zeros((0, s, s))
    return Dp, Ep


def factor(D, A):
    """(Dhat', C') of the reblocked block-tridiagonal system (O3)."""
    Dp, Ep = reblock(D, A)
    return ndchol.factor(Dp, Ep)


def solve(D, A, b) -> np.ndarray:
    """x [N, n, m] = Psi_w^{-1} b."""
    b = np.asarray(b, dtype=np.float64)
    N, n, m = b.shape
    return np.linalg.solve(assemble(D, A), b.reshape(N * n, m)).reshape(N, n, m)


def reblocked_dense(D, A) -> np.ndarray:
    """Dense assembly of (D', E') through O2's block-tridiagonal assembly (pin helper)."""
    Dp, Ep = reblock(D, A)
    return dense.assemble(Dp, Ep)
