"""Map a factor L^ of P Psi P^T onto the C-ABI storage (oracle; test infrastructure only).

The layout is the one declared in include/btd.h:

* ``Dhat[i-1]`` = the diagonal block of L^ belonging to original block i
  (lower triangular, strict upper stored as exact zeros).
* ``C[slot(l, k)]`` for slot (l, k) coupling original blocks a = k s and
  b = (k+1) s (s = 2^(l-1)) holds block (b, a) of  M + M^T, where M is L^ with
  rows and columns relabelled by original block index. Exactly one of M[b,a],
  M[a,b] is a nonzero block (the column is whichever of a, b is eliminated
  first), so for odd k this is the L^ block itself and for even k its transpose
  ("the Psi-lower orientation is kept throughout").

``Lblock(r, c)`` supplies M: the n x n block of L^ at (row r, column c) in
original indices (1-based), or None when that block is structurally zero.
"""
from __future__ import annotations

import numpy as np

from .perm import coupling_slots, position


def pack(N: int, n: int, Lblock) -> tuple[np.ndarray, np.ndarray]:
    slots = coupling_slots(N)
    Dhat = np.zeros((N, n, n))
    C = np.zeros((len(slots), n, n))
    for i in range(1, N + 1):
        Dhat[i - 1] = np.tril(Lblock(i, i))
    for q, (_lev, _k, a, b) in enumerate(slots):
        lo = Lblock(b, a)
        up = Lblock(a, b)
        assert (lo is None) != (up is None), f"slot ({_lev},{_k}) couples {a},{b}: expected exactly one block"
        C[q] = lo if lo is not None else up.T
    return Dhat, C


def check_no_extra_fill(N: int, nonzero_offdiag: set[tuple[int, int]]) -> None:
    """Every structurally nonzero off-diagonal L^ block (row r, col c) must be a coupling slot."""
    pairs = {(min(a, b), max(a, b)) for (_l, _k, a, b) in coupling_slots(N)}
    pos = position(N)
    for r, c in nonzero_offdiag:
        assert pos[r] > pos[c], "L^ block above the diagonal in permuted order"
        assert (min(r, c), max(r, c)) in pairs, f"unexpected fill block ({r},{c})"
