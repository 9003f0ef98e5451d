"""P_inf and the level structure, from their plain definitions (oracle; test infrastructure only).

PAPER.md:488-508 (§4.3, Multi-Stage Permutation): the permuted order lists the
odd-indexed blocks first (D_1, D_3, D_5, ...), then the blocks with index
= 2 (mod 4) (D_2, D_6, D_10, ...), then = 4 (mod 8) (D_4, D_12, ...), and so on,
each group ascending. Block i therefore belongs to level 1 + v2(i), where v2 is
the 2-adic valuation, and PAPER.md:569 gives floor(log2 N) + 1 levels.

Indices here are 1-based (as in the paper) unless a name says ``0``.
"""
from __future__ import annotations


def level_of(i: int) -> int:
    """Level of original block i (1-based): 1 + number of factors 2 in i."""
    assert i >= 1
    lev = 1
    while i % 2 == 0:
        i //= 2
        lev += 1
    return lev


def perm(N: int) -> list[int]:
    """perm[new position] = original block index (1-based)."""
    return sorted(range(1, N + 1), key=lambda i: (level_of(i), i))


def position(N: int) -> dict[int, int]:
    """Inverse of ``perm``: original block index -> new position (0-based)."""
    return {orig: pos for pos, orig in enumerate(perm(N))}


def num_levels(N: int) -> int:
    """Number of distinct levels present among 1..N (PAPER.md:569 states floor(log2 N)+1)."""
    return max(level_of(i) for i in range(1, N + 1))


def coupling_slots(N: int) -> list[tuple[int, int, int, int]]:
    """The C-ABI coupling slots, in storage order: (level, k, col_block, row_block).

    Slot (l, k), k = 1 .. floor(N/s) - 1 with s = 2^(l-1), couples original blocks
    k*s and (k+1)*s; it is stored in Psi's lower orientation, i.e. as block
    ((k+1)s, ks). Level-major, k ascending (include/btd.h).
    """
    out = []
    for lev in range(1, num_levels(N) + 1):
        s = 2 ** (lev - 1)
        for k in range(1, N // s):
            out.append((lev, k, k * s, (k + 1) * s))
    return out
