"""CPU oracle for the nested-dissection block-tridiagonal Cholesky (arXiv 2601.03754).

TEST INFRASTRUCTURE ONLY. The product package (``paper_2601_03754_b200``) never
imports, links or executes anything in this directory; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs do. The oracle shares no code with the CUDA path; the only
common module is the input generator package ``btdgen`` (no method arithmetic).

Contents:

* ``perm``   -- P_inf, levels and coupling-slot layout, from their plain definitions.
* ``o1``     -- O1: Algorithm 1 sequential block Cholesky + block substitution (C, fp64).
* ``dense``  -- O2: dense Cholesky of the assembled P Psi P^T and dense solve (numpy).
* ``ndchol`` -- O3: generic block-sparse right-looking Cholesky in the order P_inf,
                discovering fill symbolically (numpy); knows nothing about levels.
* ``layout`` -- mapping of a factor L^ onto the C-ABI (Dhat, C) layout (include/btd.h).
* ``metrics``-- the error measures of SURVEY.md §8(c) A16.
* ``refine`` -- §8(f) f4: classical iterative refinement on a binary32 factorization.
* ``arrow``  -- §8(f) f4: block-tridiagonal-arrow systems, dense definitions.
* ``banded`` -- §8(f) f4: block-banded systems, dense definitions + reblocking.
* ``partition`` -- §8(f) f3: partition permutation, Proposition 1 and Algorithm 2 line by line.

Parity status per function is listed in DESIGN.md ("Oracle pins").
"""
