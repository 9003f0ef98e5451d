"""Pins for the oracle extensions of SURVEY.md §8(f) (oracle/refine.py, arrow.py, banded.py,
partition.py): each is tied to something other than itself -- hand-worked instances, dense
brute force, textbook identities (Schur complement, iterative-refinement convergence) and the
closed forms of Proposition 1."""
import numpy as np
import pytest
import torch

import btdgen
from oracle import arrow, banded, dense, metrics, ndchol, partition, refine


def _np(p, j=0):
    return p.D[j].numpy(), p.E[j].numpy(), p.b[j].numpy()


# ------------------------------------------------------------------ mixed-precision refinement (f4)

def test_psi_matvec_matches_dense_assembly():
    p = btdgen.dd(1, 7, 3, m=2, seed=5)
    D, E, _ = _np(p)
    x = np.random.default_rng(0).standard_normal((7, 3, 2))
    y = refine.psi_matvec(D, E, x)
    ref = (dense.assemble(D, E) @ x.reshape(21, 2)).reshape(7, 3, 2)
    assert np.allclose(y, ref, rtol=0, atol=1e-13)
    # the upper triangle of D is never read (A13)
    Dj = D.copy()
    Dj[:, 0, 2] += 100.0
    assert np.array_equal(refine.psi_matvec(Dj, E, x), y)


@pytest.mark.parametrize("gen,N,n", [("kalman", 33, 6), ("dd", 20, 5), ("kalman", 16, 12)])
def test_refine_converges_to_binary64_solution(gen, N, n):
    """Classical IR with a binary32 factor converges to the binary64 solution: the error
    contracts by about kappa * u32 per step (Higham Thm. 12.1/12.2) down to ~u64 * kappa."""
    p = btdgen.GENERATORS[gen](1, N, n, m=2, seed=11)
    D, E, b = _np(p)
    xd = dense.solve(D, E, b)
    hist = []
    x, Dh, C = refine.refine(D, E, b, iters=4, history=hist)
    errs = [metrics.err_x(h, xd) for h in hist]
    kappa = np.linalg.cond(dense.assemble(D, E))
    u32 = 2.0 ** -24
    assert 1e-9 < errs[0] < 50 * kappa * u32          # x_0 is a binary32-accurate solution
    for k in range(1, 3):                            # contraction ~ kappa u32 per step
        assert errs[k] <= max(50 * kappa * u32 * errs[k - 1], 1e-14)
    assert errs[-1] <= 1e-13
    assert metrics.residual(D, E, x, b) <= 1e-14
    assert Dh.dtype == np.float64 and metrics.err_L(Dh, C, *ndchol.factor(D, E)) < 1e-5


def test_refine_zero_iterations_is_the_binary32_solve():
    p = btdgen.dd(1, 12, 4, seed=2)
    D, E, b = _np(p)
    x0, _, _ = refine.refine(D, E, b, iters=0)
    # binary32 dense solve of the binary32-rounded system: agreement to binary32 accuracy only
    A32 = dense.assemble(D, E).astype(np.float32)
    x32 = np.linalg.solve(A32, b.reshape(-1, 1).astype(np.float32)).astype(np.float64).reshape(b.shape)
    assert metrics.err_x(x0, x32) < 1e-5
    assert metrics.err_x(x0, dense.solve(D, E, b)) > 1e-9   # and it is NOT binary64-accurate


# ------------------------------------------------------------------ arrowhead (f4)

def test_arrow_hand_worked_scalar():
    """N=2, n=1, n_a=1: Psi = [[4,2],[2,5]], G = [2, 1], Z = 5. By hand: V = Psi^{-1} G^T =
    [1/2, 0]; Z - G V = 4, L_Z = 2; L^ = [[2,0],[1,2]] (Dhat = [2, 2], C_{1,1} = 1); with
    x = [1,1,1]: b = [8, 8], b_a = 8."""
    D = np.array([[[4.0]], [[5.0]]])
    E = np.array([[[2.0]]])
    G = np.array([[[2.0]], [[1.0]]])
    Z = np.array([[5.0]])
    Dhat, C, V, LZ = arrow.factor(D, E, G, Z)
    assert np.array_equal(Dhat.ravel(), [2.0, 2.0]) and np.array_equal(C.ravel(), [1.0])
    assert np.allclose(V.ravel(), [0.5, 0.0], atol=1e-15) and np.allclose(LZ, [[2.0]], atol=1e-15)
    x, xa = arrow.solve(D, E, G, Z, np.array([[[8.0]], [[8.0]]]), np.array([[8.0]]))
    assert np.allclose(x.ravel(), [1, 1], atol=1e-14) and np.allclose(xa, [[1.0]], atol=1e-14)


def test_arrow_decoupled_border():
    p = btdgen.arrow(1, 9, 3, 4, m=2, seed=3)
    D, E, b = _np(p)
    Z, ba = p.Z[0].numpy(), p.ba[0].numpy()
    G0 = np.zeros_like(p.G[0].numpy())
    Dhat, C, V, LZ = arrow.factor(D, E, G0, Z)
    assert np.allclose(LZ, np.linalg.cholesky(Z), atol=1e-13) and np.abs(V).max() == 0.0
    Do, Co = dense.factor(D, E)
    assert metrics.err_L(Dhat, C, Do, Co) < 1e-14
    x, xa = arrow.solve(D, E, G0, Z, b, ba)
    assert np.allclose(xa, np.linalg.solve(Z, ba), atol=1e-13)
    assert metrics.err_x(x, dense.solve(D, E, b)) < 1e-13


@pytest.mark.parametrize("N,n,na", [(9, 3, 4), (16, 2, 1), (5, 4, 7)])
def test_arrow_schur_identity_and_known_solution(N, n, na):
    p = btdgen.arrow(1, N, n, na, m=2, seed=N + na)
    D, E, b = _np(p)
    G, Z, ba = p.G[0].numpy(), p.Z[0].numpy(), p.ba[0].numpy()
    Dhat, C, V, LZ = arrow.factor(D, E, G, Z)
    S = Z - sum(G[i] @ V[i] for i in range(N))        # Schur complement of Psi in K
    assert np.allclose(LZ @ LZ.T, S, atol=1e-12)
    assert np.allclose(np.triu(LZ, 1), 0.0)
    x, xa = arrow.solve(D, E, G, Z, b, ba)
    assert metrics.err_x(x, p.xstar[0].numpy()) < 1e-12
    assert metrics.err_x(xa, p.xastar[0].numpy()) < 1e-12


# ------------------------------------------------------------------ block-banded (f4)

def test_banded_w1_is_block_tridiagonal():
    q = btdgen.banded(1, 8, 3, 1, seed=4)
    D, A = q.D[0].numpy(), q.A[0].numpy()
    Dp, Ep = banded.reblock(D, A)
    Dl = np.tril(D)
    assert np.array_equal(Dp, Dl + np.swapaxes(np.tril(D, -1), -1, -2))
    assert np.array_equal(Ep, A[0][:7])
    assert np.array_equal(banded.assemble(D, A), dense.assemble(D, A[0][:7]))


@pytest.mark.parametrize("N,n,w", [(12, 2, 3), (10, 3, 4), (9, 1, 2), (7, 2, 7)])
def test_banded_reblock_structure_and_solution(N, n, w):
    q = btdgen.banded(1, N, n, w, m=2, seed=N * w)
    D, A, b = q.D[0].numpy(), q.A[0].numpy(), q.b[0].numpy()
    assert np.array_equal(banded.reblocked_dense(D, A), banded.padded(D, A))
    Dp, Ep = banded.reblock(D, A)
    for Ei in Ep:  # block (p', q') of a super coupling is zero when p' > q' (distance > w)
        for pp in range(w):
            for qq in range(pp):
                assert not Ei[pp * n:(pp + 1) * n, qq * n:(qq + 1) * n].any()
    x = banded.solve(D, A, b)
    assert metrics.err_x(x, q.xstar[0].numpy()) < 1e-12
    Dh, C = banded.factor(D, A)
    assert metrics.reconstruction(Dp, Ep, Dh, C) < 1e-14


# ------------------------------------------------------------------ partition / Algorithm 2 (f3)

def test_prop1_sizes():
    """Proposition 1: N_1*/N_k* = 19/7, and the rounding rule on a hand-worked case:
    N = 100, p = 4: N_k* = 679/40 = 16.975; N_k = 16 -> N_1 = 49, max cost 113.33;
    N_k = 17 -> N_1 = 46, max cost 106.67 (kept)."""
    for N, p in [(100, 4), (1000, 8), (57, 3)]:
        n1 = (19 * N - 19 * p + 19) / (7 * p + 12)
        nk = (7 * N - 7 * p + 7) / (7 * p + 12)
        assert abs(n1 / nk - 19 / 7) < 1e-12
        assert abs(n1 + (p - 1) * nk - (N - (p - 1))) < 1e-9
        s = partition.chunk_sizes_prop1(N, p)
        assert sum(s) + p - 1 == N and len(s) == p
    assert partition.chunk_sizes_prop1(100, 4) == [46, 17, 17, 17]
    assert partition.chunk_sizes_prop1(9, 1) == [9]


@pytest.mark.parametrize("sizes,n", [([3, 2, 2], 2), ([1, 1], 3), ([2, 3, 1, 2], 1), ([4, 1, 3], 3),
                                     ([5], 2), ([2, 2, 2, 2, 2], 2)])
def test_algorithm2_equals_dense_factor(sizes, n):
    N = sum(sizes) + len(sizes) - 1
    p = btdgen.kalman(1, N, n, seed=N)
    D, E, _ = _np(p)
    res = partition.algorithm2(D, E, sizes)
    Lf = partition.factor_dense(D, E, sizes)
    pos = {orig: new for new, orig in enumerate(partition.perm_p(sizes))}
    scale = np.abs(Lf).max()
    for (r, c), blk in res["L"].items():
        ref = Lf[pos[r] * n:(pos[r] + 1) * n, pos[c] * n:(pos[c] + 1) * n]
        assert np.abs(blk - ref).max() <= 1e-12 * scale, (r, c)
    # every nonzero block of the dense factor is produced by Algorithm 2 (fill pattern)
    for r in range(1, N + 1):
        for c in range(1, N + 1):
            if pos[r] >= pos[c]:
                ref = Lf[pos[r] * n:(pos[r] + 1) * n, pos[c] * n:(pos[c] + 1) * n]
                if np.abs(ref).max() > 1e-13 * scale:
                    assert (r, c) in res["L"], (r, c)


@pytest.mark.parametrize("sizes,n", [([3, 2, 2], 2), ([2, 3, 1, 2], 3), ([1, 1], 2)])
def test_algorithm2_pivot_system_is_schur_complement(sizes, n):
    N = sum(sizes) + len(sizes) - 1
    p = btdgen.dd(1, N, n, seed=7)
    D, E, _ = _np(p)
    res = partition.algorithm2(D, E, sizes)
    A = dense.assemble(D, E)
    piv = res["pivots"]
    inner = [i for c in res["chunks"] for i in c]
    idx = lambda blocks: np.concatenate([np.arange((i - 1) * n, i * n) for i in blocks])
    P, I = idx(piv), idx(inner)
    S = A[np.ix_(P, P)] - A[np.ix_(P, I)] @ np.linalg.solve(A[np.ix_(I, I)], A[np.ix_(I, P)])
    q = len(piv)
    for k in range(q):
        assert np.allclose(res["S_diag"][k], S[k * n:(k + 1) * n, k * n:(k + 1) * n], atol=1e-12)
    for k in range(q - 1):
        assert np.allclose(res["S_off"][k], S[(k + 1) * n:(k + 2) * n, k * n:(k + 1) * n], atol=1e-12)
    for k in range(q):  # the reduced system is block tridiagonal
        for j in range(k + 2, q):
            assert np.abs(S[j * n:(j + 1) * n, k * n:(k + 1) * n]).max() < 1e-12


def test_algorithm2_single_chunk_is_algorithm1():
    p = btdgen.dd(1, 6, 3, seed=1)
    D, E, _ = _np(p)
    res = partition.algorithm2(D, E, [6])
    Lf = np.linalg.cholesky(dense.assemble(D, E))
    for i in range(1, 7):
        assert np.allclose(res["L"][(i, i)], Lf[(i - 1) * 3:i * 3, (i - 1) * 3:i * 3], atol=1e-13)
