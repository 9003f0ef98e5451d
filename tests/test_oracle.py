"""Pins for the CPU oracle (oracle/): each check ties it to something other than itself.

Sources of truth used here (SURVEY.md §8(c) "What pins each part"):
  * SPEC.md worked examples for the block operations and the permutation;
  * the hand-worked N=4 instance (tests/golden/nd_n4_scalar.json) and its exact
    Kronecker lift (uniqueness of the Cholesky factor);
  * the closed form for Psi = T_N (x) M, N = 2^k - 1;
  * special cases: Psi = I, E = 0, N = 1, and n = 1 against the textbook Thomas algorithm;
  * brute force: numpy's dense Cholesky / dense solve on the assembled matrix;
  * invariants: P Psi P^T = L^ L^^T, level count floor(log2 N)+1.
"""
import math

import numpy as np
import pytest
import torch

import btdgen
from oracle import dense, layout, metrics, ndchol, o1
from oracle.perm import coupling_slots, level_of, num_levels, perm, position


# ---------------------------------------------------------------- block operations

def test_spec_block_ops(golden):
    g = golden("spec_block_ops.json")
    assert np.array_equal(o1.potrf(g["potrf"]["in"]), np.array(g["potrf"]["out"], float))
    with pytest.raises(o1.NotPositiveDefinite) as ei:
        o1.potrf(g["potrf_fail"]["in"])
    assert ei.value.index == g["potrf_fail"]["pivot"]
    t = g["trsm_right"]
    assert np.array_equal(o1.trsm_right(t["e"], t["l"]), np.array(t["out"], float))
    t = g["trsm_left"]
    assert np.array_equal(o1.trsm_left(t["l"], t["e"]), np.array(t["out"], float))
    t = g["syrk_down"]
    assert np.array_equal(o1.syrk_down(t["d"], t["e"]), np.array(t["out"], float))
    t = g["gemm_neg"]
    assert np.array_equal(o1.gemm_neg(t["a"], t["b"]), np.array(t["out"], float))


def test_block_ops_identity_and_roundtrip():
    rng = np.random.default_rng(1)
    for n in (1, 3, 8, 16):
        assert np.array_equal(o1.potrf(np.eye(n)), np.eye(n))
        A = rng.standard_normal((n, n))
        S = A @ A.T + n * np.eye(n)
        L = o1.potrf(S)
        assert np.allclose(L, np.linalg.cholesky(S), rtol=0, atol=1e-12 * np.abs(S).max())
        e = rng.standard_normal((5, n))
        assert np.allclose(o1.trsm_right(e, L) @ L.T, e, atol=1e-12)
        f = rng.standard_normal((n, 4))
        assert np.allclose(L @ o1.trsm_left(L, f), f, atol=1e-12)
        assert np.allclose(o1.syrk_down(S, e.T), S - e.T @ e, atol=1e-12)
        assert np.allclose(o1.syrk_down(S, e, trans=True), S - e.T @ e, atol=1e-12)


# ---------------------------------------------------------------- permutation and counts

def test_perm_spec_examples(golden):
    g = golden("spec_block_ops.json")["perm"]
    assert perm(1) == g["1"]
    assert perm(8) == g["8"]
    assert perm(20)[:10] == g["20_prefix10"]
    assert num_levels(20) == golden("spec_block_ops.json")["levels"]["20"]


def test_perm_is_recursive_odd_even():
    """Independent recursive construction: odd positions first, recurse on the rest."""
    def rec(seq):
        if not seq:
            return []
        return seq[0::2] + rec(seq[1::2])

    for N in range(1, 300):
        assert perm(N) == rec(list(range(1, N + 1)))


def test_level_count_closed_form():
    for N in range(1, 4097):
        assert num_levels(N) == math.floor(math.log2(N)) + 1


@pytest.mark.parametrize("N,L,nC,I", [(8, 4, 11, 4), (64, 7, 120, 57), (128, 8, 247, 120),
                                      (256, 9, 502, 247), (1024, 11, 2036, 1013), (4096, 13, 8178, 4083)])
def test_config_counts(N, L, nC, I):
    """SURVEY.md §8(a) per-config counts: levels / coupling blocks / interior eliminations."""
    assert num_levels(N) == L
    slots = coupling_slots(N)
    assert len(slots) == nC
    # interior eliminations = columns with both neighbours = fill blocks = slots above level 1
    assert sum(1 for (lev, *_r) in slots if lev > 1) == I
    assert nC == (N - 1) + I


def test_fill_pattern_matches_slots():
    """O3 discovers fill symbolically; every fill block must be a declared coupling slot and the
    elimination-tree height must be floor(log2 N)+1."""
    for N in list(range(1, 40)) + [63, 64, 65, 100, 127, 128]:
        D = np.tile(np.eye(1) * 4.0, (N, 1, 1))
        E = np.full((max(N - 1, 0), 1, 1), 1.0)
        L, order = ndchol.factor_blocks(D, E)
        off = {k for k in L if k[0] != k[1]}
        layout.check_no_extra_fill(N, off)
        assert len(off) == len(coupling_slots(N))
        pos = position(N)
        parent = {c: min((r for (r, cc) in off if cc == c), key=lambda r: pos[r], default=None)
                  for c in order}
        height = {}
        for c in order:  # children precede parents in elimination order
            height.setdefault(c, 1)
            p = parent[c]
            if p is not None:
                height[p] = max(height.get(p, 1), height[c] + 1)
        assert max(height.values()) == math.floor(math.log2(N)) + 1


# ---------------------------------------------------------------- the hand-worked instance

def _golden_n4(golden):
    g = golden("nd_n4_scalar.json")
    D = np.array(g["D"]).reshape(4, 1, 1)
    E = np.array(g["E"]).reshape(3, 1, 1)
    b = np.array(g["b"]).reshape(4, 1, 1)
    return g, D, E, b


@pytest.mark.parametrize("which", ["dense", "ndchol"])
def test_golden_n4_exact(golden, which):
    g, D, E, b = _golden_n4(golden)
    assert perm(4) == g["perm"]
    Dhat, C = (dense.factor if which == "dense" else ndchol.factor)(D, E)
    assert np.array_equal(Dhat.reshape(-1), np.array(g["Dhat"]))
    slots = coupling_slots(4)
    assert [(lv, k) for (lv, k, _a, _b) in slots] == [(s[0], s[1]) for s in g["C_slots"]]
    assert np.array_equal(C.reshape(-1), np.array([s[2] for s in g["C_slots"]]))
    if which == "dense":
        assert np.array_equal(dense.factor_dense(D, E), np.array(g["Lhat_permuted"], float))
        x = dense.solve(D, E, b)
        assert np.allclose(x.reshape(-1), g["x"], rtol=0, atol=1e-15)
    else:
        _, _, x = ndchol.factor_solve(D, E, b)
        assert np.array_equal(x.reshape(-1), np.array(g["x"]))


@pytest.mark.parametrize("which", ["dense", "ndchol"])
def test_golden_n4_kronecker_lift(golden, which):
    """D_i = d_i M, E_i = e_i M with M = R R^T => L^ = L^_scalar (x) R (uniqueness).
    Expected: Dhat_i = 2R, right couplings R, left coupling (k even) stored as R^T, fill -R/2."""
    g, D1, E1, _ = _golden_n4(golden)
    R = np.array([[2.0, 0.0], [1.0, 2.0]])
    M = R @ R.T
    D = D1 * M
    E = E1 * M
    Dhat, C = (dense.factor if which == "dense" else ndchol.factor)(D, E)
    for i in range(4):
        assert np.array_equal(Dhat[i], 2 * R)
    exp = {(1, 1): R, (1, 2): R.T, (1, 3): R, (2, 1): -0.5 * R}
    for q, (lv, k, _a, _b) in enumerate(coupling_slots(4)):
        assert np.array_equal(C[q], exp[(lv, k)]), (lv, k)
    b = np.array([36, 42, 60, 70, 48, 56, 43.5, 50.75]).reshape(4, 2, 1)
    x = ndchol.factor_solve(D, E, b)[2] if which == "ndchol" else dense.solve(D, E, b)
    assert np.allclose(x, 1.0, rtol=0, atol=1e-14)
    xs = o1.seq_solve(*o1.seq_factor(D, E), b)
    assert np.allclose(xs, 1.0, rtol=0, atol=1e-14)


# ---------------------------------------------------------------- closed form T (x) M

@pytest.mark.parametrize("k", range(1, 7))
@pytest.mark.parametrize("n", [1, 3, 8])
def test_closed_form_laplacian(k, n):
    """Psi = T_N (x) M, N = 2^k - 1: at level l, Dhat = 2^{(2-l)/2} R, right-trsm'd coupling
    -2^{-l/2} R, left-trsm'd stored coupling -2^{-l/2} R^T (self-similar T/2)."""
    N = 2 ** k - 1
    rng = np.random.default_rng(k * 10 + n)
    R = np.tril(rng.uniform(-1, 1, (n, n)))
    np.fill_diagonal(R, rng.uniform(1, 2, n))
    prob = btdgen.lap(1, N, torch.from_numpy(R))
    D, E = prob.D[0].numpy(), prob.E[0].numpy()
    Dhat, C = ndchol.factor(D, E)
    for i in range(1, N + 1):
        lv = level_of(i)
        assert np.allclose(Dhat[i - 1], 2 ** ((2 - lv) / 2) * R, rtol=0, atol=1e-12)
    for q, (lv, kk, _a, _b) in enumerate(coupling_slots(N)):
        expect = -(2 ** (-lv / 2)) * (R if kk % 2 == 1 else R.T)
        assert np.allclose(C[q], expect, rtol=0, atol=1e-12), (lv, kk)
    if N * n <= 256:
        Dd, Cd = dense.factor(D, E)
        assert np.allclose(Dd, Dhat, atol=1e-13) and np.allclose(Cd, C, atol=1e-13)


# ---------------------------------------------------------------- special cases

@pytest.mark.parametrize("N", [1, 2, 3, 8, 13])
def test_identity(N):
    n = 3
    D = np.tile(np.eye(n), (N, 1, 1))
    E = np.zeros((N - 1, n, n))
    b = np.random.default_rng(N).standard_normal((N, n, 2))
    Dhat, C, x = ndchol.factor_solve(D, E, b)
    assert np.array_equal(Dhat, D) and not np.any(C)
    assert np.array_equal(x, b)
    assert np.array_equal(o1.seq_solve(*o1.seq_factor(D, E), b), b)


def test_zero_coupling():
    rng = np.random.default_rng(5)
    N, n = 9, 4
    A = rng.standard_normal((N, n, n))
    D = A @ np.swapaxes(A, 1, 2) + n * np.eye(n)
    E = np.zeros((N - 1, n, n))
    b = rng.standard_normal((N, n, 1))
    Dhat, C, x = ndchol.factor_solve(D, E, b)
    assert np.allclose(Dhat, np.linalg.cholesky(D), atol=1e-13)
    assert not np.any(C)
    assert np.allclose(x, np.linalg.solve(D, b), atol=1e-13)


def test_single_block():
    D = np.array([[[4.0, 2.0], [2.0, 5.0]]])
    E = np.zeros((0, 2, 2))
    Dhat, C = ndchol.factor(D, E)
    assert np.array_equal(Dhat[0], [[2, 0], [1, 2]]) and C.shape[0] == 0


def _thomas(a, d, c, r):
    """Textbook Thomas algorithm for a scalar tridiagonal system (sub a, diag d, super c)."""
    n = len(d)
    cp, dp = np.zeros(n), np.zeros(n)
    cp[0] = c[0] / d[0] if n > 1 else 0.0
    dp[0] = r[0] / d[0]
    for i in range(1, n):
        den = d[i] - a[i - 1] * cp[i - 1]
        cp[i] = c[i] / den if i < n - 1 else 0.0
        dp[i] = (r[i] - a[i - 1] * dp[i - 1]) / den
    x = np.zeros(n)
    x[-1] = dp[-1]
    for i in range(n - 2, -1, -1):
        x[i] = dp[i] - cp[i] * x[i + 1]
    return x


@pytest.mark.parametrize("N", [1, 2, 3, 7, 16, 33, 100])
def test_scalar_against_thomas(N):
    prob = btdgen.dd(1, N, 1, seed=11)
    D, E, b = prob.D[0].numpy(), prob.E[0].numpy(), prob.b[0].numpy()
    e = E.reshape(-1)
    xt = _thomas(e, D.reshape(-1), e, b.reshape(-1))
    assert np.allclose(ndchol.factor_solve(D, E, b)[2].reshape(-1), xt, rtol=1e-13, atol=1e-13)
    assert np.allclose(o1.seq_solve(*o1.seq_factor(D, E), b).reshape(-1), xt, rtol=1e-13, atol=1e-13)


# ---------------------------------------------------------------- brute force and invariants

GRID_N = [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33]
GRID_n = [1, 2, 3, 5, 8]


@pytest.mark.parametrize("kind", ["dd", "kalman"])
@pytest.mark.parametrize("N", GRID_N)
def test_ndchol_vs_dense(kind, N):
    for n in GRID_n:
        if N * n > 200:
            continue
        p = btdgen.make(kind, 1, N, n, m=2, seed=3)
        D, E, b = p.D[0].numpy(), p.E[0].numpy(), p.b[0].numpy()
        Dd, Cd = dense.factor(D, E)
        Dh, Ch, x = ndchol.factor_solve(D, E, b)
        assert metrics.err_L(Dh, Ch, Dd, Cd) < 1e-13
        xd = dense.solve(D, E, b)
        assert metrics.err_x(x, xd) < 1e-12
        assert metrics.reconstruction(D, E, Dh, Ch) < 1e-14
        assert metrics.residual(D, E, x, b) < 1e-14


@pytest.mark.parametrize("kind", ["dd", "kalman"])
def test_o1_against_dense(kind):
    for N, n in [(1, 4), (2, 3), (5, 2), (8, 2), (13, 3), (40, 5)]:
        p = btdgen.make(kind, 1, N, n, m=3, seed=4)
        D, E, b = p.D[0].numpy(), p.E[0].numpy(), p.b[0].numpy()
        Dh, Eh = o1.seq_factor(D, E)
        # Alg. 1's natural-order factor is chol(Psi) itself (unique factor)
        L = np.linalg.cholesky(dense.assemble(D, E))
        for i in range(N):
            assert np.allclose(Dh[i], L[i * n:(i + 1) * n, i * n:(i + 1) * n], atol=1e-12)
        for i in range(N - 1):
            assert np.allclose(Eh[i], L[(i + 1) * n:(i + 2) * n, i * n:(i + 1) * n], atol=1e-12)
        x = o1.seq_solve(Dh, Eh, b)
        assert metrics.err_x(x, dense.solve(D, E, b)) < 1e-12
        assert metrics.err_x(x, p.xstar[0].numpy()) < 1e-10


def test_o1_batch_matches_single():
    p = btdgen.dd(6, 10, 3, m=2, seed=9)
    x, info = o1.seq_batch(p.D.numpy(), p.E.numpy(), p.b.numpy(), nthreads=3)
    assert not info.any()
    for j in range(6):
        xs = o1.seq_solve(*o1.seq_factor(p.D[j].numpy(), p.E[j].numpy()), p.b[j].numpy())
        assert np.array_equal(x[j], xs)


def test_o1_reports_failing_block():
    p = btdgen.dd(1, 6, 2, seed=1)
    D = p.D[0].numpy().copy()
    D[3] = -np.eye(2)
    with pytest.raises(o1.NotPositiveDefinite) as ei:
        o1.seq_factor(D, p.E[0].numpy())
    assert ei.value.index == 4


def test_ndchol_reports_failing_block():
    p = btdgen.dd(1, 8, 2, seed=1)
    D = p.D[0].numpy().copy()
    D[5] = -np.eye(2)  # block 6, eliminated at level 2
    with pytest.raises(ndchol.NotPositiveDefinite) as ei:
        ndchol.factor(D, p.E[0].numpy())
    assert ei.value.block == 6


def test_reconstruction_detects_wrong_orientation():
    """The layout pin must notice a transposed coupling (a plausible indexing mistake)."""
    p = btdgen.dd(1, 9, 3, seed=2)
    D, E = p.D[0].numpy(), p.E[0].numpy()
    Dh, C = ndchol.factor(D, E)
    assert metrics.reconstruction(D, E, Dh, C) < 1e-14
    Cbad = C.copy()
    Cbad[1] = Cbad[1].T
    assert metrics.reconstruction(D, E, Dh, Cbad) > 1e-3


def test_larger_ndchol_reconstruction():
    for kind, N, n in [("dd", 100, 6), ("kalman", 128, 12), ("dd", 257, 4)]:
        p = btdgen.make(kind, 1, N, n, seed=7)
        D, E, b = p.D[0].numpy(), p.E[0].numpy(), p.b[0].numpy()
        Dh, C, x = ndchol.factor_solve(D, E, b)
        assert metrics.reconstruction(D, E, Dh, C) < 1e-14
        xs = o1.seq_solve(*o1.seq_factor(D, E), b)
        assert metrics.err_x(x, xs) < 1e-12
        assert metrics.err_x(x, p.xstar[0].numpy()) < 1e-10


# ---------------------------------------------------------------- generators

def test_generators_deterministic_and_shard_invariant():
    a = btdgen.dd(8, 16, 4, seed=5)
    b = btdgen.dd(3, 16, 4, seed=5, first_system=5)
    assert torch.equal(a.D[5:], b.D) and torch.equal(a.E[5:], b.E) and torch.equal(a.b[5:], b.b)
    k1 = btdgen.kalman(4, 8, 6, seed=2)
    k2 = btdgen.kalman(2, 8, 6, seed=2, first_system=2)
    assert torch.allclose(k1.D[2:], k2.D, atol=1e-12)


def test_dd_is_spd_with_margin():
    p = btdgen.dd(4, 9, 6, seed=1)
    for j in range(4):
        A = dense.assemble(p.D[j].numpy(), p.E[j].numpy())
        assert np.linalg.eigvalsh(A).min() >= 1.0 - 1e-12  # Gershgorin with shift 3n+1 (A18)


def test_kalman_is_spd():
    p = btdgen.kalman(3, 16, 5, seed=1)
    for j in range(3):
        A = dense.assemble(p.D[j].numpy(), p.E[j].numpy())
        w = np.linalg.eigvalsh(A)
        assert w.min() > 0 and w.max() / w.min() < 1e4


# ---------------------------------------------------------------- error measures (oracle/metrics.py)
# Negative pins: each measure is fed a known error and must return the value computed here by hand
# from its definition, so a dropped term, a wrong norm or a broadcasting slip
# fails. The exact factor is the hand-worked N=4 instance (tests/golden/nd_n4_scalar.json):
# Dhat = [2,2,2,2], C = [1,1,1,-0.5] (slots (1,1),(1,2),(1,3),(2,1)), x = [1,1,1,1].

def _golden_factor(golden):
    g = golden("nd_n4_scalar.json")
    Dh = np.array(g["Dhat"], float).reshape(4, 1, 1)
    C = np.array([s[2] for s in g["C_slots"]], float).reshape(4, 1, 1)
    return g, Dh, C


def test_err_L_exact_on_golden_perturbations(golden):
    _, Dh, C = _golden_factor(golden)
    assert metrics.err_L(Dh, C, Dh, C) == 0.0
    # one perturbed element of D^ (block 3): |0.25| / max|L^_o| = 0.25 / 2
    Dp = Dh.copy()
    Dp[2, 0, 0] += 0.25
    assert metrics.err_L(Dp, C, Dh, C) == 0.125
    # one perturbed element of the level-2 fill slot C(2,1): -0.5 -> -0.25, again 0.25 / 2
    Cp = C.copy()
    Cp[3, 0, 0] = -0.25
    assert metrics.err_L(Dh, Cp, Dh, C) == 0.125
    # both at once: the max, not the sum, of the two block-set errors
    assert metrics.err_L(Dp, Cp, Dh, C) == 0.125


def test_err_L_denominator_includes_couplings():
    """max|L^_o| runs over D^ AND every coupling block: with max|C_o| = 4 > max|D^_o| = 1 an error
    of 1 in D^ reads 1/4 (a denominator over D^ alone would give 1)."""
    Dh = np.ones((2, 1, 1))
    C = np.array([4.0]).reshape(1, 1, 1)
    Dp = Dh.copy()
    Dp[1, 0, 0] = 2.0
    assert metrics.err_L(Dp, C, Dh, C) == 0.25
    Cp = C + 1.0  # error only in C: 1/4 (a numerator over D^ alone would give 0)
    assert metrics.err_L(Dh, Cp, Dh, C) == 0.25


def test_err_x_exact():
    xo = np.array([1.0, -4.0, 2.0, 0.5]).reshape(4, 1, 1)
    assert metrics.err_x(xo, xo) == 0.0
    assert metrics.err_x(2 * xo, xo) == 1.0                     # scaled x: max|x_o| / max|x_o|
    xp = xo.copy()
    xp[1] += -1.0                                               # |dx| = 1 at the largest entry
    assert metrics.err_x(xp, xo) == 0.25                        # / max|x_o| = 4 (not max|x| = 5)
    xp = xo.copy()
    xp[2] += 0.5
    assert metrics.err_x(xp, xo) == 0.125                       # inf-norm, not 2-norm
    xm = np.stack([xo[..., 0], 3 * xo[..., 0]], -1)             # m = 2 right-hand sides
    assert metrics.err_x(xm + np.array([0.0, 6.0]), xm) == 0.5  # 6 / max|x_o| = 6 / 12


def test_residual_exact_on_golden(golden):
    g = golden("nd_n4_scalar.json")
    D = np.array(g["D"]).reshape(4, 1, 1)
    E = np.array(g["E"]).reshape(3, 1, 1)
    b = np.array(g["b"]).reshape(4, 1, 1)
    x = np.ones((4, 1, 1))
    assert metrics.residual(D, E, x, b) == 0.0
    # x off by one in block 3: r = Psi e_3 = column 3 of Psi = [0, E_2, D_3, E_3] = [0, 2, 4, 2]
    xp = x.copy()
    xp[2] += 1.0
    exp = math.sqrt(0 + 4 + 16 + 4) / math.sqrt(6 ** 2 + 10 ** 2 + 8 ** 2 + 7.25 ** 2)
    assert metrics.residual(D, E, xp, b) == pytest.approx(exp, rel=1e-15)
    # scaled x: r = Psi (2x) - b = b, so the relative residual is exactly 1
    assert metrics.residual(D, E, 2 * x, b) == pytest.approx(1.0, rel=1e-15)


def test_residual_orientation_and_lower_triangle():
    """n = 2, N = 2 by hand: E_1 = [[1,2],[0,1]] is block (2,1), block (1,2) is E_1^T; only the lower
    triangle of D_i is read (garbage above the diagonal must not change the result).
    Psi = [[4,0,1,0],[0,4,2,1],[1,2,4,0],[0,1,0,4]]; Psi e_1 = [4,0,1,0], Psi e_2 = [0,4,2,1]."""
    D = np.array([[[4.0, 99.0], [0.0, 4.0]], [[4.0, -7.0], [0.0, 4.0]]])
    E = np.array([[[1.0, 2.0], [0.0, 1.0]]])
    e1 = np.array([1.0, 0, 0, 0]).reshape(2, 2, 1)
    e2 = np.array([0, 1.0, 0, 0]).reshape(2, 2, 1)
    assert metrics.residual(D, E, e1, np.array([4.0, 0, 1, 0]).reshape(2, 2, 1)) == 0.0
    assert metrics.residual(D, E, e2, np.array([0, 4.0, 2, 1]).reshape(2, 2, 1)) == 0.0
    # the transposed coupling would give Psi e_1 = [4,0,1,2]: relative residual 2 / |[4,0,1,2]|
    bt = np.array([4.0, 0, 1, 2]).reshape(2, 2, 1)
    assert metrics.residual(D, E, e1, bt) == pytest.approx(2.0 / math.sqrt(21.0), rel=1e-15)
