"""GPU parity of the §8(f) extensions (csrc/btd_ext.cu through the C ABI) against the CPU oracle.

Tolerances as tests/test_gpu_parity.py (BASELINE.json north_star, normwise per system):
fp64 err <= 1e-10, residual <= 1e-12; fp32 err <= 1e-4, residual <= 1e-5.
Mixed precision is held to the fp64 tolerances: iterative refinement reaches the binary64
solution (oracle/refine.py pins the convergence), so the binary64 bar applies to its x.
"""
import numpy as np
import pytest
import torch

import btdgen
import paper_2601_03754_b200 as btd
from paper_2601_03754_b200 import ext, partition as part
from oracle import arrow, banded, dense, metrics, ndchol, o1, refine
from oracle import partition as opart

pytestmark = pytest.mark.gpu

TOL = {torch.float64: dict(L=1e-10, x=1e-10, r=1e-12), torch.float32: dict(L=1e-4, x=1e-4, r=1e-5)}


def _o1(D, E, b):
    """x by O1 (Algorithm 1 + block substitution, binary64)."""
    return o1.seq_solve(*o1.seq_factor(D, E), b)


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


# ------------------------------------------------------------------ f4a mixed precision

MIXED_CASES = [("kalman", 4, 37, 12, 1), ("dd", 3, 64, 16, 2), ("kalman", 1, 1024, 32, 1), ("kalman", 2, 20, 48, 1),
               ("dd", 5, 1, 8, 1), ("kalman", 148, 128, 12, 1)]


@pytest.mark.parametrize("gen,B,N,n,m", MIXED_CASES)
def test_mixed_refinement_reaches_binary64(gen, B, N, n, m):
    dev = _dev()
    prob = btdgen.make(gen, B, N, n, m=m, seed=300 + N)
    D, E, b = prob.D.to(dev), prob.E.to(dev), prob.b.to(dev)
    Dhat, C, x, info, resid = ext.mixed_factor_solve(D, E, b, iters=4, want_resid=True)
    torch.cuda.synchronize()
    assert int(info.abs().sum()) == 0
    xs = x.cpu().numpy()
    for j in sorted({0, B // 2, B - 1}):
        Dj, Ej, bj = prob.D[j].numpy(), prob.E[j].numpy(), prob.b[j].numpy()
        xo = _o1(Dj, Ej, bj)
        assert metrics.err_x(xs[j], xo) <= 1e-10
        r = metrics.residual(Dj, Ej, xs[j], bj)
        assert r <= 1e-12
        # the library's own residual report: at this level the residual is rounding noise of its
        # own evaluation (different summation orders), so only its size is comparable
        assert float(resid[j]) <= 1e-12 and float(resid[j]) <= 4 * r + 1e-15
    # the binary32 factor is the factor of fl32(Psi) (A17 tolerance vs the fp64 oracle)
    j = B - 1
    D32, E32 = prob.D[j].float().double().numpy(), prob.E[j].float().double().numpy()
    Do, Co = ndchol.factor(D32, E32)
    assert metrics.err_L(Dhat[j].cpu().double().numpy(), C[j].cpu().double().numpy(), Do, Co) <= 1e-4


def test_mixed_zero_iterations_is_the_binary32_path():
    """iters = 0 returns exactly the binary32 solution of the core path on fl32(D, E, b), and it
    agrees with the oracle's binary32 refinement start x_0 to binary32 accuracy."""
    dev = _dev()
    prob = btdgen.kalman(6, 50, 12, seed=9)
    D, E, b = prob.D.to(dev), prob.E.to(dev), prob.b.to(dev)
    Dh, C, x, info, res0 = ext.mixed_factor_solve(D, E, b, iters=0, want_resid=True)
    Dh32, C32, x32, _ = btd.factor_solve(D.float(), E.float(), b.float())
    torch.cuda.synchronize()
    assert torch.equal(Dh, Dh32) and torch.equal(C, C32)
    assert torch.equal(x, x32.double())
    x0, _, _ = refine.refine(prob.D[2].numpy(), prob.E[2].numpy(), prob.b[2].numpy(), iters=0)
    assert metrics.err_x(x[2].cpu().numpy(), x0) <= 1e-4
    # a binary32-level residual is far above the evaluation noise: the report matches closely
    for j in range(6):
        r = metrics.residual(prob.D[j].numpy(), prob.E[j].numpy(), x[j].cpu().numpy(), prob.b[j].numpy())
        assert 1e-9 < r < 1e-5 and abs(float(res0[j]) - r) <= 1e-6 * r


def test_mixed_solve_reuses_the_binary32_factor():
    """btd_mixed_solve with the factor of btd_mixed_factor_solve reaches the binary64 solution of a
    NEW right-hand side, and agrees with the factor+solve result for the same b (x_0 comes from the
    solve-only kernel instead of the interlaced one: equal to binary64 rounding, not bitwise)."""
    dev = _dev()
    prob = btdgen.kalman(5, 64, 12, m=2, seed=31)
    D, E, b = prob.D.to(dev), prob.E.to(dev), prob.b.to(dev)
    Dh, C, x1, info, _ = ext.mixed_factor_solve(D, E, b, iters=3)
    x2, _ = ext.mixed_solve(D, E, b, Dh, C, iters=3)
    torch.cuda.synchronize()
    assert int(info.abs().sum()) == 0
    assert float((x1 - x2).abs().max() / x1.abs().max()) <= 1e-13
    b2 = torch.randn_like(b)
    x3, res = ext.mixed_solve(D, E, b2, Dh, C, iters=4, want_resid=True)
    torch.cuda.synchronize()
    for j in (0, 4):
        Dj, Ej = prob.D[j].numpy(), prob.E[j].numpy()
        bj = b2[j].cpu().numpy()
        assert metrics.err_x(x3[j].cpu().numpy(), _o1(Dj, Ej, bj)) <= 1e-10
        assert metrics.residual(Dj, Ej, x3[j].cpu().numpy(), bj) <= 1e-12 and float(res[j]) <= 1e-12


def test_mixed_error_contracts_per_iteration():
    dev = _dev()
    prob = btdgen.kalman(2, 128, 12, seed=21)
    D, E, b = prob.D.to(dev), prob.E.to(dev), prob.b.to(dev)
    xo = _o1(prob.D[0].numpy(), prob.E[0].numpy(), prob.b[0].numpy())
    errs = []
    for it in range(4):
        x = ext.mixed_factor_solve(D, E, b, iters=it)[2]
        errs.append(metrics.err_x(x[0].cpu().numpy(), xo))
    assert errs[0] > 1e-9 and errs[0] < 1e-4
    assert errs[1] < 1e-2 * errs[0] and errs[3] <= 1e-12


# ------------------------------------------------------------------ f4b arrowhead

@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("B,N,n,na,mb", [(3, 33, 8, 4, 2), (2, 1, 3, 2, 1), (1, 128, 12, 16, 1), (4, 17, 2, 1, 3),
                                         (1, 64, 32, 8, 1)])
def test_arrow_parity(dtype, B, N, n, na, mb):
    dev = _dev()
    tol = TOL[dtype]
    prob = btdgen.arrow(B, N, n, na, m=mb, seed=N + na).cast(dtype)
    t = prob.to(dev)
    Dhat, C, Y, LZ, x, xa, info = ext.arrow_factor_solve(t.D, t.E, t.G, t.Z, t.b, t.ba)
    torch.cuda.synchronize()
    assert int(info.abs().sum()) == 0
    for j in sorted({0, B - 1}):
        args = [a[j].double().numpy() for a in (prob.D, prob.E, prob.G, prob.Z)]
        Do, Co, Vo, LZo = arrow.factor(*args)
        xo, xao = arrow.solve(*args, prob.b[j].double().numpy(), prob.ba[j].double().numpy())
        Dg, Cg = Dhat[j].cpu().double().numpy(), C[j].cpu().double().numpy()
        assert metrics.err_L(Dg, Cg, Do, Co) <= tol["L"]
        Vg = Y[j, :, :, :na].cpu().double().numpy()
        assert np.abs(Vg - Vo).max() <= tol["L"] * max(np.abs(Vo).max(), 1.0)
        LZg = LZ[j].cpu().double().numpy()
        assert np.abs(LZg - LZo).max() <= tol["L"] * np.abs(LZo).max() and not np.triu(LZg, 1).any()
        full = np.concatenate([x[j].cpu().double().numpy().ravel(), xa[j].cpu().double().numpy().ravel()])
        ref = np.concatenate([xo.ravel(), xao.ravel()])
        assert np.abs(full - ref).max() <= tol["x"] * np.abs(ref).max()


def test_arrow_indefinite_border_reports_block_N_plus_1():
    dev = _dev()
    prob = btdgen.arrow(3, 9, 4, 3, seed=1)
    prob.Z[1] = -prob.Z[1]
    t = prob.to(dev)
    info = ext.arrow_factor_solve(t.D, t.E, t.G, t.Z, t.b, t.ba)[-1].cpu()
    assert info.tolist() == [0, 10, 0]


# ------------------------------------------------------------------ f4c block banded

@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("B,N,n,w,m", [(2, 13, 4, 3, 1), (3, 12, 3, 2, 2), (1, 256, 8, 4, 1), (2, 5, 2, 7, 1),
                                       (2, 40, 6, 1, 1)])
def test_banded_parity(dtype, B, N, n, w, m):
    dev = _dev()
    tol = TOL[dtype]
    prob = btdgen.banded(B, N, n, w, m=m, seed=N * w).cast(dtype)
    t = prob.to(dev)
    Dhat, C, x, info = ext.banded_factor_solve(t.D, t.A, t.b)
    torch.cuda.synchronize()
    assert int(info.abs().sum()) == 0
    for j in sorted({0, B - 1}):
        Dj, Aj, bj = prob.D[j].double().numpy(), prob.A[j].double().numpy(), prob.b[j].double().numpy()
        xo = banded.solve(Dj, Aj, bj)
        assert metrics.err_x(x[j].cpu().double().numpy(), xo) <= tol["x"]
        Do, Co = banded.factor(Dj, Aj)
        assert metrics.err_L(Dhat[j].cpu().double().numpy(), C[j].cpu().double().numpy(), Do, Co) <= tol["L"]


# ------------------------------------------------------------------ f3 partition

@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("N,n,p,rule", [(100, 8, 2, "equal"), (100, 8, 4, "prop1"), (37, 3, 3, "equal"),
                                        (1024, 32, 8, "equal"), (9, 2, 5, "equal"), (300, 16, 1, "equal")])
def test_partition_parity(dtype, N, n, p, rule):
    dev = _dev()
    tol = TOL[dtype]
    prob = btdgen.kalman(1, N, n, m=2, seed=N + p).cast(dtype)
    D, E, b = prob.D[0].to(dev), prob.E[0].to(dev), prob.b[0].to(dev)
    x, st = part.solve(D, E, b, p, rule=rule)
    torch.cuda.synchronize()
    assert all(int(i.abs().sum()) == 0 for i in st["info"])
    Dn, En, bn = (a[0].double().numpy() for a in (prob.D, prob.E, prob.b))
    xo = _o1(Dn, En, bn)
    xg = x.cpu().double().numpy()
    assert metrics.err_x(xg, xo) <= tol["x"]
    assert metrics.residual(Dn, En, xg, bn) <= tol["r"]
    if p > 1:
        # the pivot system equals Algorithm 2's after its parallel phase
        ref = opart.algorithm2(Dn, En, st["sizes"])
        red = st["reduce"]
        scale = max(np.abs(s).max() for s in ref["S_diag"])
        for q in range(p - 1):
            got = np.tril(red["DS"][q].cpu().double().numpy())
            assert np.abs(got - np.tril(ref["S_diag"][q])).max() <= tol["L"] * scale
        for q in range(p - 2):
            assert np.abs(red["ES"][q].cpu().double().numpy() - ref["S_off"][q]).max() <= tol["L"] * scale
        # and its factor is the nested-dissection factor of that system (O3)
        Do, Co = ndchol.factor(np.stack(ref["S_diag"]), np.stack(ref["S_off"]) if p > 2 else np.zeros((0, n, n)))
        assert metrics.err_L(red["DhatS"].cpu().double().numpy(), red["CS"].cpu().double().numpy(), Do, Co) <= tol["L"]


def test_extension_failure_reporting():
    """A non-SPD block is reported through info by every extension path (LAPACK style)."""
    dev = _dev()
    # mixed: the binary32 pivot of block 5 of system 1 fails
    prob = btdgen.dd(3, 16, 4, seed=2)
    prob.D[1, 4] = -prob.D[1, 4]
    info = ext.mixed_factor_solve(prob.D.to(dev), prob.E.to(dev), prob.b.to(dev), iters=1)[3].cpu()
    assert info[0] == 0 and info[2] == 0 and info[1] != 0
    # banded: a failing super-block pivot
    q = btdgen.banded(2, 12, 2, 3, seed=3)
    q.D[0, 7] = -q.D[0, 7]
    t = q.to(dev)
    info = ext.banded_factor_solve(t.D, t.A, t.b)[3].cpu()
    assert info[0] != 0 and info[1] == 0
    # partition: a failing chunk block shows up in that chunk's info
    p = btdgen.dd(1, 40, 3, seed=4)
    p.D[0, 2] = -p.D[0, 2]
    _, st = part.solve(p.D[0].to(dev), p.E[0].to(dev), p.b[0].to(dev), 3)
    assert sum(int(i.abs().sum()) != 0 for i in st["info"]) >= 1
