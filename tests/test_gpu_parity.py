"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star; SURVEY.md §8(c) A16 normwise per system):
  fp64: err_L <= 1e-10, err_x <= 1e-10, residual <= 1e-12
  fp32: err_L <= 1e-4,  err_x <= 1e-4,  residual <= 1e-5
fp32 results are compared with the fp64 oracle run on the fp32-rounded inputs (A17).
"""
import numpy as np
import pytest
import torch

import btdgen
import paper_2601_03754_b200 as btd
from oracle import metrics, ndchol, o1

pytestmark = pytest.mark.gpu

TOL = {torch.float64: dict(L=1e-10, x=1e-10, r=1e-12), torch.float32: dict(L=1e-4, x=1e-4, r=1e-5)}


def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _run(prob, dtype, variant, op="factor_solve"):
    dev = _dev()
    p = prob.cast(dtype)
    D, E, b = p.D.to(dev), p.E.to(dev), p.b.to(dev)
    if op == "factor_solve":
        Dhat, C, x, info = btd.factor_solve(D, E, b, variant=variant)
    else:
        Dhat, C, info = btd.factor(D, E, variant=variant)
        x = btd.solve(Dhat, C, b, variant=variant)
    torch.cuda.synchronize()
    return p, Dhat.cpu(), C.cpu(), x.cpu(), info.cpu()


def _check(prob_cast, Dhat, C, x, info, dtype, systems=None, check_L=True):
    tol = TOL[dtype]
    ref = prob_cast.f64()
    assert int(info.abs().sum()) == 0, info
    systems = range(ref.batch) if systems is None else systems
    worst = dict(L=0.0, x=0.0, r=0.0)
    for j in systems:
        D, E, b = ref.D[j].numpy(), ref.E[j].numpy(), ref.b[j].numpy()
        Do, Co, xo = ndchol.factor_solve(D, E, b)
        xg = x[j].double().numpy()
        if check_L:
            worst["L"] = max(worst["L"], metrics.err_L(Dhat[j].double().numpy(), C[j].double().numpy(), Do, Co))
        worst["x"] = max(worst["x"], metrics.err_x(xg, xo))
        worst["r"] = max(worst["r"], metrics.residual(D, E, xg, b))
    assert worst["L"] <= tol["L"] and worst["x"] <= tol["x"] and worst["r"] <= tol["r"], worst
    # strict upper triangle of every D^ block is exactly zero (include/btd.h layout)
    assert torch.all(torch.triu(Dhat, 1) == 0)
    return worst


SMALL_N = [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33]


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide", "atomic"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 12, 16])
def test_small_grid(variant, dtype, n):
    for N in SMALL_N:
        for kind in ("dd", "kalman"):
            prob = btdgen.make(kind, 3, N, n, m=1, seed=100 + N)
            _check(*_run(prob, dtype, variant), dtype)


@pytest.mark.parametrize("dtype,n", [(torch.float32, 12), (torch.float32, 9), (torch.float64, 8)])
def test_fused_r_horizons(dtype, n):
    """FUSED-R at horizons that switch its shared-memory backward cache between levels >= 3,
    >= 4 and off, split level 1 into 1-4 rounds of 32 column ops and stage D in one or two
    commit groups (N = 37 .. 255; n = 9 runs the padded instantiation, n = 12 / 8 the exact one)."""
    for N in (37, 63, 64, 65, 100, 128, 129, 200, 255):
        prob = btdgen.make("kalman", 2, N, n, m=1, seed=300 + N)
        _check(*_run(prob, dtype, "fused"), dtype)


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide", "atomic"])
@pytest.mark.parametrize("n", [6, 24, 32])
def test_larger_blocks_and_padding(variant, n):
    for dtype in (torch.float64, torch.float32):
        for N in (7, 20, 64):
            if variant == "fused":
                try:
                    btd.Plan(N, n, 2, 1, dtype, variant="fused")
                except btd.BtdError:
                    continue  # does not fit one SM's shared memory; AUTO would pick "level"
            prob = btdgen.kalman(2, N, n, seed=7 + n)
            _check(*_run(prob, dtype, variant), dtype)


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide", "atomic"])
@pytest.mark.parametrize("m", [2, 3, 4])
def test_multiple_rhs(variant, m):
    for dtype in (torch.float64, torch.float32):
        prob = btdgen.dd(3, 13, 3, m=m, seed=5)
        _check(*_run(prob, dtype, variant), dtype)
        prob = btdgen.dd(2, 40, 12, m=m, seed=6)
        _check(*_run(prob, dtype, variant), dtype)


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide", "atomic"])
def test_separate_factor_and_solve(variant):
    for dtype in (torch.float64, torch.float32):
        prob = btdgen.kalman(5, 45, 12, m=2, seed=9)
        _check(*_run(prob, dtype, variant, op="factor+solve"), dtype)


def _golden_n4(golden, lift):
    g = golden("nd_n4_scalar.json")
    D = torch.tensor(g["D"], dtype=torch.float64).reshape(1, 4, 1, 1)
    E = torch.tensor(g["E"], dtype=torch.float64).reshape(1, 3, 1, 1)
    b = torch.tensor(g["b"], dtype=torch.float64).reshape(1, 4, 1, 1)
    if lift:
        R = torch.tensor([[2.0, 0.0], [1.0, 2.0]], dtype=torch.float64)
        M = R @ R.T
        D, E = D * M, E * M
        b = btdgen.block_tridiag_matvec(D, E, torch.ones(1, 4, 2, 1, dtype=torch.float64))
    return g, btdgen.Problem(D, E, b, None)


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide", "atomic"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("lift", [False, True])
def test_golden_n4_bitwise(golden, variant, dtype, lift):
    """The hand-worked instance is exactly representable: zero tolerance."""
    g, prob = _golden_n4(golden, lift)
    p, Dhat, C, x, info = _run(prob, dtype, variant)
    assert int(info[0]) == 0
    if not lift:
        assert Dhat.reshape(-1).tolist() == g["Dhat"]
        assert C.reshape(-1).tolist() == [s[2] for s in g["C_slots"]]
        assert x.reshape(-1).tolist() == g["x"]
    else:
        R = torch.tensor([[2.0, 0.0], [1.0, 2.0]], dtype=dtype)
        for i in range(4):
            assert torch.equal(Dhat[0, i], 2 * R)
        exp = [R, R.T, R, -0.5 * R]
        for q in range(4):
            assert torch.equal(C[0, q], exp[q]), q
        assert torch.equal(x, torch.ones_like(x))


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide", "atomic"])
@pytest.mark.parametrize("k", [3, 5, 7])
def test_closed_form_laplacian(variant, k):
    N, n = 2 ** k - 1, 4
    R = torch.tensor(np.tril(np.random.default_rng(k).uniform(-1, 1, (n, n))) + 2 * np.eye(n))
    prob = btdgen.lap(2, N, R)
    p, Dhat, C, x, info = _run(prob, torch.float64, variant)
    from oracle.perm import coupling_slots, level_of

    for i in range(1, N + 1):
        assert torch.allclose(Dhat[0, i - 1], 2 ** ((2 - level_of(i)) / 2) * R, atol=1e-12)
    for q, (lv, kk, _a, _b) in enumerate(coupling_slots(N)):
        exp = -(2 ** (-lv / 2)) * (R if kk % 2 else R.T)
        assert torch.allclose(C[1, q], exp, atol=1e-12), (lv, kk)


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide", "atomic"])
def test_identity_and_zero_coupling(variant):
    dev = _dev()
    N, n = 19, 5
    D = torch.eye(n, dtype=torch.float64).expand(2, N, n, n).contiguous()
    E = torch.zeros(2, N - 1, n, n, dtype=torch.float64)
    b = torch.randn(2, N, n, 1, dtype=torch.float64)
    Dhat, C, x, info = btd.factor_solve(D.to(dev), E.to(dev), b.to(dev), variant=variant)
    assert torch.equal(Dhat.cpu(), D) and not C.any() and torch.equal(x.cpu(), b)
    A = torch.randn(2, N, n, n, dtype=torch.float64)
    D = A @ A.transpose(-1, -2) + n * torch.eye(n, dtype=torch.float64)
    Dhat, C, x, info = btd.factor_solve(D.to(dev), E.to(dev), b.to(dev), variant=variant)
    assert torch.allclose(Dhat.cpu(), torch.linalg.cholesky(D), atol=1e-12) and not C.any()
    assert torch.allclose(x.cpu(), torch.linalg.solve(D, b), atol=1e-12)


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide", "atomic"])
def test_lower_triangle_only_is_read(variant):
    prob = btdgen.dd(2, 21, 6, seed=3)
    garbage = prob.D + torch.triu(torch.full_like(prob.D, 1e30), 1)
    junk = btdgen.Problem(garbage, prob.E, prob.b, None)
    _, Dh1, C1, x1, _ = _run(prob, torch.float64, variant)
    _, Dh2, C2, x2, _ = _run(junk, torch.float64, variant)
    if variant == "atomic":  # nondeterministic summation order: equal to rounding (1e30 garbage would show)
        for a, b in ((Dh1, Dh2), (C1, C2), (x1, x2)):
            assert float((a - b).abs().max()) <= 1e-12 * float(a.abs().max())
    else:
        assert torch.equal(Dh1, Dh2) and torch.equal(C1, C2) and torch.equal(x1, x2)


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide", "atomic"])
def test_failure_info(variant):
    dev = _dev()
    prob = btdgen.dd(4, 16, 3, seed=2)
    D = prob.D.clone()
    D[0, 5] = -torch.eye(3, dtype=torch.float64)   # block 6 (level 2)
    D[1, 2] = -torch.eye(3, dtype=torch.float64)   # block 3 (level 1)
    D[1, 7] = -torch.eye(3, dtype=torch.float64)   # block 8 (level 4): level 1 failure wins
    D[3, 15] = torch.zeros(3, 3, dtype=torch.float64)  # block 16 (level 5), zero pivot
    _, _, _, info = btd.factor_solve(D.to(dev), prob.E.to(dev), prob.b.to(dev), variant=variant)
    assert info.cpu().tolist() == [6, 3, 0, 16]
    _, _, info2 = btd.factor(D.to(dev), prob.E.to(dev), variant=variant)
    assert info2.cpu().tolist() == [6, 3, 0, 16]


@pytest.mark.parametrize("variant", ["fused", "level", "persist", "wide"])
def test_deterministic_and_shard_invariant(variant):
    prob = btdgen.kalman(12, 50, 12, seed=4).cast(torch.float32)
    dev = _dev()
    D, E, b = prob.D.to(dev), prob.E.to(dev), prob.b.to(dev)
    r1 = btd.factor_solve(D, E, b, variant=variant)
    r2 = btd.factor_solve(D, E, b, variant=variant)
    for a, c in zip(r1, r2):
        assert torch.equal(a, c)
    sub = btd.factor_solve(D[5:9].contiguous(), E[5:9].contiguous(), b[5:9].contiguous(), variant=variant)
    for a, c in zip(r1, sub):
        assert torch.equal(a[5:9], c)


def test_variants_agree():
    prob = btdgen.dd(3, 77, 12, seed=8)
    _, Dh1, C1, x1, _ = _run(prob, torch.float64, "fused")
    for v in ("level", "persist", "wide", "atomic"):
        _, Dh2, C2, x2, _ = _run(prob, torch.float64, v)
        assert (Dh1 - Dh2).abs().max() < 1e-13 and (C1 - C2).abs().max() < 1e-13 and (x1 - x2).abs().max() < 1e-12


@pytest.mark.parametrize("n", [4, 12, 32])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_atomic_schedule_agrees_with_deferred(n, dtype):
    """Alg. 5 (atomic right-looking) vs Alg. 4 (deferred) on the same inputs: factors and solutions
    agree to rounding -- <= 1e-12 relative in fp64, 1e-5 in fp32 -- and every system
    matches the oracle (the atomic order is nondeterministic, so agreement is not bitwise)."""
    for N in (5, 16, 33, 100, 257):
        prob = btdgen.kalman(1, N, n, seed=7 * N + n)
        p, Dh1, C1, x1, i1 = _run(prob, dtype, "wide")
        _, Dh2, C2, x2, i2 = _run(prob, dtype, "atomic")
        tol = 1e-12 if dtype == torch.float64 else 1e-5
        rel = lambda a, b: float((a.double() - b.double()).abs().max() / b.double().abs().max())  # noqa: E731
        assert rel(Dh2, Dh1) <= tol and rel(C2, C1) <= tol and rel(x2, x1) <= tol, (N, rel(Dh2, Dh1), rel(C2, C1), rel(x2, x1))
        _check(p, Dh2, C2, x2, i2, dtype)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_config_c3_atomic(dtype):
    prob = btdgen.make("kalman", 1, 1024, 32, seed=3)
    _check(*_run(prob, dtype, "atomic"), dtype)


@pytest.mark.parametrize("n", [33, 48, 64, 96, 128])
def test_large_blocks_persist(n):
    """n > 32 runs only on the PERSIST variant (AUTO picks it)."""
    for dtype in (torch.float64, torch.float32):
        for N in (1, 2, 7, 16):
            prob = btdgen.kalman(2, N, n, m=2 if n == 48 else 1, seed=n + N)
            _check(*_run(prob, dtype, "auto"), dtype)


def test_host_entry_point():
    _dev()
    prob = btdgen.kalman(6, 33, 12, seed=12).cast(torch.float32)
    plan = btd.Plan(33, 12, 6, 1, torch.float32)
    ws = btd.HostWorkspace(plan)
    D, E, b = (t.pin_memory() for t in (prob.D, prob.E, prob.b))
    for chunks in (1, 4, 8):  # 8 > batch: one system per slice
        Dhat, C, x, info = btd.factor_solve_host(D, E, b, ws, chunks=chunks)
        torch.cuda.synchronize()
        _check(prob, Dhat.clone(), C.clone(), x.clone(), info.clone(), torch.float32)


# ------------------------------------------------------------------ BASELINE.json configs at full size

def test_config_c1_fp64_n2_N8():
    for kind in ("dd", "kalman"):
        prob = btdgen.make(kind, 1, 8, 2, seed=1)
        _check(*_run(prob, torch.float64, "auto"), torch.float64)
    prob = btdgen.lap(1, 7, torch.tensor([[2.0, 0.0], [1.0, 2.0]]))
    _check(*_run(prob, torch.float64, "auto"), torch.float64)


def test_config_c2_fp64_n16_N64():
    for kind in ("dd", "kalman"):
        prob = btdgen.make(kind, 1, 64, 16, seed=2)
        _check(*_run(prob, torch.float64, "auto"), torch.float64)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_config_c3_n32_N1024(dtype):
    for kind in ("dd", "kalman"):
        prob = btdgen.make(kind, 1, 1024, 32, seed=3)
        _check(*_run(prob, dtype, "auto"), dtype)


def test_config_c4_fp64_n128_N256():
    for kind in ("dd", "kalman"):
        prob = btdgen.make(kind, 1, 256, 128, seed=4)
        _check(*_run(prob, torch.float64, "auto"), torch.float64)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_config_c3_sweep(dtype):
    for N in (8, 15, 16, 17, 63, 64, 65, 255, 256, 257, 2047, 4096):
        prob = btdgen.kalman(1, N, 32, seed=N)
        _check(*_run(prob, dtype, "auto"), dtype)


def test_config_c5_batched_fp32_n12_N128():
    """8192 systems in the bench's launch configuration; oracle on sampled systems, residual on all."""
    dev = _dev()
    B, N, n = 8192, 128, 12
    for kind in ("kalman", "dd"):
        prob = btdgen.make(kind, B, N, n, seed=5, device=dev).cast(torch.float32)
        Dhat, C, x, info = btd.factor_solve(prob.D, prob.E, prob.b)
        torch.cuda.synchronize()
        assert int(info.abs().sum()) == 0
        sample = [0, 1, 777, 4095, 4096, 8190, 8191]
        cpu = btdgen.Problem(prob.D[sample].cpu(), prob.E[sample].cpu(), prob.b[sample].cpu(), None)
        _check(cpu, Dhat[sample].cpu(), C[sample].cpu(), x[sample].cpu(), info[sample].cpu(), torch.float32)
        # residual of every system, evaluated in fp64 on the device
        Dd, Ed, xd, bd = prob.D.double(), prob.E.double(), x.double(), prob.b.double()
        r = btdgen.block_tridiag_matvec(Dd, Ed, xd) - bd
        rel = r.flatten(1).norm(dim=1) / bd.flatten(1).norm(dim=1)
        assert float(rel.max()) <= 1e-5, float(rel.max())


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_auto_short_systems_with_32_wide_blocks(dtype):
    """AUTO picks WIDE for short single systems with n = 32 (N >= 4 fp64, N >= 12 fp32) and for
    long ones up to 2048 / 1024 level-1 columns: parity at the switch points."""
    for N in (2, 3, 4, 5, 8, 11, 12, 15, 2047, 2049):
        prob = btdgen.kalman(1, N, 32, m=1, seed=N)
        _check(*_run(prob, dtype, "auto"), dtype, check_L=N < 1000)


def test_c_abi_from_plain_c():
    """tools/c_api_demo.c (gcc -std=c11, no Python/torch): plan, cudaMalloc'd buffers, btd_factor_solve,
    known solution -- the boundary is usable from C as include/btd.h documents it."""
    import subprocess

    _dev()
    from paper_2601_03754_b200 import build

    exe = build.build_c_demo()
    for args in ([], ["1", "3"], ["1000", "32"], ["37", "12"]):
        r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and "c_api_demo ok" in r.stdout, (args, r.stdout, r.stderr)
