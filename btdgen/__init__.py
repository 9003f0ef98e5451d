"""Seeded synthetic inputs for SPD block-tridiagonal systems.

This module is shared by the tests, ``bench.py`` and the oracle drivers. It
holds none of the factorization/solve arithmetic of the method (SURVEY.md
§8(d) "Generators"); it only draws the matrices ``D``, ``E``, a known solution
``x*`` and the right-hand side ``b = Psi x*``.

Randomness is a counter-based hash (``lowbias32`` mixing, integer-exact in
int64 torch arithmetic), keyed by ``(config seed, global system index,
element counter)``. The random BITS are therefore identical on CPU and GPU
and for any sharding of a batch across ranks. The floating-point values built
from them are bit-identical under any sharding on ONE device type; across CPU
and GPU they agree only to rounding (``kalman`` uses ``torch.linalg.qr`` and
matmuls, and the Box-Muller transform uses log/cos, whose last bits differ
between the CPU and CUDA libraries).

Generators:

* ``dd``     -- SPEC.md:429/446 mapping with the provably-SPD shift 3n+1
               (SURVEY.md §8(c) A18): D_i = S_i + (3n+1) I, S_i symmetric
               uniform[-1,1]; E_i uniform[-1,1].
* ``kalman`` -- information matrix of a time-varying linear-Gaussian
               state-space model (PAPER.md:20 names MPC/Kalman filtering;
               recipe in SURVEY.md §8(d)).
* ``lap``    -- T_N (x) M with T = tridiag(-1, 2, -1), M = R R^T (closed-form pin).

All generators produce float64 tensors; ``cast`` rounds them to the working
dtype and the oracle always consumes the rounded values upcast back to
float64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

_M32 = 0xFFFFFFFF


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for 0 <= x < 2^32 without int64 overflow."""
    lo = x & 0xFFFF
    hi = x >> 16
    return ((lo * c) + (((hi * c) & 0xFFFF) << 16)) & _M32


def _mix32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32 integer hash (public-domain mixing constants)."""
    x = x & _M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def hash_u32(seed: int, system: torch.Tensor, counter: torch.Tensor) -> torch.Tensor:
    """Counter-based 32-bit hash of (seed, system, counter); broadcasting int64 tensors."""
    s = _mix32(torch.as_tensor(seed & _M32, dtype=torch.int64, device=system.device) ^ 0x5BD1E995)
    h = _mix32(s ^ (system & _M32))
    h = _mix32(h ^ (counter & _M32))
    h = _mix32(h ^ ((counter >> 32) + 0x27D4EB2F))
    return h


def uniform(seed: int, system: torch.Tensor, counter: torch.Tensor) -> torch.Tensor:
    """Uniform on [-1, 1) with 24-bit resolution (every value exact in fp32)."""
    h = hash_u32(seed, system, counter)
    return (h >> 8).to(torch.float64) * (2.0 ** -23) - 1.0


def normal(seed: int, system: torch.Tensor, counter: torch.Tensor) -> torch.Tensor:
    """Standard normal by Box-Muller from two hashed uniforms (counters 2c, 2c+1)."""
    u1 = (hash_u32(seed, system, 2 * counter) >> 8).to(torch.float64)
    u2 = (hash_u32(seed, system, 2 * counter + 1) >> 8).to(torch.float64)
    u1 = (u1 + 0.5) * (2.0 ** -24)  # (0, 1)
    u2 = u2 * (2.0 ** -24)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


@dataclass
class Problem:
    """A batch of block-tridiagonal systems, float64, batch-outermost layout.

    D: [B, N, n, n] symmetric; E: [B, N-1, n, n] (E[k-1] is block (k+1, k));
    b: [B, N, n, m]; xstar: [B, N, n, m] (the solution used to build b, or None).
    """

    D: torch.Tensor
    E: torch.Tensor
    b: torch.Tensor
    xstar: torch.Tensor | None

    def __post_init__(self):
        self.D, self.E, self.b = self.D.contiguous(), self.E.contiguous(), self.b.contiguous()

    @property
    def batch(self) -> int:
        return self.D.shape[0]

    @property
    def N(self) -> int:
        return self.D.shape[1]

    @property
    def n(self) -> int:
        return self.D.shape[2]

    @property
    def m(self) -> int:
        return self.b.shape[3]

    def cast(self, dtype: torch.dtype) -> "Problem":
        """Round D, E, b to ``dtype`` (x* is kept in float64)."""
        return Problem(self.D.to(dtype), self.E.to(dtype), self.b.to(dtype), self.xstar)

    def to(self, device) -> "Problem":
        xs = None if self.xstar is None else self.xstar.to(device)
        return Problem(self.D.to(device), self.E.to(device), self.b.to(device), xs)

    def f64(self) -> "Problem":
        """Upcast the (possibly rounded) inputs back to float64 for the oracle."""
        xs = self.xstar
        return Problem(self.D.double(), self.E.double(), self.b.double(), xs)


def _systems(batch: int, first: int, device) -> torch.Tensor:
    return torch.arange(first, first + batch, dtype=torch.int64, device=device)


def block_tridiag_matvec(D: torch.Tensor, E: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """Psi x for Psi = tridiag(E, D, E^T); float64 in, float64 out."""
    y = D @ x
    if D.shape[1] > 1:
        y[:, 1:] += E @ x[:, :-1]
        y[:, :-1] += E.transpose(-1, -2) @ x[:, 1:]
    return y


def rhs_from_solution(D, E, seed: int, systems: torch.Tensor, m: int, counter_base: int):
    B, N, n, _ = D.shape
    cnt = torch.arange(N * n * m, dtype=torch.int64, device=D.device) + counter_base
    xs = normal(seed, systems[:, None], cnt[None, :]).reshape(B, N, n, m)
    return block_tridiag_matvec(D, E, xs), xs


def dd(batch: int, N: int, n: int, m: int = 1, seed: int = 0, first_system: int = 0,
       device="cpu") -> Problem:
    """Diagonally dominant generator ``dd`` (shift 3n+1 per A18)."""
    sys_ = _systems(batch, first_system, device)
    nn = n * n
    cD = torch.arange(N * nn, dtype=torch.int64, device=device)
    U = uniform(seed, sys_[:, None], cD[None, :]).reshape(batch, N, n, n)
    low = torch.tril(U)
    S = low + torch.tril(U, -1).transpose(-1, -2)
    eye = torch.eye(n, dtype=torch.float64, device=device)
    D = S + (3 * n + 1) * eye
    if N > 1:
        cE = torch.arange((N - 1) * nn, dtype=torch.int64, device=device) + N * nn
        E = uniform(seed, sys_[:, None], cE[None, :]).reshape(batch, N - 1, n, n)
    else:
        E = torch.zeros(batch, 0, n, n, dtype=torch.float64, device=device)
    b, xs = rhs_from_solution(D, E, seed, sys_, m, counter_base=(2 * N) * nn)
    return Problem(D, E, b, xs)


def kalman(batch: int, N: int, n: int, m: int = 1, seed: int = 0, first_system: int = 0,
           device="cpu") -> Problem:
    """Kalman/MPC-shaped information matrix (SURVEY.md §8(d) ``kalman``).

    A_k = 0.98 Q_k (Q_k orthogonal from a QR of a Gaussian), C_k Gaussian ceil(n/2) x n,
    Q = 0.1 I, R = I, P0 = I:
      D_1 = P0^-1 + A_1^T Q^-1 A_1 + C_1^T R^-1 C_1
      D_k = Q^-1 + A_k^T Q^-1 A_k + C_k^T R^-1 C_k   (1 < k < N)
      D_N = Q^-1 + C_N^T R^-1 C_N
      E_k = -Q^-1 A_k
    """
    sys_ = _systems(batch, first_system, device)
    p = (n + 1) // 2
    nn = n * n
    cA = torch.arange(N * nn, dtype=torch.int64, device=device)
    G = normal(seed, sys_[:, None], cA[None, :]).reshape(batch, N, n, n)
    Qk, Rk = torch.linalg.qr(G)
    # sign-fix so the orthogonal factor is a deterministic function of G
    sgn = torch.sign(torch.diagonal(Rk, dim1=-2, dim2=-1))
    sgn = torch.where(sgn == 0, torch.ones_like(sgn), sgn)
    A = 0.98 * (Qk * sgn[..., None, :])
    cC = torch.arange(N * p * n, dtype=torch.int64, device=device) + N * nn
    Cm = normal(seed, sys_[:, None], cC[None, :]).reshape(batch, N, p, n)
    qinv = 10.0
    eye = torch.eye(n, dtype=torch.float64, device=device)
    CtC = Cm.transpose(-1, -2) @ Cm
    AtA = A.transpose(-1, -2) @ A
    D = CtC.clone()
    D[:, 0] += eye  # P0^-1
    if N > 1:
        D[:, 1:] += qinv * eye
        D[:, :-1] += qinv * AtA[:, :-1]
        E = -qinv * A[:, :-1]
    else:
        E = torch.zeros(batch, 0, n, n, dtype=torch.float64, device=device)
    D = 0.5 * (D + D.transpose(-1, -2))
    b, xs = rhs_from_solution(D, E, seed, sys_, m, counter_base=(2 * N + 2) * nn)
    return Problem(D, E, b, xs)


def lap(batch: int, N: int, R: torch.Tensor, m: int = 1, seed: int = 0, first_system: int = 0,
        device="cpu") -> Problem:
    """Psi = T_N (x) M, T = tridiag(-1, 2, -1), M = R R^T (SURVEY.md §8(c) closed-form pin)."""
    R = R.to(torch.float64).to(device)
    n = R.shape[0]
    M = R @ R.T
    D = (2.0 * M).expand(batch, N, n, n).clone()
    E = (-M).expand(batch, max(N - 1, 0), n, n).clone()
    sys_ = _systems(batch, first_system, device)
    b, xs = rhs_from_solution(D, E, seed, sys_, m, counter_base=0)
    return Problem(D, E, b, xs)


GENERATORS = {"dd": dd, "kalman": kalman}


def make(kind: str, batch: int, N: int, n: int, m: int = 1, seed: int = 0, first_system: int = 0,
         device="cpu") -> Problem:
    return GENERATORS[kind](batch, N, n, m=m, seed=seed, first_system=first_system, device=device)


# ----------------------------------------------------------------------------- extensions (§8(f) f4)

@dataclass
class ArrowProblem:
    """Block-tridiagonal-arrow systems K = [[Psi, G^T], [G, Z]] (oracle/arrow.py), float64.

    D, E, b as in ``Problem``; G: [B, N, n_a, n] (G[i-1] = border block of original block i);
    Z: [B, n_a, n_a]; ba: [B, n_a, m]; xstar / xastar: the solution used to build (b, ba).
    """

    D: torch.Tensor
    E: torch.Tensor
    G: torch.Tensor
    Z: torch.Tensor
    b: torch.Tensor
    ba: torch.Tensor
    xstar: torch.Tensor
    xastar: torch.Tensor

    def cast(self, dtype):
        return ArrowProblem(*(t.to(dtype).contiguous() for t in (self.D, self.E, self.G, self.Z, self.b, self.ba)),
                            self.xstar, self.xastar)

    def to(self, device):
        return ArrowProblem(*(t.to(device) for t in (self.D, self.E, self.G, self.Z, self.b, self.ba,
                                                      self.xstar, self.xastar)))


def arrow(batch: int, N: int, n: int, na: int, m: int = 1, seed: int = 0, first_system: int = 0,
          device="cpu") -> ArrowProblem:
    """``dd`` block-tridiagonal part plus a border: G_i entries uniform[-1,1] / sqrt(N n) (so
    ||G||_F^2 <= n_a), Z = S_Z + (4 n_a + 1) I with S_Z symmetric uniform[-1,1]. Provably SPD:
    lambda_min(Psi) >= 1 (A18) and lambda_min(Z) >= n_a + 1 > ||G Psi^{-1} G^T||."""
    base = dd(batch, N, n, m=m, seed=seed, first_system=first_system, device=device)
    sys_ = _systems(batch, first_system, device)
    c0 = (2 * N + 2) * n * n + 2 * N * n * m + 1_000_003
    cG = torch.arange(N * na * n, dtype=torch.int64, device=device) + c0
    G = uniform(seed, sys_[:, None], cG[None, :]).reshape(batch, N, na, n) / math.sqrt(N * n)
    cZ = torch.arange(na * na, dtype=torch.int64, device=device) + c0 + N * na * n
    U = uniform(seed, sys_[:, None], cZ[None, :]).reshape(batch, na, na)
    Z = torch.tril(U) + torch.tril(U, -1).transpose(-1, -2) + (4 * na + 1) * torch.eye(
        na, dtype=torch.float64, device=device)
    cx = torch.arange(na * m, dtype=torch.int64, device=device) + c0 + N * na * n + na * na
    xa = normal(seed, sys_[:, None], cx[None, :]).reshape(batch, na, m)
    xs = base.xstar
    # b = Psi x* + G^T x_a*,  b_a = G x* + Z x_a*
    b = block_tridiag_matvec(base.D, base.E, xs) + G.transpose(-1, -2) @ xa[:, None]
    ba = torch.einsum("bian,binm->bam", G, xs) + Z @ xa
    return ArrowProblem(base.D, base.E, G, Z, b, ba, xs, xa)


@dataclass
class BandedProblem:
    """Block-banded systems of block bandwidth w (oracle/banded.py), float64.

    D: [B, N, n, n]; A: [B, w, N, n, n] with A[:, k-1, i-1] = block (i+k, i) (entries with
    i + k > N are zero and never read); b, xstar: [B, N, n, m].
    """

    D: torch.Tensor
    A: torch.Tensor
    b: torch.Tensor
    xstar: torch.Tensor

    def cast(self, dtype):
        return BandedProblem(self.D.to(dtype).contiguous(), self.A.to(dtype).contiguous(),
                             self.b.to(dtype).contiguous(), self.xstar)

    def to(self, device):
        return BandedProblem(self.D.to(device), self.A.to(device), self.b.to(device), self.xstar.to(device))


def banded_matvec(D: torch.Tensor, A: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """Psi_w x (float64): y_i = D_i x_i + sum_k (A_k[i-k] x_{i-k} + A_k[i]^T x_{i+k})."""
    y = D @ x
    N = D.shape[1]
    for k in range(1, A.shape[1] + 1):
        if N > k:
            Ak = A[:, k - 1, :N - k]
            y[:, k:] += Ak @ x[:, :N - k]
            y[:, :N - k] += Ak.transpose(-1, -2) @ x[:, k:]
    return y


def banded(batch: int, N: int, n: int, w: int, m: int = 1, seed: int = 0, first_system: int = 0,
           device="cpu") -> BandedProblem:
    """D_i = S_i + ((2w+1) n + 1) I (S_i symmetric uniform[-1,1]), A_k[i] uniform[-1,1]:
    Gershgorin gives lambda_min >= 1 (the w = 1 case is ``dd``'s shift 3n+1)."""
    sys_ = _systems(batch, first_system, device)
    nn = n * n
    cD = torch.arange(N * nn, dtype=torch.int64, device=device)
    U = uniform(seed, sys_[:, None], cD[None, :]).reshape(batch, N, n, n)
    D = torch.tril(U) + torch.tril(U, -1).transpose(-1, -2) + ((2 * w + 1) * n + 1) * torch.eye(
        n, dtype=torch.float64, device=device)
    cA = torch.arange(w * N * nn, dtype=torch.int64, device=device) + N * nn
    A = uniform(seed, sys_[:, None], cA[None, :]).reshape(batch, w, N, n, n)
    for k in range(1, w + 1):
        A[:, k - 1, max(N - k, 0):] = 0.0
    cx = torch.arange(N * n * m, dtype=torch.int64, device=device) + (w + 1) * N * nn
    xs = normal(seed, sys_[:, None], cx[None, :]).reshape(batch, N, n, m)
    return BandedProblem(D, A, banded_matvec(D, A, xs), xs)
