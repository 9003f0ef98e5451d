"""Bindings of the §8(f) extension entry points of include/btd.h (argument marshalling only).

* ``mixed_factor_solve``  -- btd_mixed_factor_solve: binary32 factor + binary64 iterative refinement.
* ``mixed_solve``         -- btd_mixed_solve: the refinement for a new right-hand side, same factor.
* ``arrow_factor_solve``  -- btd_arrow_factor_solve: block-tridiagonal-arrow systems.
* ``banded_factor_solve`` -- btd_banded_factor_solve: block-banded systems (bandwidth w).

All arithmetic runs in libbtd.so (csrc/btd_ext.cu + the core kernels); this module checks
shapes/dtypes/devices, allocates outputs and workspaces with torch, and passes pointers and the
current stream. No CPU fallback.
"""
from __future__ import annotations

import ctypes

import torch

from .btd import Plan, _check, _check_in, _ptr, _shapes, _stream, lib


def mixed_workspace_bytes(plan: Plan) -> int:
    out = ctypes.c_size_t(0)
    _check(lib().btd_mixed_workspace_bytes(plan.handle, ctypes.byref(out)), "btd_mixed_workspace_bytes")
    return int(out.value)


def mixed_factor_solve(D: torch.Tensor, E: torch.Tensor, b: torch.Tensor, iters: int = 3, plan: Plan | None = None,
                       want_resid: bool = False, stream=None, work: torch.Tensor | None = None):
    """btd_mixed_factor_solve: binary64 (D, E, b) -> (Dhat32, C32, x64, info, resid64 | None)."""
    B, N, n, _ = D.shape
    m = b.shape[3]
    if plan is None:
        plan = Plan(N, n, B, m, torch.float32)
    if plan.dtype != torch.float32 or (plan.batch, plan.N, plan.n, plan.m) != (B, N, n, m):
        raise ValueError("mixed_factor_solve needs a float32 plan of the system's shape")
    sh = _shapes(plan)
    dev = D.device
    _check_in("D", D, sh["D"], torch.float64, dev)
    _check_in("E", E, sh["E"], torch.float64, dev)
    _check_in("b", b, sh["b"], torch.float64, dev)
    Dhat = torch.empty(sh["D"], dtype=torch.float32, device=dev)
    C = torch.empty(sh["C"], dtype=torch.float32, device=dev)
    x = torch.empty(sh["b"], dtype=torch.float64, device=dev)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    resid = torch.empty(B, dtype=torch.float64, device=dev) if want_resid else None
    nbytes = mixed_workspace_bytes(plan)
    if work is None:
        work = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
    elif work.numel() < nbytes or not work.is_cuda or work.data_ptr() % 16:
        raise ValueError(f"work must be a 16-byte aligned device buffer of >= {nbytes} bytes")
    with torch.cuda.device(dev):
        _check(lib().btd_mixed_factor_solve(plan.handle, _ptr(D), _ptr(E) if N > 1 else None, _ptr(b), _ptr(Dhat),
                                            _ptr(C), _ptr(x), _ptr(info), int(iters), _ptr(resid), _ptr(work),
                                            _stream(stream, dev)), "btd_mixed_factor_solve")
    return Dhat, C, x, info, resid


def mixed_solve(D: torch.Tensor, E: torch.Tensor, b: torch.Tensor, Dhat: torch.Tensor, C: torch.Tensor,
                iters: int = 3, plan: Plan | None = None, want_resid: bool = False, stream=None,
                work: torch.Tensor | None = None):
    """btd_mixed_solve: refinement for a new binary64 b with the binary32 factor (Dhat, C) of
    mixed_factor_solve -> (x64, resid64 | None)."""
    B, N, n, _ = D.shape
    m = b.shape[3]
    if plan is None:
        plan = Plan(N, n, B, m, torch.float32)
    if plan.dtype != torch.float32 or (plan.batch, plan.N, plan.n, plan.m) != (B, N, n, m):
        raise ValueError("mixed_solve needs a float32 plan of the system's shape")
    sh = _shapes(plan)
    dev = D.device
    _check_in("D", D, sh["D"], torch.float64, dev)
    _check_in("E", E, sh["E"], torch.float64, dev)
    _check_in("b", b, sh["b"], torch.float64, dev)
    _check_in("Dhat", Dhat, sh["D"], torch.float32, dev)
    _check_in("C", C, sh["C"], torch.float32, dev)
    x = torch.empty(sh["b"], dtype=torch.float64, device=dev)
    resid = torch.empty(B, dtype=torch.float64, device=dev) if want_resid else None
    nbytes = mixed_workspace_bytes(plan)
    if work is None:
        work = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
    elif work.numel() < nbytes or not work.is_cuda or work.data_ptr() % 16:
        raise ValueError(f"work must be a 16-byte aligned device buffer of >= {nbytes} bytes")
    with torch.cuda.device(dev):
        _check(lib().btd_mixed_solve(plan.handle, _ptr(D), _ptr(E) if N > 1 else None, _ptr(b), _ptr(Dhat), _ptr(C),
                                     _ptr(x), int(iters), _ptr(resid), _ptr(work), _stream(stream, dev)),
               "btd_mixed_solve")
    return x, resid


def arrow_factor_solve(D, E, G, Z, b, ba, plan: Plan | None = None, stream=None):
    """btd_arrow_factor_solve -> (Dhat, C, Y, LZ, x, xa, info); Y[..., :na] = Psi^{-1} G^T."""
    B, N, n, _ = D.shape
    na = G.shape[2]
    mb = b.shape[3]
    dt = D.dtype
    if plan is None:
        plan = Plan(N, n, B, na + mb, dt)
    if (plan.batch, plan.N, plan.n, plan.m, plan.dtype) != (B, N, n, na + mb, dt):
        raise ValueError("arrow_factor_solve needs the plan of Psi with m = na + mb")
    sh = _shapes(plan)
    dev = D.device
    _check_in("D", D, sh["D"], dt, dev)
    _check_in("E", E, sh["E"], dt, dev)
    _check_in("G", G, (B, N, na, n), dt, dev, align=max(dt.itemsize, 1))
    _check_in("Z", Z, (B, na, na), dt, dev, align=dt.itemsize)
    _check_in("b", b, (B, N, n, mb), dt, dev, align=dt.itemsize)
    _check_in("ba", ba, (B, na, mb), dt, dev, align=dt.itemsize)
    Dhat = torch.empty(sh["D"], dtype=dt, device=dev)
    C = torch.empty(sh["C"], dtype=dt, device=dev)
    R = torch.empty(sh["b"], dtype=dt, device=dev)
    Y = torch.empty(sh["b"], dtype=dt, device=dev)
    LZ = torch.empty((B, na, na), dtype=dt, device=dev)
    x = torch.empty((B, N, n, mb), dtype=dt, device=dev)
    xa = torch.empty((B, na, mb), dtype=dt, device=dev)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _check(lib().btd_arrow_factor_solve(plan.handle, int(na), _ptr(D), _ptr(E) if N > 1 else None, _ptr(G),
                                            _ptr(Z), _ptr(b), _ptr(ba), _ptr(Dhat), _ptr(C), _ptr(R), _ptr(Y),
                                            _ptr(LZ), _ptr(x), _ptr(xa), _ptr(info), _stream(stream, dev)),
               "btd_arrow_factor_solve")
    return Dhat, C, Y, LZ, x, xa, info


def banded_factor_solve(D, A, b, plan: Plan | None = None, stream=None):
    """btd_banded_factor_solve -> (Dhat', C', x, info); D [B,N,n,n], A [B,w,N,n,n], b [B,N,n,m]."""
    B, N, n, _ = D.shape
    w = A.shape[1]
    m = b.shape[3]
    dt = D.dtype
    Np = -(-N // w)
    if plan is None:
        plan = Plan(Np, w * n, B, m, dt)
    if (plan.batch, plan.N, plan.n, plan.m, plan.dtype) != (B, Np, w * n, m, dt):
        raise ValueError("banded_factor_solve needs the plan of the super-block system (ceil(N/w), w n)")
    dev = D.device
    _check_in("D", D, (B, N, n, n), dt, dev, align=dt.itemsize)
    _check_in("A", A, (B, w, N, n, n), dt, dev, align=dt.itemsize)
    _check_in("b", b, (B, N, n, m), dt, dev, align=dt.itemsize)
    sh = _shapes(plan)
    Dp = torch.empty(sh["D"], dtype=dt, device=dev)
    Ep = torch.empty(sh["E"], dtype=dt, device=dev)
    bp = torch.empty(sh["b"], dtype=dt, device=dev)
    xp = torch.empty(sh["b"], dtype=dt, device=dev)
    Dhat = torch.empty(sh["D"], dtype=dt, device=dev)
    C = torch.empty(sh["C"], dtype=dt, device=dev)
    x = torch.empty((B, N, n, m), dtype=dt, device=dev)
    info = torch.empty(B, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _check(lib().btd_banded_factor_solve(plan.handle, N, n, w, _ptr(D), _ptr(A), _ptr(b), _ptr(Dp),
                                             _ptr(Ep) if Np > 1 else None, _ptr(bp), _ptr(Dhat),
                                             _ptr(C) if Np > 1 else None, _ptr(xp), _ptr(x), _ptr(info),
                                             _stream(stream, dev)), "btd_banded_factor_solve")
    return Dhat, C, x, info
