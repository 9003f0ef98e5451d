"""Thin Python binding of the C ABI in include/btd.h (argument marshalling only).

Every step of the factorization and solve runs in the CUDA kernels of ``libbtd.so``; this
module only checks tensor shapes/dtypes/devices, allocates outputs with torch and passes raw
device pointers plus the current CUDA stream. There is no CPU fallback: if the shared library
or a CUDA device is missing, calls raise.

Names follow include/btd.h: ``Plan`` (btd_plan), ``factor`` (btd_factor), ``solve`` (btd_solve),
``factor_solve`` (btd_factor_solve), ``factor_solve_host`` (btd_factor_solve_host),
``permutation`` (btd_permutation).
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BTD_LIB") or os.path.join(_HERE, "libbtd.so")  # BTD_LIB: dev override (timing build)

BTD_F32, BTD_F64 = 0, 1
VARIANTS = {"auto": 0, "fused": 1, "level": 2, "persist": 3, "wide": 4, "atomic": 5}
VARIANT_NAMES = {1: "fused", 2: "level", 3: "persist", 4: "wide", 5: "atomic"}
_STATUS = {0: "BTD_OK", 1: "BTD_EINVAL", 2: "BTD_ECUDA", 3: "BTD_ENOMEM", 4: "BTD_EUNSUPPORTED"}

_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32

# (name, restype, argtypes) for every entry point declared in include/btd.h
SIGNATURES = [
    ("btd_plan_create", ctypes.c_int, [ctypes.POINTER(_vp), _i64, _i64, _i64, _i64, ctypes.c_int]),
    ("btd_plan_create_ex", ctypes.c_int, [ctypes.POINTER(_vp), _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int]),
    ("btd_plan_destroy", None, [_vp]),
    ("btd_num_levels", _i32, [_vp]),
    ("btd_num_coupling_blocks", _i64, [_vp]),
    ("btd_level_offset", _i64, [_vp, _i32]),
    ("btd_permutation", ctypes.c_int, [_vp, ctypes.POINTER(_i64)]),
    ("btd_plan_variant", _i32, [_vp]),
    ("btd_plan_launches", _i32, [_vp, _i32]),
    ("btd_plan_smem_bytes", _i64, [_vp]),
    ("btd_factor", ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("btd_solve", ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    ("btd_factor_solve", ctypes.c_int, [_vp] * 9),
    ("btd_factor_solve_host", ctypes.c_int, [_vp] * 15 + [_i32, _vp]),
    ("btd_mixed_workspace_bytes", ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_size_t)]),
    ("btd_mixed_factor_solve", ctypes.c_int, [_vp] * 8 + [_i32, _vp, _vp, _vp]),
    ("btd_mixed_solve", ctypes.c_int, [_vp] * 7 + [_i32, _vp, _vp, _vp]),
    ("btd_arrow_factor_solve", ctypes.c_int, [_vp, _i64] + [_vp] * 15),
    ("btd_banded_factor_solve", ctypes.c_int, [_vp, _i64, _i64, _i64] + [_vp] * 12),
    ("btd_partition_local", ctypes.c_int, [_vp] * 15),
    ("btd_partition_reduce", ctypes.c_int, [_vp, _i32] + [_vp] * 9),
    ("btd_partition_finish", ctypes.c_int, [_vp] * 6),
    ("btd_status_string", ctypes.c_char_p, [ctypes.c_int]),
    ("btd_last_error", ctypes.c_char_p, []),
]


class BtdError(RuntimeError):
    pass


def lib():
    """Load libbtd.so (built by ``paper_2601_03754_b200.build``); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BtdError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().btd_last_error().decode()
        raise BtdError(f"{what}: {_STATUS.get(rc, rc)} {msg}")


def _dt(dtype: torch.dtype) -> int:
    if dtype == torch.float32:
        return BTD_F32
    if dtype == torch.float64:
        return BTD_F64
    raise TypeError(f"unsupported dtype {dtype} (float32 or float64)")


class Plan:
    """btd_plan: symbolic analysis for ``batch`` systems of N blocks of size n, m right-hand sides."""

    def __init__(self, N: int, n: int, batch: int = 1, m: int = 1, dtype: torch.dtype = torch.float64,
                 variant: str = "auto"):
        self.N, self.n, self.batch, self.m, self.dtype = int(N), int(n), int(batch), int(m), dtype
        h = _vp()
        _check(lib().btd_plan_create_ex(ctypes.byref(h), self.N, self.n, self.batch, self.m, _dt(dtype),
                                        VARIANTS[variant]), "btd_plan_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.btd_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def levels(self) -> int:
        return lib().btd_num_levels(self._h)

    @property
    def num_coupling_blocks(self) -> int:
        return lib().btd_num_coupling_blocks(self._h)

    def level_offset(self, level: int) -> int:
        return lib().btd_level_offset(self._h, level)

    def permutation(self) -> list[int]:
        arr = (_i64 * self.N)()
        _check(lib().btd_permutation(self._h, arr), "btd_permutation")
        return list(arr)

    @property
    def variant(self) -> str:
        return VARIANT_NAMES[lib().btd_plan_variant(self._h)]

    def launches(self, op: str = "factor_solve") -> int:
        return lib().btd_plan_launches(self._h, {"factor": 0, "solve": 1, "factor_solve": 2}[op])

    @property
    def smem_bytes(self) -> int:
        return lib().btd_plan_smem_bytes(self._h)


def _ptr(t: torch.Tensor | None):
    return None if t is None else _vp(t.data_ptr())


def _stream(stream, device: torch.device) -> _vp:
    """The stream to launch on: the caller's (must belong to ``device``) or ``device``'s current one."""
    if stream is None:
        stream = torch.cuda.current_stream(device)
    elif stream.device != device:
        raise ValueError(f"stream is on {stream.device}, tensors on {device}")
    return _vp(stream.cuda_stream)


def _check_in(name, t, shape, dtype, device: torch.device | None = None, align: int = 16):
    """Every buffer handed to the library (inputs AND caller-supplied outputs): a contiguous CUDA
    tensor of the plan's shape and dtype, aligned for the kernels' vector accesses, on ``device``."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise BtdError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device} (all tensors must share one device)")
    if t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.data_ptr() % align:
        raise ValueError(f"{name} must be {align}-byte aligned")


def _check_host(name, t, shape, dtype):
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise ValueError(f"{name} must be a host tensor")
    if t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous {dtype} host tensor of shape {tuple(shape)}, got "
                         f"{t.dtype} {tuple(t.shape)}")


def _plan_for(D: torch.Tensor, m: int, plan: Plan | None, variant: str) -> Plan:
    B, N, n, _ = D.shape
    if plan is None:
        return Plan(N, n, B, m, D.dtype, variant)
    if (plan.batch, plan.N, plan.n, plan.dtype) != (B, N, n, D.dtype) or plan.m != m:
        raise ValueError("plan does not match the tensors")
    return plan


def _shapes(plan: Plan):
    B, N, n, m = plan.batch, plan.N, plan.n, plan.m
    return dict(D=(B, N, n, n), E=(B, max(N - 1, 0), n, n), C=(B, plan.num_coupling_blocks, n, n),
                b=(B, N, n, m))


def factor(D: torch.Tensor, E: torch.Tensor, plan: Plan | None = None, variant: str = "auto", stream=None,
           out: tuple | None = None):
    """btd_factor: returns (Dhat, C, info). D [B,N,n,n], E [B,N-1,n,n] on the GPU."""
    p = _plan_for(D, 1 if plan is None else plan.m, plan, variant)
    sh = _shapes(p)
    dev = D.device
    _check_in("D", D, sh["D"], p.dtype, dev)
    _check_in("E", E, sh["E"], p.dtype, dev)
    if out is None:
        Dhat = torch.empty(sh["D"], dtype=p.dtype, device=dev)
        C = torch.empty(sh["C"], dtype=p.dtype, device=dev)
        info = torch.empty(p.batch, dtype=torch.int32, device=dev)
    else:
        Dhat, C, info = out
        _check_in("out Dhat", Dhat, sh["D"], p.dtype, dev)
        _check_in("out C", C, sh["C"], p.dtype, dev)
        _check_in("out info", info, (p.batch,), torch.int32, dev, align=4)
    with torch.cuda.device(dev):
        _check(lib().btd_factor(p.handle, _ptr(D), _ptr(E) if p.N > 1 else None, _ptr(Dhat), _ptr(C), _ptr(info),
                                _stream(stream, dev)), "btd_factor")
    return Dhat, C, info


def solve(Dhat: torch.Tensor, C: torch.Tensor, b: torch.Tensor, plan: Plan | None = None, variant: str = "auto",
          stream=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """btd_solve: x = Psi^{-1} b from a factor (Dhat, C) of btd_factor."""
    p = _plan_for(Dhat, b.shape[3], plan, variant)
    sh = _shapes(p)
    dev = Dhat.device
    _check_in("Dhat", Dhat, sh["D"], p.dtype, dev)
    _check_in("C", C, sh["C"], p.dtype, dev)
    _check_in("b", b, sh["b"], p.dtype, dev)
    x = torch.empty_like(b) if out is None else out
    _check_in("out x", x, sh["b"], p.dtype, dev)
    with torch.cuda.device(dev):
        _check(lib().btd_solve(p.handle, _ptr(Dhat), _ptr(C), _ptr(b), _ptr(x), _stream(stream, dev)), "btd_solve")
    return x


def factor_solve(D: torch.Tensor, E: torch.Tensor, b: torch.Tensor, plan: Plan | None = None,
                 variant: str = "auto", stream=None, out: tuple | None = None):
    """btd_factor_solve: returns (Dhat, C, x, info)."""
    p = _plan_for(D, b.shape[3], plan, variant)
    sh = _shapes(p)
    dev = D.device
    _check_in("D", D, sh["D"], p.dtype, dev)
    _check_in("E", E, sh["E"], p.dtype, dev)
    _check_in("b", b, sh["b"], p.dtype, dev)
    if out is None:
        Dhat = torch.empty(sh["D"], dtype=p.dtype, device=dev)
        C = torch.empty(sh["C"], dtype=p.dtype, device=dev)
        x = torch.empty(sh["b"], dtype=p.dtype, device=dev)
        info = torch.empty(p.batch, dtype=torch.int32, device=dev)
    else:
        Dhat, C, x, info = out
        _check_in("out Dhat", Dhat, sh["D"], p.dtype, dev)
        _check_in("out C", C, sh["C"], p.dtype, dev)
        _check_in("out x", x, sh["b"], p.dtype, dev)
        _check_in("out info", info, (p.batch,), torch.int32, dev, align=4)
    with torch.cuda.device(dev):
        _check(lib().btd_factor_solve(p.handle, _ptr(D), _ptr(E) if p.N > 1 else None, _ptr(b), _ptr(Dhat),
                                      _ptr(C), _ptr(x), _ptr(info), _stream(stream, dev)), "btd_factor_solve")
    return Dhat, C, x, info


class HostWorkspace:
    """Pinned host outputs + device staging for ``factor_solve_host`` (allocated once, reused)."""

    def __init__(self, plan: Plan, device="cuda"):
        sh = _shapes(plan)
        dt = plan.dtype
        self.plan = plan
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.dev = {k: torch.empty(sh[k2], dtype=dt, device=device)
                    for k, k2 in [("D", "D"), ("E", "E"), ("b", "b"), ("Dhat", "D"), ("C", "C"), ("x", "b")]}
        self.dev["info"] = torch.empty(plan.batch, dtype=torch.int32, device=device)
        self.host = {k: torch.empty(sh[k2], dtype=dt, pin_memory=True)
                     for k, k2 in [("Dhat", "D"), ("C", "C"), ("x", "b")]}
        self.host["info"] = torch.empty(plan.batch, dtype=torch.int32, pin_memory=True)


def factor_solve_host(D: torch.Tensor, E: torch.Tensor, b: torch.Tensor, ws: HostWorkspace, chunks: int = 1,
                      stream=None):
    """btd_factor_solve_host: host (pinned) D, E, b in; host Dhat, C, x, info out (all async on stream)."""
    p = ws.plan
    sh = _shapes(p)
    for name, t in (("D", D), ("E", E), ("b", b)):
        _check_host(name, t, sh[name], p.dtype)
    d, h = ws.dev, ws.host
    with torch.cuda.device(ws.device):
        _check(lib().btd_factor_solve_host(
            p.handle, _ptr(D), _ptr(E) if p.N > 1 else None, _ptr(b), _ptr(h["Dhat"]), _ptr(h["C"]), _ptr(h["x"]),
            _ptr(h["info"]), _ptr(d["D"]), _ptr(d["E"]) if p.N > 1 else None, _ptr(d["b"]), _ptr(d["Dhat"]),
            _ptr(d["C"]), _ptr(d["x"]), _ptr(d["info"]), int(chunks), _stream(stream, ws.device)),
            "btd_factor_solve_host")
    return h["Dhat"], h["C"], h["x"], h["info"]


def permutation(N: int) -> list[int]:
    """btd_permutation: P_inf, perm[new position] = original index (0-based)."""
    return Plan(N, 1, 1, 1, torch.float64).permutation()
