"""O1: ctypes front-end of oracle/seqchol.c (test infrastructure only).

Algorithm 1 and the block forward/backward substitution of
SPEC.md:201-204, in plain fp64 C loops. ``build()`` compiles the shared object
with gcc; it is called by ``__graft_entry__.build()`` and lazily on first use.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "seqchol.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", _LIB, _SRC,
                               "-lm", "-lpthread"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.orc_potrf.argtypes = [ctypes.c_int, _dp]
        L.orc_potrf.restype = ctypes.c_int
        L.orc_trsm_right.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.orc_trsm_left.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.orc_trsm_left_trans.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.orc_syrk_down.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_int]
        L.orc_gemm_neg.argtypes = [ctypes.c_int] * 3 + [_dp, _dp, _dp, ctypes.c_int]
        L.orc_seq_factor.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, _dp]
        L.orc_seq_factor.restype = ctypes.c_int
        L.orc_seq_solve.argtypes = [ctypes.c_int] * 3 + [_dp] * 4
        L.orc_seq_batch.argtypes = [ctypes.c_int] * 4 + [_dp] * 4 + [_ip, ctypes.c_int]
        L.orc_seq_batch.restype = ctypes.c_int
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class NotPositiveDefinite(Exception):
    def __init__(self, index: int):
        super().__init__(f"not positive definite at {index}")
        self.index = index


# --- Table 1 block operations (SPEC.md:36-76 examples) --------------------

def potrf(d):
    a = _c(d).copy()
    rc = lib().orc_potrf(a.shape[0], _p(a))
    if rc:
        raise NotPositiveDefinite(rc)
    return a


def trsm_right(e, l):
    e = _c(e).copy()
    lib().orc_trsm_right(e.shape[0], e.shape[1], _p(e), _p(_c(l)))
    return e


def trsm_left(l, e):
    e = _c(e).copy()
    lib().orc_trsm_left(e.shape[0], e.shape[1], _p(e), _p(_c(l)))
    return e


def syrk_down(d, e, trans=False):
    d = _c(d).copy()
    e = _c(e)
    k = e.shape[0] if trans else e.shape[1]
    lib().orc_syrk_down(d.shape[0], k, _p(d), _p(e), int(trans))
    return d


def gemm_neg(a, b, c=None):
    a, b = _c(a), _c(b)
    out = np.zeros((a.shape[0], b.shape[1])) if c is None else _c(c).copy()
    lib().orc_gemm_neg(a.shape[0], a.shape[1], b.shape[1], _p(a), _p(b), _p(out), int(c is not None))
    return out


# --- Algorithm 1 and the sequential solve ---------------------------------------------------

def seq_factor(D, E):
    D = _c(D)
    N, n, _ = D.shape
    E = _c(E) if N > 1 else np.zeros((1, n, n))
    Dhat = np.zeros_like(D)
    Ehat = np.zeros((max(N - 1, 1), n, n))
    rc = lib().orc_seq_factor(N, n, _p(D), _p(E), _p(Dhat), _p(Ehat))
    if rc:
        raise NotPositiveDefinite(rc)
    return Dhat, Ehat[: N - 1]


def seq_solve(Dhat, Ehat, b):
    Dhat, b = _c(Dhat), _c(b)
    N, n, m = b.shape
    Ehat = _c(Ehat) if N > 1 else np.zeros((1, n, n))
    x = np.zeros_like(b)
    lib().orc_seq_solve(N, n, m, _p(Dhat), _p(Ehat), _p(b), _p(x))
    return x


def seq_batch(D, E, b, nthreads: int | None = None):
    """x for B independent systems (D [B,N,n,n], E [B,N-1,n,n], b [B,N,n,m]); returns (x, info)."""
    D, b = _c(D), _c(b)
    B, N, n, _ = D.shape
    m = b.shape[3]
    E = _c(E) if N > 1 else np.zeros((B, 1, n, n))
    x = np.zeros_like(b)
    info = np.zeros(B, dtype=np.int32)
    nt = nthreads or os.cpu_count() or 1
    lib().orc_seq_batch(B, N, n, m, _p(D), _p(E), _p(b), _p(x),
                        info.ctypes.data_as(_ip), int(nt))
    return x, info
