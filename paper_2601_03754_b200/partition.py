"""Partition permutation for one long system split over ranks (
PAPER.md:195-389, Algorithm 2, Proposition 1; reading R10).

p - 1 pivot blocks cut the N blocks into p chunks; rank k owns chunk k (and its left pivot
A_k). Each rank eliminates its chunk independently -- the parallel phase of Algorithm 2 -- with
the nested-dissection kernels (``btd_partition_local``: the chunk's border columns B_k, F_k^T
ride as extra right-hand sides), producing a fixed-size packet: its contributions to the
block-tridiagonal pivot system. One all-gather of the packets (NCCL: the only exchange step)
gives every rank the p packets; each rank factors and solves the (p-1)-block pivot system
redundantly (``btd_partition_reduce``, the sequential phase) and back-substitutes its chunk
(``btd_partition_finish``). All arithmetic runs in libbtd.so; this module holds the host logic:
chunk sizes, slicing of the global arrays, the exchange and the assembly of the solution.

The three library steps are reached through a ``backend`` object (default: the CUDA library);
the multi-process CPU tests pass a stand-in so that the host logic and the exchange can be run
with ``gloo`` on a machine without a GPU.
"""
from __future__ import annotations

import math

import torch


def chunk_sizes(N: int, p: int, rule: str = "equal") -> list[int]:
    """[N_1..N_p] with sum N_k = N - (p - 1).

    ``equal``: as even as possible (the chunks are processed concurrently by identical kernels);
    ``prop1``: Proposition 1: N_1*/N_k* = 19/7, N_k* rounded down and up,
    N_1 from the block count, the choice with the lower maximum of the phase costs of
    PAPER.md:315-321 ((7/3 N_1 - 1) n^3 vs (19/3 N_k - 1) n^3)."""
    if p < 1 or N < 2 * p - 1:
        raise ValueError(f"need N >= 2p - 1 blocks for p = {p} chunks (N = {N})")
    if p == 1:
        return [N]
    inner = N - (p - 1)
    if rule == "equal":
        q, r = divmod(inner, p)
        return [q + (1 if k < r else 0) for k in range(p)]
    if rule != "prop1":
        raise ValueError(rule)
    nk_star = (7 * N - 7 * p + 7) / (7 * p + 12)
    best = None
    for nk in sorted({math.floor(nk_star), math.ceil(nk_star)}):
        n1 = inner - (p - 1) * nk
        if nk < 1 or n1 < 1:
            continue
        cost = max(7 / 3 * n1 - 1, 19 / 3 * nk - 1)
        if best is None or cost < best[0]:
            best = (cost, [n1] + [nk] * (p - 1))
    return best[1]


def layout(sizes: list[int]):
    """(starts, pivots): 0-based first block of every chunk and 0-based index of every pivot
    (pivot q sits between chunk q and chunk q+1, 0-based)."""
    starts, pivots, i = [], [], 0
    for k, Nk in enumerate(sizes):
        starts.append(i)
        i += Nk
        if k < len(sizes) - 1:
            pivots.append(i)
            i += 1
    return starts, pivots


def _fresh(t: torch.Tensor) -> torch.Tensor:
    """A contiguous, 16-byte aligned copy when the view is not (the kernels use vector accesses)."""
    if t.is_contiguous() and t.data_ptr() % 16 == 0:
        return t
    return t.contiguous().clone()


def local_views(D: torch.Tensor, E: torch.Tensor, b: torch.Tensor, sizes: list[int], k: int) -> dict:
    """The data rank k (0-based chunk index) needs, sliced from one system's global arrays
    D [N, n, n], E [N-1, n, n], b [N, n, m]. Bk = Psi[D_1k, A_k] = E[piv_left],
    Fk = Psi[A_{k+1}, D_{N_k k}] = E[piv_right - 1], Ak = D[piv_left], ak = b[piv_left]."""
    starts, pivots = layout(sizes)
    s, Nk = starts[k], sizes[k]
    out = dict(D=_fresh(D[s:s + Nk]), E=_fresh(E[s:s + Nk - 1]), b=_fresh(b[s:s + Nk]), Bk=None, Fk=None,
               Ak=None, ak=None)
    if k > 0:
        pl = pivots[k - 1]
        out.update(Bk=_fresh(E[pl]), Ak=_fresh(D[pl]), ak=_fresh(b[pl]))
    if k < len(sizes) - 1:
        out.update(Fk=_fresh(E[pivots[k] - 1]))
    return out


def packet_len(n: int, m: int) -> int:
    return 3 * n * n + 2 * n * m


class CudaBackend:
    """The three library steps on the GPU (btd_partition_local / _reduce / _finish)."""

    def local(self, v: dict, n: int, m: int):
        from .btd import Plan, _check, _ptr, _stream, lib

        dev, dt = v["D"].device, v["D"].dtype
        Nk = v["D"].shape[0]
        mR = (n if v["Bk"] is not None else 0) + (n if v["Fk"] is not None else 0) + m
        plan = Plan(Nk, n, 1, mR, dt)
        R = torch.empty((Nk, n, mR), dtype=dt, device=dev)
        Y = torch.empty_like(R)
        Dhat = torch.empty((Nk, n, n), dtype=dt, device=dev)
        C = torch.empty((max(plan.num_coupling_blocks, 1), n, n), dtype=dt, device=dev)
        P = torch.empty(packet_len(n, m), dtype=dt, device=dev)
        info = torch.empty(1, dtype=torch.int32, device=dev)
        with torch.cuda.device(dev):
            _check(lib().btd_partition_local(plan.handle, _ptr(v["D"]), _ptr(v["E"]) if Nk > 1 else None,
                                             _ptr(v["Bk"]), _ptr(v["Fk"]), _ptr(v["Ak"]), _ptr(v["ak"]),
                                             _ptr(v["b"]), _ptr(R), _ptr(Dhat), _ptr(C), _ptr(Y), _ptr(P),
                                             _ptr(info), _stream(None, dev)), "btd_partition_local")
        return dict(plan=plan, Y=Y, Dhat=Dhat, C=C, info=info), P

    def reduce(self, packets: torch.Tensor, p: int, n: int, m: int):
        from .btd import Plan, _check, _ptr, _stream, lib

        dev, dt = packets.device, packets.dtype
        ps = Plan(p - 1, n, 1, m, dt)
        DS = torch.empty((p - 1, n, n), dtype=dt, device=dev)
        ES = torch.empty((max(p - 2, 1), n, n), dtype=dt, device=dev)
        bS = torch.empty((p - 1, n, m), dtype=dt, device=dev)
        DhS = torch.empty_like(DS)
        CS = torch.empty((max(ps.num_coupling_blocks, 1), n, n), dtype=dt, device=dev)
        xS = torch.empty_like(bS)
        infoS = torch.empty(1, dtype=torch.int32, device=dev)
        with torch.cuda.device(dev):
            _check(lib().btd_partition_reduce(ps.handle, p, _ptr(packets), _ptr(DS), _ptr(ES), _ptr(bS), _ptr(DhS),
                                              _ptr(CS), _ptr(xS), _ptr(infoS), _stream(None, dev)),
                   "btd_partition_reduce")
        return dict(DS=DS, ES=ES[:p - 2], bS=bS, DhatS=DhS, CS=CS[:ps.num_coupling_blocks], xS=xS, infoS=infoS)

    def finish(self, st: dict, xL, xR, n: int, m: int):
        from .btd import _check, _ptr, _stream, lib

        Y = st["Y"]
        x = torch.empty((Y.shape[0], n, m), dtype=Y.dtype, device=Y.device)
        with torch.cuda.device(Y.device):
            _check(lib().btd_partition_finish(st["plan"].handle, _ptr(Y), _ptr(xL), _ptr(xR), _ptr(x),
                                              _stream(None, Y.device)), "btd_partition_finish")
        return x


def solve(D: torch.Tensor, E: torch.Tensor, b: torch.Tensor, p: int, rule: str = "equal", group=None,
          backend=None):
    """x = Psi^{-1} b for ONE system (D [N,n,n], E [N-1,n,n], b [N,n,m]) by the partition method.

    group=None: all p chunks in this process, one after another (single GPU). With a
    torch.distributed group of size p: rank k runs chunk k, the packets are all-gathered, and
    every rank returns the full x (its own chunk from its back-substitution, the other chunks
    from an all-gather of the chunk solutions -- the latter only to hand back a complete x).
    Returns (x, info_dict)."""
    backend = backend or CudaBackend()
    N, n, _ = D.shape
    m = b.shape[2]
    sizes = chunk_sizes(N, p, rule)
    starts, pivots = layout(sizes)
    if p == 1:
        v = local_views(D, E, b, sizes, 0)
        st, _ = backend.local(v, n, m)
        return backend.finish(st, None, None, n, m), dict(sizes=sizes, info=[st["info"]])
    if group is None:
        states, pk = [], []
        for k in range(p):
            st, P = backend.local(local_views(D, E, b, sizes, k), n, m)
            states.append(st)
            pk.append(P)
        packets = torch.stack(pk)
        red = backend.reduce(packets, p, n, m)
        x = torch.empty_like(b)
        for k in range(p):
            xL = red["xS"][k - 1] if k > 0 else None
            xR = red["xS"][k] if k < p - 1 else None
            x[starts[k]:starts[k] + sizes[k]] = backend.finish(states[k], xL, xR, n, m)
        for q, piv in enumerate(pivots):
            x[piv] = red["xS"][q]
        return x, dict(sizes=sizes, info=[s["info"] for s in states] + [red["infoS"]], reduce=red)
    import torch.distributed as dist

    k = dist.get_rank(group)
    if dist.get_world_size(group) != p:
        raise ValueError("the process group must have exactly p ranks (one chunk per rank)")
    st, P = backend.local(local_views(D, E, b, sizes, k), n, m)
    parts = [torch.empty_like(P) for _ in range(p)]
    dist.all_gather(parts, P.contiguous(), group=group)                  # the exchange step
    packets = torch.stack(parts)
    red = backend.reduce(packets, p, n, m)
    xL = red["xS"][k - 1] if k > 0 else None
    xR = red["xS"][k] if k < p - 1 else None
    xk = backend.finish(st, xL, xR, n, m)
    # hand back the full x: gather the (unequal) chunk solutions, padded to the largest chunk
    width = max(sizes)
    pad = torch.zeros((width, n, m), dtype=xk.dtype, device=xk.device)
    pad[:sizes[k]] = xk
    allx = [torch.empty_like(pad) for _ in range(p)]
    dist.all_gather(allx, pad, group=group)
    x = torch.empty_like(b)
    for q in range(p):
        x[starts[q]:starts[q] + sizes[q]] = allx[q][:sizes[q]]
    for q, piv in enumerate(pivots):
        x[piv] = red["xS"][q]
    return x, dict(sizes=sizes, info=[st["info"], red["infoS"]], reduce=red, packets=packets)
