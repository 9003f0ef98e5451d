"""Host logic of the partition path (paper_2601_03754_b200/partition.py) on CPU:
chunk sizes against Proposition 1 (oracle/partition.py), the slicing of the global arrays into
chunk/pivot/border blocks, and the multi-rank exchange (torch.distributed + gloo, world sizes 2
and 3) with the three library steps replaced by a dense host stand-in (test infrastructure:
plain numpy solves of the chunk systems). The end-to-end result must be the dense solution, so
a wrong slice, a wrong packet order or a misplaced pivot fails."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import btdgen
from oracle import dense
from oracle import partition as opart
from paper_2601_03754_b200 import partition as part


@pytest.mark.parametrize("N,p", [(100, 4), (1000, 8), (57, 3), (9, 5), (16, 2), (300, 7)])
def test_prop1_sizes_match_oracle(N, p):
    assert part.chunk_sizes(N, p, "prop1") == opart.chunk_sizes_prop1(N, p)
    eq = part.chunk_sizes(N, p, "equal")
    assert sum(eq) + p - 1 == N and max(eq) - min(eq) <= 1


def test_layout_matches_oracle_split():
    for sizes in ([3, 2, 2], [1, 1], [5], [46, 17, 17, 17]):
        chunks, pivots = opart.split(sizes)
        starts, piv0 = part.layout(sizes)
        assert [c[0] - 1 for c in chunks] == starts and [q - 1 for q in pivots] == piv0


def test_local_views_are_the_paper_blocks():
    """B_k = Psi[D_1k, A_k], F_k = Psi[A_{k+1}, D_{N_k k}], read off the dense Psi."""
    sizes = [3, 2, 4]
    N, n = sum(sizes) + 2, 2
    prob = btdgen.dd(1, N, n, m=1, seed=3)
    D, E, b = prob.D[0], prob.E[0], prob.b[0]
    A = dense.assemble(D.numpy(), E.numpy())
    chunks, pivots = opart.split(sizes)
    blk = lambda r, c: A[(r - 1) * n:r * n, (c - 1) * n:c * n]
    for k in range(3):
        v = part.local_views(D, E, b, sizes, k)
        assert v["D"].shape[0] == sizes[k]
        if k > 0:
            assert np.array_equal(v["Bk"].numpy(), blk(chunks[k][0], pivots[k - 1]))
            assert np.array_equal(np.tril(v["Ak"].numpy()), np.tril(blk(pivots[k - 1], pivots[k - 1])))
        else:
            assert v["Bk"] is None and v["Ak"] is None
        if k < 2:
            assert np.array_equal(v["Fk"].numpy(), blk(pivots[k], chunks[k][-1]))
        else:
            assert v["Fk"] is None


class DenseBackend:
    """Host stand-in for btd_partition_local / _reduce / _finish (same packet definition as
    include/btd.h), by dense numpy solves. Test infrastructure only."""

    def local(self, v, n, m):
        D, E, b = (v[k].double().numpy() for k in ("D", "E", "b"))
        Nk = D.shape[0]
        cols = []
        if v["Bk"] is not None:
            R = np.zeros((Nk, n, n)); R[0] = v["Bk"].double().numpy(); cols.append(R)
        if v["Fk"] is not None:
            R = np.zeros((Nk, n, n)); R[-1] = v["Fk"].double().numpy().T; cols.append(R)
        cols.append(b)
        R = np.concatenate(cols, axis=2)
        Y = np.linalg.solve(dense.assemble(D, E), R.reshape(Nk * n, -1)).reshape(Nk, n, -1)
        nb = n if v["Bk"] is not None else 0
        nf = n if v["Fk"] is not None else 0
        P = np.zeros(part.packet_len(n, m))
        nn = n * n
        if nb:
            Bk, Ak, ak = (v[k].double().numpy() for k in ("Bk", "Ak", "ak"))
            Al = np.tril(Ak) + np.tril(Ak, -1).T
            P[:nn] = (Al - Bk.T @ Y[0][:, :n]).ravel()
            P[3 * nn:3 * nn + n * m] = (ak - Bk.T @ Y[0][:, nb + nf:]).ravel()
        if nf:
            Fk = v["Fk"].double().numpy()
            P[nn:2 * nn] = (Fk @ Y[-1][:, nb:nb + n]).ravel()
            P[3 * nn + n * m:] = (Fk @ Y[-1][:, nb + nf:]).ravel()
            if nb:
                P[2 * nn:3 * nn] = (-Fk @ Y[-1][:, :n]).ravel()
        return dict(Y=Y, nb=nb, nf=nf, info=torch.zeros(1, dtype=torch.int32)), torch.from_numpy(P)

    def reduce(self, packets, p, n, m):
        Pk = packets.double().numpy()
        nn = n * n
        DS = np.stack([Pk[q + 1][:nn].reshape(n, n) - Pk[q][nn:2 * nn].reshape(n, n) for q in range(p - 1)])
        ES = np.stack([Pk[q + 1][2 * nn:3 * nn].reshape(n, n) for q in range(p - 2)]) if p > 2 else np.zeros((0, n, n))
        bS = np.stack([Pk[q + 1][3 * nn:3 * nn + n * m].reshape(n, m) - Pk[q][3 * nn + n * m:].reshape(n, m)
                       for q in range(p - 1)])
        xS = dense.solve(DS, ES, bS)
        return dict(DS=torch.from_numpy(DS), ES=torch.from_numpy(ES), xS=torch.from_numpy(xS),
                    infoS=torch.zeros(1, dtype=torch.int32))

    def finish(self, st, xL, xR, n, m):
        Y, nb, nf = st["Y"], st["nb"], st["nf"]
        x = Y[:, :, nb + nf:].copy()
        if nb:
            x -= Y[:, :, :nb] @ xL.double().numpy()
        if nf:
            x -= Y[:, :, nb:nb + nf] @ xR.double().numpy()
        return torch.from_numpy(x)


@pytest.mark.parametrize("sizes_rule,p", [("equal", 1), ("equal", 3), ("prop1", 4)])
def test_single_process_orchestration_with_dense_backend(sizes_rule, p):
    prob = btdgen.kalman(1, 41, 3, m=2, seed=5)
    D, E, b = prob.D[0], prob.E[0], prob.b[0]
    x, st = part.solve(D, E, b, p, rule=sizes_rule, backend=DenseBackend())
    xo = dense.solve(D.numpy(), E.numpy(), b.numpy())
    assert np.abs(x.numpy() - xo).max() <= 1e-10 * np.abs(xo).max()
    if p > 1:  # the pivot system is Algorithm 2's
        ref = opart.algorithm2(D.numpy(), E.numpy(), st["sizes"])
        for q in range(p - 1):
            assert np.allclose(np.tril(st["reduce"]["DS"][q].numpy()), np.tril(ref["S_diag"][q]), atol=1e-10)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = btdgen.kalman(1, 29, 2, m=1, seed=17)
    x, st = part.solve(prob.D[0], prob.E[0], prob.b[0], world, group=dist.group.WORLD, backend=DenseBackend())
    q.put((rank, x.numpy(), st["packets"].numpy(), st["sizes"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    prob = btdgen.kalman(1, 29, 2, m=1, seed=17)
    xo = dense.solve(prob.D[0].numpy(), prob.E[0].numpy(), prob.b[0].numpy())
    xs1, st1 = part.solve(prob.D[0], prob.E[0], prob.b[0], world, backend=DenseBackend())
    for rank, x, packets, sizes in res:
        assert np.abs(x - xo).max() <= 1e-10 * np.abs(xo).max(), rank
        assert sizes == st1["sizes"]
        assert np.array_equal(packets, res[0][2])   # every rank holds the same gathered packets
