"""Multi-GPU schedule exercised on CPU with world_size 2
(torch.distributed gloo, 127.0.0.1): the 1D column-block-cyclic layout comes
from the C library's host functions (rqrcp_shard_columns /
rqrcp_shard_global_index); each rank holds its shard and runs the same
per-rank exchange as the CUDA driver (rqrcp.cu Run::panel / moves.cuh):
pivot columns packed full height and delivered to the panel owner by an
INTEGER-SUM reduce of their bit patterns (one contributor per element: exact),
the owner's panel QR and broadcast of V / tau / R11, the broadcast of the
owner's displaced slot columns to the move destinations, local trailing and
sample updates, the sample allgather -- with numpy arithmetic.  The result
must equal the single-process oracle: identical pivots, R and tau to rounding.
(The same driver runs on one B200 through the loopback transport in
tests/test_gpu_multirank.py, bitwise against P = 1.)
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _householder(x):
    """LAPACK dlarfg convention (reading R-G7)."""
    alpha = x[0]
    xn2 = float(np.dot(x[1:], x[1:]))
    v = np.zeros_like(x)
    v[0] = 1.0
    if xn2 == 0.0:
        return v, 0.0, alpha
    nrm = np.sqrt(alpha * alpha + xn2)
    beta = -nrm if alpha >= 0 else nrm
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def _perm_and_moves(piv, nb):
    """The transpositions j <-> piv[j] applied in order (reading R-G5) as the
    kernels leave them: perm[q] = original position of the column that ends at
    q (q < nb), and the (dst <- src) moves of every touched position."""
    where = {}
    for j in range(nb):
        s = int(piv[j])
        if s == j:
            continue
        a, b = where.get(j, j), where.get(s, s)
        where[j], where[s] = b, a
    perm = [where.get(q, q) for q in range(nb)]
    moves = [(d, s) for d, s in where.items() if d != s]
    return perm, moves


def _worker(rank, world, port, A, k, b, p, seed, out, P_layout=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1804_05138_b200 as rq
    m, n = A.shape
    P = world
    cols = [rq.shard_columns(n, b, P, r) for r in range(P)]
    mine = cols[rank]
    Al = np.array(A[:, mine], order="F")
    l = b + p
    Om = oracle.omega(seed, l, m)

    def owner(j):
        return (j // b) % P

    def local(j):
        return (j // (b * P)) * b + j % b

    def gather_global(Bloc, gcols):
        # all_gather of per-rank blocks (padded), then global order by the layout
        cmax = max(len(c) for c in gcols)
        buf = np.zeros((Bloc.shape[0], cmax))
        buf[:, :Bloc.shape[1]] = Bloc
        parts = [torch.zeros(Bloc.shape[0], cmax, dtype=torch.float64) for _ in range(P)]
        dist.all_gather(parts, torch.from_numpy(buf))
        allc = sorted((g, r, q) for r in range(P) for q, g in enumerate(gcols[r]))
        return np.stack([parts[r].numpy()[:, q] for g, r, q in allc], axis=1)

    # sketch: local columns, replicated sample in global order
    B = gather_global(oracle.sketch(Om, Al), cols)
    jpvt = np.arange(n)
    tau = np.zeros(k)
    i = 0
    while i < k:
        bb = min(b, k - i)
        q = oracle.sample_qrcp(B[:, i:], bb)           # replicated on every rank
        Rh = q["R"]                                     # transformed sample, pivoted order
        perm, moves = _perm_and_moves(q["piv"], bb)
        own = owner(i)
        # ---- (1) pack: the pivot columns this rank owns, full height, zeros
        #      elsewhere; (3) integer-sum reduce to the owner: exact bits ----
        pk = np.zeros((m, bb))
        for qq in range(bb):
            jg = i + perm[qq]
            if owner(jg) == rank:
                pk[:, qq] = Al[:, local(jg)]
        bits = torch.from_numpy(pk.view(np.int64).copy())
        dist.reduce(bits, own, op=dist.ReduceOp.SUM)
        Pbuf = bits.numpy().view(np.float64).copy() if rank == own else None
        # ---- (4) panel QR on the owner (unblocked Householder), broadcast ----
        pkv = torch.zeros(m - i + 1, bb, dtype=torch.float64)  # V (m-i rows) + tau row
        r11 = torch.zeros(bb, bb, dtype=torch.float64)
        if rank == own:
            for j in range(bb):
                v, t, beta = _householder(Pbuf[i + j:, j].copy())
                Pbuf[i + j, j] = beta
                Pbuf[i + j + 1:, j] = v[1:]
                for c in range(j + 1, bb):
                    Pbuf[i + j:, c] -= t * v * (v @ Pbuf[i + j:, c])
                pkv[j:m - i, j] = torch.from_numpy(v)
                pkv[m - i, j] = t
            r11[:] = torch.from_numpy(np.triu(Pbuf[i:i + bb, :bb]))
        dist.broadcast(pkv, own)
        dist.broadcast(r11, own)
        V = pkv[:m - i].numpy()
        tau[i:i + bb] = pkv[m - i].numpy()
        R11 = r11.numpy()
        # ---- (6) displaced: the owner's original slot columns go to the move
        #      destinations >= bb (fact (b): their sources are slots) ----
        disp = torch.zeros(m, bb, dtype=torch.float64)
        if rank == own:
            disp[:] = torch.from_numpy(Al[:, local(i):local(i) + bb].copy())
        dist.broadcast(disp, own)
        for d, s_ in moves:
            if d >= bb:
                assert s_ < bb
                if owner(i + d) == rank:
                    Al[:, local(i + d)] = disp.numpy()[:, s_]
        if rank == own:
            Al[:, local(i):local(i) + bb] = Pbuf
        jv = jpvt.copy()
        for d, s_ in moves:
            jpvt[i + d] = jv[i + s_]
        # ---- local trailing update (each reflector in order, like the oracle) ----
        tr = [q_ for q_, g in enumerate(mine) if g >= i + bb]
        for c in tr:
            for j in range(bb):
                Al[i + j:, c] -= tau[i + j] * V[j:, j] * (V[j:, j] @ Al[i + j:, c])
        # ---- local sample update (Eq. (4)), gathered in global order ----
        if i + bb < k:
            Bl = np.zeros((l, len(tr)))
            for e, c in enumerate(tr):
                pos = mine[c] - i
                x = np.linalg.solve(R11, Al[i:i + bb, c]) if bb > 0 else np.zeros(0)
                Bl[:bb, e] = Rh[:bb, pos] - np.triu(Rh[:bb, :bb]) @ x
                Bl[bb:, e] = Rh[bb:, pos]
            gcols = [[g for g in cols[r] if g >= i + bb] for r in range(P)]
            Bt = gather_global(Bl, gcols)
            B = np.zeros((l, n))
            B[:, i + bb:] = Bt
        i += bb
    # assemble the global factored matrix on rank 0
    gath = gather_global(Al, cols)
    if rank == 0:
        out.put((gath, jpvt, tau))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m,n,k,b,p", [(96, 90, 40, 8, 4), (120, 101, 45, 7, 3)])
def test_block_cyclic_schedule_matches_oracle(m, n, k, b, p):
    rng = np.random.default_rng(m + n)
    A = rng.standard_normal((m, n)) * np.exp(-np.arange(n) / 30.0)
    seed = 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, A, k, b, p, seed, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    gath, jpvt, tau = q.get(timeout=180)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    o = oracle.rqrcp(A, k, b, p, seed=seed)
    assert np.array_equal(jpvt, o["jpvt"])
    assert np.allclose(tau, o["tau"], rtol=0, atol=1e-13)
    R1, R2 = np.triu(gath[:k]), np.triu(o["A"][:k])
    assert np.max(np.abs(np.abs(np.diag(R1)) - np.abs(np.diag(R2)))) <= 1e-12 * np.abs(R2).max()
    assert np.max(np.abs(R1 - R2)) <= 1e-11 * np.abs(R2).max()


def test_layout_functions():
    """Layout host functions: a partition of the columns, block-cyclic, in order."""
    import paper_1804_05138_b200 as rq
    for n, b, P in [(10, 2, 2), (1000, 64, 8), (4097, 128, 3), (5, 7, 4)]:
        shards = [rq.shard_columns(n, b, P, r) for r in range(P)]
        allc = sorted(c for s in shards for c in s)
        assert allc == list(range(n))
        for r, s in enumerate(shards):
            assert s == sorted(s)
            assert all((c // b) % P == r for c in s)


def test_transposition_facts():
    """The two facts the pack / displaced exchange relies on (moves.cuh),
    brute force over random transposition sequences j <-> s_j, s_j >= j
    (reading R-G5): (a) slot q ends up holding the column from perm[q];
    (b) every touched position >= bb receives an original slot column."""
    rng = np.random.default_rng(0)
    for _ in range(2000):
        nn = int(rng.integers(1, 40))
        bb = int(rng.integers(1, nn + 1))
        piv = [int(rng.integers(j, nn)) for j in range(bb)]
        arr = list(range(nn))
        for j, s in enumerate(piv):
            arr[j], arr[s] = arr[s], arr[j]
        perm, moves = _perm_and_moves(piv, bb)
        assert perm == arr[:bb]
        for d, s in moves:
            assert arr[d] == s
            if d >= bb:
                assert s < bb
        touched = {d for d, _ in moves}
        assert all(arr[q] == q for q in range(nn) if q not in touched)
