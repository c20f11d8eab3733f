"""Multi-rank host logic on CPU (gloo, world_size 2): the symmetric super-tile
partition of K1 and the row shards of the sketch, emulated tile by tile in NumPy with
exactly the ownership / reduction rules the CUDA path uses (gauss_matvec.cu header,
krr_capi.cu precond_apply_dev), all-reduced over gloo and checked against the oracle.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _emulate_k1_rank(x, sigma, v, n, world, rank, krr):
    """This rank's local out vector: the partial sums of its owned super-tiles."""
    st, ns, tiles = krr.schedule(n, world, rank)
    n_pad = ns * st
    xp = np.zeros((n_pad, x.shape[1]))
    xp[:n] = x
    vp = np.zeros(n_pad)
    vp[:n] = v
    scale = 1.0 / (2.0 * sigma * sigma)
    part = np.zeros((ns, n_pad))
    written = np.zeros((ns, n_pad), dtype=bool)
    for a, b in tiles:
        ra = slice(a * st, (a + 1) * st)
        rb = slice(b * st, (b + 1) * st)
        d2 = ((xp[ra, None, :] - xp[None, rb, :]) ** 2).sum(-1)
        e = np.exp(-np.maximum(0.0, d2) * scale)
        if a == b:
            e = np.triu(e, 1)  # strictly above the diagonal; K_ii added by finish
            comb = e @ vp[rb] + e.T @ vp[ra]
            assert not written[a, ra].any()
            part[a, ra] = comb
            written[a, ra] = True
        else:
            assert not written[b, ra].any() and not written[a, rb].any()
            part[b, ra] = e @ vp[rb]        # row sums -> slot b of rows of a
            part[a, rb] = e.T @ vp[ra]      # column sums -> slot a of rows of b
            written[b, ra] = written[a, rb] = True
    # finish: sum the owned slots of each row in fixed order; rank 0 adds K_ii = 1
    out = np.zeros(n_pad)
    for i in range(n):
        y = i // st
        for s_ in range(ns):
            a, b = min(s_, y), max(s_, y)
            if any((a == ta and b == tb) for ta, tb in tiles):
                out[i] += part[s_, i]
    if rank == 0:
        out[:n] += vp[:n]
    return out[:n]


def _worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist
        sys.path.insert(0, str(ROOT))
        import paper_1611_03220_b200 as krr
        from oracle import oracle_ffi as oracle

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        n, d, sigma, lam = 700, 3, 1.3, 0.2
        x = oracle.random_matrix(n, d, 1)
        v = oracle.random_vector(n, 2)
        local = _emulate_k1_rank(x, sigma, v, n, world, rank, krr)
        t = torch.from_numpy(local.copy())
        dist.all_reduce(t)
        got = t.numpy() + lam * v
        want = oracle.kernel_matvec(x, sigma, lam, v)
        err1 = float(np.linalg.norm(got - want) / np.linalg.norm(want))

        # sketch row shards: W = sum_r U_r r_r (all-reduce), z rows then all-gather-by-sum
        z = oracle.random_matrix(n, 40, 3)
        u, _ = oracle.build_preconditioner(z, 0.1)
        r = oracle.random_vector(n, 4)
        z0, z1 = krr.shard_rows(n, world, rank)
        w = torch.from_numpy(u[:, z0:z1] @ r[z0:z1])
        dist.all_reduce(w)
        zz = np.zeros(n)
        zz[z0:z1] = (r[z0:z1] - u[:, z0:z1].T @ w.numpy()) / 0.1
        tz = torch.from_numpy(zz)
        dist.all_reduce(tz)
        want2 = oracle.precond_apply(u, 0.1, r)
        err2 = float(np.linalg.norm(tz.numpy() - want2) / np.linalg.norm(want2))
        dist.destroy_process_group()
        q.put((rank, err1, err2, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, None, repr(e)))


@pytest.mark.parametrize("world", [2])
def test_sharded_matvec_and_precond_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, e1, e2, err in results:
        assert err is None, err
        assert e1 <= 1e-13, (rank, e1)
        assert e2 <= 1e-12, (rank, e2)
