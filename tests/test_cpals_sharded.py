"""Row-sharded CP-ALS (paper_1902_03317_b200/cpals.py).

CPU (gloo, world_size 2): the exchange logic -- lambda all-reduce, owned
row-block all-gather, fit all-reduce -- with the oracle's fp64 MTTKRP as the
per-rank compute, against the same algorithm with G simulated ranks in one
process and against a plain numpy CP-ALS. GPU: the sm_100a kernels on
simulated G = 2, 3, 4 row shards against the single-GPU cp_als."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import HostTensor, Oracle


def _tensor(seed, dims, nnz):
    rng = np.random.default_rng(seed)
    lin = rng.choice(int(np.prod(dims)), size=nnz, replace=False)
    idx = []
    for d in reversed(dims):
        idx.append((lin % d).astype(np.uint32))
        lin //= d
    return HostTensor(dims, idx[::-1], rng.uniform(0, 1, nnz).astype(np.float32), None, True)


DIMS, R, NNZ, ITERS = [50, 40, 30], 6, 8000, 4


def _inputs():
    x = _tensor(11, DIMS, NNZ)
    rng = np.random.default_rng(12)
    init = [torch.from_numpy(rng.uniform(0, 1, (d, R)).astype(np.float32)) for d in DIMS]
    return x, init


def _sorted(x, mode):
    xs = x.copy()
    Oracle().sort_lexicographic(xs, [mode] + [d for d in range(x.order) if d != mode])
    return xs


def _oracle_mttkrp(O):
    return lambda s, f, n: torch.from_numpy(O.mttkrp(s, [u.numpy() for u in f], n)[1].copy())


def _run(world, ranks_obj, my_ranks):
    from paper_1902_03317_b200 import cpals
    x, init = _inputs()
    O = Oracle()
    shards, blocks = [], []
    for n in range(3):
        xs = _sorted(x, n)
        row = []
        for g in my_ranks:
            s, b = cpals.row_shard(xs, n, world, g)
            row.append(s)
        shards.append(row)
        blocks.append(b)
    return cpals.cp_als_rowsharded(shards, blocks, DIMS, R, ranks_obj, iters=ITERS, tol=0.0,
                                   init=init, mttkrp_fn=_oracle_mttkrp(O))


def _worker(rank, world, port, q):
    from paper_1902_03317_b200 import cpals
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _run(world, cpals.DistRanks(), [rank])
        q.put((rank, res.weights.numpy(), [u.numpy() for u in res.factors], res.fits))
    finally:
        dist.destroy_process_group()


def _np_cpals(x, init):
    O = Oracle()
    U = [u.numpy().astype(np.float64) for u in init]
    for _ in range(ITERS):
        for n in range(3):
            M = O.mttkrp(x, [u.astype(np.float32) for u in U], n)[1]
            V = np.ones((R, R))
            for m in range(3):
                if m != n:
                    V *= U[m].T @ U[m]
            Un = M @ np.linalg.pinv(V)
            lam = np.linalg.norm(Un, axis=0)
            lam[lam == 0] = 1
            U[n] = (Un / lam).astype(np.float32).astype(np.float64)
    return lam, U


def test_two_rank_gloo_matches_simulated_and_numpy():
    from paper_1902_03317_b200 import cpals
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (w, f, fits)) for r, w, f, fits in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sim = _run(2, cpals.SimRanks(2), [0, 1])
    x, init = _inputs()
    lam_ref, U_ref = _np_cpals(x, init)
    for r in (0, 1):
        w, f, fits = got[r]
        np.testing.assert_allclose(w, sim.weights.numpy(), rtol=1e-6)
        for a, b in zip(f, sim.factors):
            np.testing.assert_allclose(a, b.numpy(), rtol=1e-5, atol=1e-7)
        np.testing.assert_allclose(fits, sim.fits, rtol=1e-9)
    np.testing.assert_allclose(sim.weights.numpy(), lam_ref, rtol=1e-4)
    for a, b in zip(sim.factors, U_ref):
        np.testing.assert_allclose(a.numpy(), b, rtol=1e-3, atol=1e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 3, 4])
def test_gpu_rowsharded_matches_single_gpu(G):
    from paper_1902_03317_b200 import cpals, generate
    x = generate.coo([3000, 800, 500], 400_000, 21, [1.1, 0, 0], 0.0, 1.0)
    Rk = 16
    init = [generate.uniform((d, Rk), 21, 700 + k, 0.0, 1.0) for k, d in enumerate(x.dims)]
    single = cpals.cp_als(x, Rk, iters=5, tol=0.0, init=init)
    shards, blocks = [], []
    for n in range(3):
        xs = cpals.mode_sorted(x, n)
        row = []
        for g in range(G):
            s, b = cpals.row_shard(xs, n, G, g)
            row.append(s)
        shards.append(row)
        blocks.append(b)
    res = cpals.cp_als_rowsharded(shards, blocks, x.dims, Rk, cpals.SimRanks(G), iters=5,
                                  tol=0.0, init=init)
    torch.testing.assert_close(res.weights, single.weights, rtol=1e-5, atol=0)
    for a, b in zip(res.factors, single.factors):
        torch.testing.assert_close(a, b, rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(res.fits, single.fits, rtol=1e-6)
