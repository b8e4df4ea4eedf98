"""Multi-rank host logic (paper_1902_03317_b200/parallel.py) with world_size 2
on CPU (gloo). The per-rank compute is the CPU oracle here (on the B200 box it
is the sm_100a kernel and the collective is NCCL); what is tested is the
sharding, the exchange step and that the combined result equals the
single-process result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import HostTensor, Oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tensor(seed, dims, nnz):
    rng = np.random.default_rng(seed)
    lin = rng.choice(int(np.prod(dims)), size=nnz, replace=False)
    idx = []
    for d in reversed(dims):
        idx.append((lin % d).astype(np.uint32))
        lin //= d
    return HostTensor(dims, idx[::-1], rng.uniform(0, 1, nnz).astype(np.float32), None, True)


def _worker(rank, world, port, q):
    from paper_1902_03317_b200 import parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O = Oracle()
    try:
        dims, R = [60, 50, 40], 16
        x = _tensor(3, dims, 20000)
        rng = np.random.default_rng(4)
        fs = [rng.uniform(0, 1, (d, R)).astype(np.float32) for d in dims]
        out = {}
        # MTTKRP: mode-sorted nnz shards + all-reduce of the partials
        for mode in range(3):
            xs = x.copy()
            O.sort_lexicographic(xs, [mode] + [d for d in range(3) if d != mode])
            lo, hi = parallel.shard_range(xs.nnz, world, rank)
            shard = parallel.slice_coo(xs, lo, hi)
            part_fn = lambda s, f, m: torch.from_numpy(O.mttkrp(s, f, m)[1].copy())  # fp64 partial
            got = parallel.mttkrp_allreduce(shard, fs, mode, dims[mode], R, part_fn)
            out[f"mttkrp{mode}"] = got.numpy()
        # TS / TEW-eq: no communication, shards concatenate in rank order
        lo, hi = parallel.shard_range(x.nnz, world, rank)
        z = O.ts(parallel.slice_coo(x, lo, hi), 2.5, 1)
        parts = [None] * world
        dist.all_gather_object(parts, z.values)
        out["ts"] = np.concatenate(parts)
        # TEW merge: key-range split
        y = _tensor(5, dims, 15000)
        xs, ys = x.copy(), y.copy()
        O.sort_lexicographic(xs, [0, 1, 2])
        O.sort_lexicographic(ys, [0, 1, 2])
        kx, ky = parallel.pack_keys(xs, [0, 1, 2]), parallel.pack_keys(ys, [0, 1, 2])
        (xl, xh), (yl, yh) = parallel.tew_key_ranges(kx, ky, world)[rank]
        zr, _ = O.tew(parallel.slice_coo(xs, xl, xh), parallel.slice_coo(ys, yl, yh), 0)
        parts = [None] * world
        dist.all_gather_object(parts, (zr.indices, zr.values))
        out["tew_idx"] = [np.concatenate([p[0][d] for p in parts]) for d in range(3)]
        out["tew_val"] = np.concatenate([p[1] for p in parts])
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O = Oracle()
    dims, R = [60, 50, 40], 16
    x = _tensor(3, dims, 20000)
    rng = np.random.default_rng(4)
    fs = [rng.uniform(0, 1, (d, R)).astype(np.float32) for d in dims]
    for mode in range(3):
        _, want, absum = O.mttkrp(x, fs, mode)
        got = out[f"mttkrp{mode}"]
        assert np.all(np.abs(got - want) <= 1e-12 * np.maximum(absum, 1e-300))
    assert np.array_equal(out["ts"].view(np.uint32), O.ts(x, 2.5, 1).values.view(np.uint32))
    y = _tensor(5, dims, 15000)
    z, _ = O.tew(x.copy(), y.copy(), 0)
    for d in range(3):
        assert np.array_equal(out["tew_idx"][d], z.indices[d])
    assert np.array_equal(out["tew_val"].view(np.uint32), z.values.view(np.uint32))


def test_shard_range_partitions():
    from paper_1902_03317_b200.parallel import shard_range
    for n in (0, 1, 7, 1000, 1001):
        for w in (1, 2, 3, 8):
            r = [shard_range(n, w, k) for k in range(w)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert max(h - l for l, h in r) - min(h - l for l, h in r) <= 1
