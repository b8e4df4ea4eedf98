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
            # row-aligned shards + all-gather of the owned row blocks
            rr = parallel.row_aligned_ranges(xs.indices[mode], world)
            blocks = parallel.row_blocks(xs.indices[mode], rr, dims[mode])
            shard = parallel.slice_coo(xs, *rr[rank])
            got = parallel.mttkrp_row_allgather(shard, fs, mode, dims[mode], R, blocks, part_fn)
            out[f"mttkrp_ag{mode}"] = got.numpy()
        # TS / TEW-eq: no communication, shards concatenate in rank order
        lo, hi = parallel.shard_range(x.nnz, world, rank)
        z = O.ts(parallel.slice_coo(x, lo, hi), 2.5, 1)
        parts = [None] * world
        dist.all_gather_object(parts, z.values)
        out["ts"] = np.concatenate(parts)
        # TEW merge: key-range split
        # y has other dims (the output dims are the per-mode max): both key
        # layouts must use the common dims or matches would split across ranks
        y = _tensor(5, [70, 50, 33], 15000)
        xs, ys = x.copy(), y.copy()
        O.sort_lexicographic(xs, [0, 1, 2])
        O.sort_lexicographic(ys, [0, 1, 2])
        (xl, xh), (yl, yh) = parallel.tew_shards(xs, ys, [0, 1, 2], world)[rank]
        zr, _ = O.tew(parallel.slice_coo(xs, xl, xh), parallel.slice_coo(ys, yl, yh), 0)
        parts = [None] * world
        dist.all_gather_object(parts, (zr.indices, zr.values))
        out["tew_idx"] = [np.concatenate([p[0][d] for p in parts]) for d in range(3)]
        out["tew_val"] = np.concatenate([p[1] for p in parts])
        # TTV / TTM: fiber-aligned shards, outputs concatenated in rank order
        for mode in range(3):
            xs = x.copy()
            O.sort_lexicographic(xs, [d for d in range(3) if d != mode] + [mode])
            fptr = O.build_fiber_index(xs, mode)
            lo, hi, f_lo, f_hi = parallel.fiber_aligned_ranges(fptr, world)[rank]
            shard = parallel.slice_coo(xs, lo, hi)
            sf = parallel.fiber_shard_index(fptr, f_lo, f_hi)
            v = np.linspace(-1, 1, dims[mode]).astype(np.float32)
            u = np.linspace(-1, 1, dims[mode] * 3).astype(np.float32).reshape(dims[mode], 3)
            zv, _, _ = O.ttv(shard, v, mode, sf)
            zm, _, _ = O.ttm(shard, u, mode, sf)
            parts = [None] * world
            dist.all_gather_object(parts, (zv.indices, zv.values, zm.indices, zm.values))
            out[f"ttv{mode}"] = ([np.concatenate([p[0][d] for p in parts]) for d in range(2)],
                                 np.concatenate([p[1] for p in parts]))
            out[f"ttm{mode}"] = ([np.concatenate([p[2][d] for p in parts]) for d in range(3)],
                                 np.concatenate([p[3] for p in parts]))
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
        # row-aligned: every row is computed whole, in the same entry order, on
        # one rank -> identical to one process on the same mode-sorted tensor
        xs = x.copy()
        O.sort_lexicographic(xs, [mode] + [d for d in range(3) if d != mode])
        assert np.array_equal(out[f"mttkrp_ag{mode}"], O.mttkrp(xs, fs, mode)[1])
    assert np.array_equal(out["ts"].view(np.uint32), O.ts(x, 2.5, 1).values.view(np.uint32))
    for mode in range(3):  # fiber shards concatenate to the single-process output
        xs = x.copy()
        O.sort_lexicographic(xs, [d for d in range(3) if d != mode] + [mode])
        v = np.linspace(-1, 1, dims[mode]).astype(np.float32)
        u = np.linspace(-1, 1, dims[mode] * 3).astype(np.float32).reshape(dims[mode], 3)
        zv, _, _ = O.ttv(xs, v, mode)
        zm, _, _ = O.ttm(xs, u, mode)
        gi, gv = out[f"ttv{mode}"]
        assert all(np.array_equal(a, b) for a, b in zip(gi, zv.indices))
        assert np.array_equal(gv.view(np.uint32), zv.values.view(np.uint32))
        gi, gv = out[f"ttm{mode}"]
        assert all(np.array_equal(a, b) for a, b in zip(gi, zm.indices))
        assert np.array_equal(gv.view(np.uint32), zm.values.view(np.uint32))
    y = _tensor(5, [70, 50, 33], 15000)
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


def test_fiber_aligned_ranges():
    from paper_1902_03317_b200.parallel import fiber_aligned_ranges, fiber_shard_index
    rng = np.random.default_rng(3)
    for nf, world in ((100, 2), (100, 8), (3, 8), (1, 4)):
        lens = rng.integers(1, 50, nf)
        fptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
        rr = fiber_aligned_ranges(fptr, world)
        assert rr[0][0] == 0 and rr[-1][1] == fptr[-1] and rr[-1][3] == nf
        for (lo, hi, a, b), (lo2, _, a2, _) in zip(rr, rr[1:]):
            assert hi == lo2 and b == a2
        for lo, hi, a, b in rr:
            assert fptr[a] == lo and fptr[b] == hi  # cuts on fiber starts
            sf = fiber_shard_index(fptr, a, b)
            assert sf[0] == 0 and sf[-1] == hi - lo and len(sf) == b - a + 1


def test_row_aligned_ranges_and_blocks():
    from paper_1902_03317_b200.parallel import row_aligned_ranges, row_blocks
    rng = np.random.default_rng(7)
    for n_rows, nnz, world in ((50, 1000, 2), (50, 1000, 8), (1000, 37, 4), (5, 300, 8)):
        rows = np.sort(rng.zipf(1.3, nnz) % n_rows).astype(np.uint32)
        rr = row_aligned_ranges(rows, world)
        assert rr[0][0] == 0 and rr[-1][1] == nnz
        assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
        for lo, hi in rr:  # no row split across ranks
            if lo > 0 and lo < nnz:
                assert rows[lo] != rows[lo - 1]
        bl = row_blocks(rows, rr, n_rows)
        assert bl[0][0] == 0 and max(b for _, b in bl) == n_rows
        covered = sorted(b for b in bl if b[1] > b[0])
        assert all(a[1] == b[0] for a, b in zip(covered, covered[1:]))
        for (lo, hi), (a, b) in zip(rr, bl):  # every entry's row lies in its rank's block
            assert np.all((rows[lo:hi] >= a) & (rows[lo:hi] < b))
        # the in-place tensor search (device arrays) gives the same cuts
        t = torch.from_numpy(rows.astype(np.int32))
        assert row_aligned_ranges(t, world) == rr and row_blocks(t, rr, n_rows) == bl


def test_lower_bound_tuple_matches_packed_keys():
    """The per-mode narrowing search used to cut y at x's splitter tuples
    (device tensors in production; CPU tensors here) equals searchsorted on
    packed keys, for present, absent, smallest and largest tuples."""
    from types import SimpleNamespace
    from paper_1902_03317_b200 import parallel
    rng = np.random.default_rng(3)
    dims = [40, 30, 20]
    n = 5000
    idx = np.stack([rng.integers(0, d, n) for d in dims])
    order = [2, 0, 1]
    key = (idx[2].astype(np.int64) * 40 + idx[0]) * 30 + idx[1]
    perm = np.argsort(key, kind="stable")
    idx, key = idx[:, perm], key[perm]
    t = SimpleNamespace(indices=[torch.from_numpy(a.astype(np.int32)) for a in idx])
    probes = [tuple(int(idx[d][i]) for d in order) for i in (0, 17, n // 2, n - 1)]
    probes += [(0, 0, 0), (19, 39, 29), (7, 3, 29), (7, 4, 0)]
    for tup in probes:
        k = (tup[0] * 40 + tup[1]) * 30 + tup[2]
        assert parallel._lower_bound_tuple(t, order, tup) == int(np.searchsorted(key, k, "left"))
