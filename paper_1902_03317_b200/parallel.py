"""Multi-GPU partitioning on one box (one process per GPU, torch.distributed).

SURVEY.md section 8(e):
  * MTTKRP shards naturally with ONE exchange step: contiguous equal-nnz
    ranges of the mode-n-sorted tensor go to the ranks, each rank computes a
    full dims[n] x R partial with the segmented kernel (rows outside its range
    come out zero-filled), and the partials are summed with an all-reduce --
    NCCL over NVLink/NVSwitch on the B200 box (the reference's only analogue
    is the private-buffer reduction of par::mttkrp, P/src/kernels_par.cpp:290-319).
    A row-aligned variant (mttkrp_row_allgather) cuts the shards at row
    starts instead, so every output row is owned by exactly one rank and the
    exchange is an all-gather of the owners' row blocks: (G-1)/G of the output
    per rank instead of the all-reduce's 2(G-1)/G.
  * TEW-eq and TS shard with no communication (contiguous nnz ranges; the
    output stays sharded, rank order = global order).
  * TTV / TTM shard by fibers (fiber_aligned_ranges): a tensor sorted with
    the mode last is cut at the fiber start nearest below each equal-nnz
    point, every rank computes the output entries of its own fibers, and the
    outputs concatenate in rank order -- the single-process output, entry for
    entry (the fiber loops of par::ttv / par::ttm, P/src/kernels_par.cpp:
    199-212, :244-263, over rank-sized fiber ranges). No communication.
  * TEW (merge) shards by key range, the distributed form of
    par::partition_for_tew (P/src/kernels_par.cpp:93-142): splitter keys taken
    from x at equal-nnz positions, y cut at the same keys, each rank merges its
    pair of ranges, outputs concatenate in rank order.
The collective and the sharding logic are device-agnostic so the world_size-2
tests run them with the gloo backend on CPU (tests/test_parallel.py); on the
GPU the partial comes from the sm_100a kernel and the all-reduce is NCCL.
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple:
    """Contiguous, balanced [lo, hi) share of n items for `rank`."""
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def slice_coo(t, lo: int, hi: int):
    """View of entries [lo, hi) of a DeviceCOO/HostCOO-like tensor (same
    dims, sort order and coalesced flag: a contiguous range of a sorted,
    coalesced tensor is sorted and coalesced)."""
    return type(t)(list(t.dims), [ix[lo:hi] for ix in t.indices], t.values[lo:hi],
                   None if t.sort_order is None else list(t.sort_order), t.coalesced)


def mttkrp_allreduce(x_shard, factors: Sequence, mode: int, rows: int, rank_R: int,
                     partial_fn: Optional[Callable] = None, group=None) -> torch.Tensor:
    """Sum over ranks of the shard-local MTTKRP partials (rows x R).

    `partial_fn(x_shard, factors, mode) -> tensor` defaults to the segmented
    sm_100a kernel (ops.mttkrp); tests substitute the CPU oracle."""
    if partial_fn is None:
        from . import ops
        partial_fn = lambda xs, fs, m: ops.mttkrp(xs, fs, m, ops.MTTKRP_AUTO)  # noqa: E731
    part = partial_fn(x_shard, factors, mode)
    assert tuple(part.shape) == (rows, rank_R)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    return part


def pack_keys(t, order: Sequence[int], dims: Optional[Sequence[int]] = None) -> np.ndarray:
    """Host u64 keys of a sorted tensor (sort-order significance); used only
    to choose key-range splitters (needs sum of index widths <= 64). Two
    tensors whose keys are compared must be packed with the same `dims` --
    the TEW output dims, per-mode max (P/src/kernel_detail.hpp:97-102)."""
    dims = list(t.dims) if dims is None else list(dims)
    widths = [max(1, int(np.ceil(np.log2(max(2, dims[d]))))) for d in order]
    if sum(widths) > 64:
        raise OverflowError("key-range split needs <= 64 key bits")
    key = np.zeros(len(t.values), np.uint64)
    for d, w in zip(order, widths):
        ix = t.indices[d]
        ix = ix.cpu().numpy() if isinstance(ix, torch.Tensor) else ix
        key = (key << np.uint64(w)) | ix.view(np.uint32).astype(np.uint64)
    return key


def _lower_bound_tuple(t, order: Sequence[int], tup: Sequence[int]) -> int:
    """First entry of the sorted device tensor t whose tuple (in `order`
    significance) is >= tup: one searchsorted pair per mode on the narrowing
    range, nothing but a few scalars leaves the device."""
    lo, hi = 0, int(t.indices[0].shape[0])
    for d, v in zip(order, tup):
        if lo == hi:
            break
        a = t.indices[d][lo:hi]
        if v >= 1 << 31 or (a.dtype == torch.int32 and int(a[-1].item()) < 0):
            raise OverflowError("ids >= 2^31 in an int32 device array: split on the host")
        key = torch.tensor([v], dtype=a.dtype, device=a.device)
        l = int(torch.searchsorted(a, key, right=False).item())
        r = int(torch.searchsorted(a, key, right=True).item())
        if l == r:
            return lo + l
        lo, hi = lo + l, lo + r
    return lo


def tew_shards(x, y, order: Sequence[int], world: int) -> list:
    """Per-rank key-range shards of two sorted TEW operands: x cut at
    equal-nnz positions, y cut at the same tuples, so matched tuples always
    land on the same rank. Device tensors are searched in place (only the
    world-1 splitter tuples come to the host); host tensors, and device ids
    >= 2^31, go through packed u64 keys with the common (per-mode max) dims."""
    if isinstance(x.indices[0], torch.Tensor) and x.indices[0].is_cuda:
        try:
            nx, ny = len(x.values), len(y.values)
            cuts_x = [shard_range(nx, world, r)[0] for r in range(world)] + [nx]
            cuts_y = [0]
            for c in cuts_x[1:-1]:
                if c >= nx:
                    cuts_y.append(ny)
                    continue
                tup = [int(x.indices[d][c].item()) & 0xFFFFFFFF for d in order]
                cuts_y.append(_lower_bound_tuple(y, order, tup))
            cuts_y.append(ny)
            return [((cuts_x[r], cuts_x[r + 1]), (cuts_y[r], cuts_y[r + 1]))
                    for r in range(world)]
        except OverflowError:
            pass
    dims = [max(a, b) for a, b in zip(x.dims, y.dims)]
    return tew_key_ranges(pack_keys(x, order, dims), pack_keys(y, order, dims), world)


def tew_key_ranges(x_keys: np.ndarray, y_keys: np.ndarray, world: int) -> list:
    """Per-rank ((x_lo, x_hi), (y_lo, y_hi)): x cut at equal-nnz positions, y
    cut at the same keys, so matched tuples always land on the same rank."""
    cuts_x = [shard_range(len(x_keys), world, r)[0] for r in range(world)] + [len(x_keys)]
    split_keys = [x_keys[c] if c < len(x_keys) else np.uint64(np.iinfo(np.uint64).max)
                  for c in cuts_x[1:-1]]
    cuts_y = [0] + [int(np.searchsorted(y_keys, k, side="left")) for k in split_keys] + [len(y_keys)]
    return [((cuts_x[r], cuts_x[r + 1]), (cuts_y[r], cuts_y[r + 1])) for r in range(world)]


def _row_at(rows):
    """rows[i] as a Python int (u32 values stored in int32 device arrays)."""
    if isinstance(rows, torch.Tensor):
        return lambda i: int(rows[i].item()) & 0xFFFFFFFF
    a = np.asarray(rows)
    return lambda i: int(a[i]) & 0xFFFFFFFF


def _row_search(rows):
    """(i, right) -> first / one-past-last position of row rows[i]; device
    arrays are searched in place (1B-entry tensors stay on the GPU)."""
    if isinstance(rows, torch.Tensor):
        def f(i, right):
            v = rows[i:i + 1]
            if rows.dtype == torch.int32 and int(v.item()) < 0:
                raise OverflowError("row ids >= 2^31 in an int32 device array: search on the host")
            return int(torch.searchsorted(rows, v, right=right).item())
        return f
    a = np.asarray(rows)
    a = a.view(np.uint32) if a.dtype == np.int32 else a
    return lambda i, right: int(np.searchsorted(a, a[i], side="right" if right else "left"))


def row_aligned_ranges(rows, world: int) -> list:
    """Per-rank [lo, hi) entry ranges of a tensor sorted with the output mode
    leading (`rows` = its mode-n index array, non-decreasing), cut at the row
    start nearest below each equal-nnz point, so no row is split: a rank owns
    the rows its entries start. A row longer than nnz/world makes the cut fall
    back to that row's end (ranks may then be empty)."""
    find = _row_search(rows)
    n = len(rows)
    cuts = [0]
    for r in range(1, world):
        t = shard_range(n, world, r)[0]
        c = n if t >= n else find(t, False)
        if c <= cuts[-1]:  # the row at t started before the previous cut
            c = n if t >= n else find(t, True)
        cuts.append(max(c, cuts[-1]))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def row_blocks(rows, ranges: Sequence, n_rows: int) -> list:
    """Output row block [row_lo, row_hi) owned by each rank: from the first row
    of its entries to the first row of the next non-empty rank (rows without
    entries in between belong to the block that precedes them; they are zero
    in its partial)."""
    at = _row_at(rows)
    starts = [at(lo) if hi > lo else None for lo, hi in ranges]
    blocks, nxt = [None] * len(ranges), n_rows
    for r in range(len(ranges) - 1, -1, -1):
        if starts[r] is None:
            blocks[r] = (nxt, nxt)
        else:
            blocks[r] = (starts[r], nxt)
            nxt = starts[r]
    first = next((r for r in range(len(ranges)) if starts[r] is not None), None)
    if first is not None:
        blocks[first] = (0, blocks[first][1])
    return blocks


def fiber_aligned_ranges(fptr, world: int) -> list:
    """Per-rank [lo, hi) entry ranges of a tensor sorted with `mode` last,
    cut at fiber starts (fptr = build_fiber_index's nfibs+1 offsets): the
    first fiber start at or after each equal-nnz point, so no fiber is
    split. Returns [(lo, hi, f_lo, f_hi)]: entry range and fiber range."""
    f = fptr.cpu().numpy() if isinstance(fptr, torch.Tensor) else np.asarray(fptr)
    f = (f.view(np.uint32) if f.dtype == np.int32 else f).astype(np.int64)
    n, nf = int(f[-1]), len(f) - 1
    cuts = [0]
    for r in range(1, world):
        t = shard_range(n, world, r)[0]
        k = int(np.searchsorted(f, t, side="left"))  # first fiber starting at or after t
        cuts.append(max(min(k, nf), cuts[-1]))
    cuts.append(nf)
    return [(int(f[cuts[r]]), int(f[cuts[r + 1]]), cuts[r], cuts[r + 1]) for r in range(world)]


def fiber_shard_index(fptr, f_lo: int, f_hi: int):
    """The shard's own fiber index: fptr[f_lo..f_hi] rebased to 0."""
    if isinstance(fptr, torch.Tensor):
        f = fptr[f_lo:f_hi + 1].to(torch.int64) & 0xFFFFFFFF
        return (f - f[0]).to(fptr.dtype)
    f = np.asarray(fptr)[f_lo:f_hi + 1].astype(np.int64)
    return f - f[0]


def mttkrp_row_allgather(x_shard, factors: Sequence, mode: int, rows: int, rank_R: int,
                         blocks: Sequence, partial_fn: Optional[Callable] = None,
                         group=None) -> torch.Tensor:
    """MTTKRP over row-aligned shards: each rank's partial is exact on the rows
    it owns (`blocks[rank]`, from row_blocks), and one all-gather of the owned
    blocks (padded to the largest) assembles the full rows x R result on every
    rank. Same arithmetic per row as the single-process kernel (no cross-rank
    sums), half the all-reduce's exchange volume."""
    if partial_fn is None:
        from . import ops
        partial_fn = lambda xs, fs, m: ops.mttkrp(xs, fs, m, ops.MTTKRP_AUTO)  # noqa: E731
    part = partial_fn(x_shard, factors, mode)
    assert tuple(part.shape) == (rows, rank_R)
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return part
    world, me = dist.get_world_size(group), dist.get_rank(group)
    B = max(1, max(hi - lo for lo, hi in blocks))
    lo, hi = blocks[me]
    send = torch.zeros((B, rank_R), dtype=part.dtype, device=part.device)
    send[: hi - lo] = part[lo:hi]
    recv = torch.empty((world * B, rank_R), dtype=part.dtype, device=part.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    out = torch.empty_like(part)
    for r, (a, b) in enumerate(blocks):
        out[a:b] = recv[r * B: r * B + (b - a)]
    return out


def mttkrp_multi(x_sorted, factors_per_dev: Sequence[Sequence[torch.Tensor]], mode: int,
                 R: int) -> list:
    """Single-process multi-GPU MTTKRP through the C-ABI (spt_row_aligned_cuts
    + spt_mttkrp_f32_multi): x_sorted (mode leading) lives on device 0, its
    row-aligned shards are copied to the devices of `factors_per_dev`, every
    device gets the whole dims[mode] x R result. Returns the per-device outputs."""
    import ctypes
    from . import _lib
    from .coo import DeviceCOO
    lib = _lib.load()
    G = len(factors_per_dev)
    N = x_sorted.order
    ctx0 = _lib.Context.get(x_sorted.device.index or 0)
    cuts = (ctypes.c_uint64 * (G + 1))()
    rlo = (ctypes.c_uint32 * (G + 1))()
    d = x_sorted.descriptor()
    _lib.check(lib.spt_row_aligned_cuts(ctx0.handle, ctypes.byref(d), mode, G, cuts, rlo,
                                        torch.cuda.current_stream(x_sorted.device).cuda_stream))
    ctxs = (ctypes.c_void_p * G)()
    shards = (_lib.SptCoo * G)()
    fps = (ctypes.c_void_p * (G * N))()
    outs, streams, keep = [], (ctypes.c_void_p * G)(), []
    rows = (ctypes.c_uint64 * N)(*[x_sorted.dims[k] for k in range(N)])
    cols = (ctypes.c_uint64 * N)(*[R] * N)
    outp = (ctypes.c_void_p * G)()
    for k, fs in enumerate(factors_per_dev):
        dev = fs[0].device if fs[0] is not None else fs[1].device
        sh = slice_coo(x_sorted, int(cuts[k]), int(cuts[k + 1]))
        sh = DeviceCOO(list(sh.dims), [i.to(dev) for i in sh.indices], sh.values.to(dev),
                       list(sh.sort_order), True)
        keep.append(sh)
        ctxs[k] = _lib.Context.get(dev.index or 0).handle
        shards[k] = sh.descriptor()
        for j in range(N):
            fps[k * N + j] = fs[j].data_ptr() if (j != mode and fs[j] is not None) else None
        o = torch.empty((x_sorted.dims[mode], R), dtype=torch.float32, device=dev)
        outs.append(o)
        outp[k] = o.data_ptr()
        streams[k] = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(lib.spt_mttkrp_f32_multi(G, ctxs, shards, rlo, fps, rows, cols, mode, outp,
                                        streams))
    return outs
