"""Multi-GPU partitioning on one box (one process per GPU, torch.distributed).

SURVEY.md section 8(e):
  * MTTKRP shards naturally with ONE exchange step: contiguous equal-nnz
    ranges of the mode-n-sorted tensor go to the ranks, each rank computes a
    full dims[n] x R partial with the segmented kernel (rows outside its range
    come out zero-filled), and the partials are summed with an all-reduce --
    NCCL over NVLink/NVSwitch on the B200 box (the reference's only analogue
    is the private-buffer reduction of par::mttkrp, P/src/kernels_par.cpp:290-319).
  * TEW-eq and TS shard with no communication (contiguous nnz ranges; the
    output stays sharded, rank order = global order).
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


def pack_keys(t, order: Sequence[int]) -> np.ndarray:
    """Host u64 keys of a sorted tensor (sort-order significance); used only
    to choose key-range splitters (needs sum of index widths <= 64)."""
    widths = [max(1, int(np.ceil(np.log2(max(2, t.dims[d]))))) for d in order]
    if sum(widths) > 64:
        raise OverflowError("key-range split needs <= 64 key bits")
    key = np.zeros(len(t.values), np.uint64)
    for d, w in zip(order, widths):
        ix = t.indices[d]
        ix = ix.cpu().numpy() if isinstance(ix, torch.Tensor) else ix
        key = (key << np.uint64(w)) | ix.view(np.uint32).astype(np.uint64)
    return key


def tew_key_ranges(x_keys: np.ndarray, y_keys: np.ndarray, world: int) -> list:
    """Per-rank ((x_lo, x_hi), (y_lo, y_hi)): x cut at equal-nnz positions, y
    cut at the same keys, so matched tuples always land on the same rank."""
    cuts_x = [shard_range(len(x_keys), world, r)[0] for r in range(world)] + [len(x_keys)]
    split_keys = [x_keys[c] if c < len(x_keys) else np.uint64(np.iinfo(np.uint64).max)
                  for c in cuts_x[1:-1]]
    cuts_y = [0] + [int(np.searchsorted(y_keys, k, side="left")) for k in split_keys] + [len(y_keys)]
    return [((cuts_x[r], cuts_x[r + 1]), (cuts_y[r], cuts_y[r + 1])) for r in range(world)]
