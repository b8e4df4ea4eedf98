"""Host <-> device staging for callers that hold their tensors in host memory
(the reference's situation: SparseTensorCOO<float> lives in std::vectors).

`PinnedCOO` is a page-locked host mirror of a COO tensor; `Pipeline` owns
the CUDA streams (H2D copy, kernels -- a second kernel stream for work that
is independent of the first -- and D2H copy) so that, with chunked
uploads, PCIe host->device, the kernels and PCIe device->host all run at
once (PCIe is full duplex). Only copies live here; every kernel still goes
through `ops` / the C-ABI.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from .coo import DeviceCOO, HostCOO


def view(t: DeviceCOO, lo: int, hi: int) -> DeviceCOO:
    """Entries [lo, hi) of t as a DeviceCOO sharing t's storage. A slice of a
    sorted / coalesced tensor is still sorted / coalesced."""
    return DeviceCOO(list(t.dims), [i[lo:hi] for i in t.indices], t.values[lo:hi],
                     None if t.sort_order is None else list(t.sort_order), t.coalesced)


def chunk_bounds(n: int, chunks: int, align: int = 1024) -> list:
    """chunks+1 increasing offsets covering [0, n]; interior offsets are
    multiples of `align` so every chunk keeps the 16-byte vector paths."""
    b = [0]
    for c in range(1, chunks):
        b.append(max(b[-1], min(n, (n * c // chunks) // align * align)))
    b.append(n)
    return b


class PinnedCOO:
    """Page-locked host buffers for a COO tensor of up to `capacity` entries."""

    def __init__(self, dims: Sequence[int], capacity: int,
                 sort_order: Optional[list] = None, coalesced: bool = False):
        self.dims = list(dims)
        self.capacity = int(capacity)
        self.idx = [torch.empty(capacity, dtype=torch.int32).pin_memory() for _ in dims]
        self.val = torch.empty(capacity, dtype=torch.float32).pin_memory()
        self.sort_order = None if sort_order is None else list(sort_order)
        self.coalesced = coalesced
        self.nnz = 0

    @staticmethod
    def from_host(h: HostCOO) -> "PinnedCOO":
        p = PinnedCOO(h.dims, h.nnz, h.sort_order, h.coalesced)
        for a, b in zip(p.idx, h.indices):
            a.copy_(torch.from_numpy(np.ascontiguousarray(b).view(np.int32)))
        p.val.copy_(torch.from_numpy(np.ascontiguousarray(h.values, dtype=np.float32)))
        p.nnz = h.nnz
        return p

    def nbytes(self, lo: int, hi: int) -> int:
        return (hi - lo) * 4 * (len(self.dims) + 1)

    def upload(self, dst: DeviceCOO, lo: int, hi: int, stream: torch.cuda.Stream) -> int:
        """Async H2D of entries [lo, hi) into dst (same offsets) on `stream`."""
        with torch.cuda.stream(stream):
            for a, b in zip(self.idx, dst.indices):
                b[lo:hi].copy_(a[lo:hi], non_blocking=True)
            dst.values[lo:hi].copy_(self.val[lo:hi], non_blocking=True)
        return self.nbytes(lo, hi)

    def download(self, src: DeviceCOO, stream: torch.cuda.Stream, at: int = 0) -> int:
        """Async D2H of all of src into entries [at, at+src.nnz) on `stream`;
        takes src's dims / sort_order / coalesced."""
        lo, hi = at, at + src.nnz
        with torch.cuda.stream(stream):
            for a, b in zip(self.idx, src.indices):
                a[lo:hi].copy_(b, non_blocking=True)
            self.val[lo:hi].copy_(src.values, non_blocking=True)
        self.dims = list(src.dims)
        self.sort_order = None if src.sort_order is None else list(src.sort_order)
        self.coalesced = src.coalesced
        self.nnz = max(self.nnz, hi)
        return self.nbytes(lo, hi)

    def to_host(self) -> HostCOO:
        """numpy views of the first nnz entries (valid once the copies landed)."""
        n = self.nnz
        return HostCOO(list(self.dims), [a[:n].numpy().view(np.uint32) for a in self.idx],
                       self.val[:n].numpy(), self.sort_order, self.coalesced)


class Pipeline:
    """H2D / kernel / D2H streams on one device, joined to and from the
    caller's current stream by `begin()` / `end()`."""

    def __init__(self, device: int | torch.device = 0):
        self.device = torch.device("cuda", device) if isinstance(device, int) else device
        self.h2d = torch.cuda.Stream(self.device)
        self.cmp = torch.cuda.Stream(self.device)
        self.cmp2 = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)

    def begin(self) -> None:
        cur = torch.cuda.current_stream(self.device)
        for s in (self.h2d, self.cmp, self.cmp2, self.d2h):
            s.wait_stream(cur)

    def end(self) -> None:
        cur = torch.cuda.current_stream(self.device)
        for s in (self.h2d, self.cmp, self.cmp2, self.d2h):
            cur.wait_stream(s)

    @staticmethod
    def mark(stream: torch.cuda.Stream) -> torch.cuda.Event:
        ev = torch.cuda.Event()
        ev.record(stream)
        return ev
