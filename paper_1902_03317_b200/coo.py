"""Device-resident COO store and its host mirror.

`DeviceCOO` is the B200 layout of the reference's `SparseTensorCOO<float>`
(P/include/spten/tensor.hpp:22-57): one u32 index array per mode
(structure-of-arrays, each a separate 16-byte-aligned HBM allocation, stored
as torch.int32 bit patterns), one fp32 value array, `dims`, the optional
`sort_order` and the `coalesced` flag. `HostCOO` is the same tensor in numpy
(what the reference holds in std::vectors) and is what crosses PCIe.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib


@dataclass
class HostCOO:
    """Host mirror of SparseTensorCOO<float> (numpy arrays)."""

    dims: list
    indices: list  # list of np.uint32 arrays, one per mode
    values: np.ndarray  # float32
    sort_order: Optional[list] = None
    coalesced: bool = False

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def copy(self) -> "HostCOO":
        return HostCOO(list(self.dims), [i.copy() for i in self.indices], self.values.copy(),
                       None if self.sort_order is None else list(self.sort_order), self.coalesced)

    def to_device(self, device: int | str | torch.device = 0, pin: bool = False) -> "DeviceCOO":
        dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)

        def up(a: np.ndarray) -> torch.Tensor:
            t = torch.from_numpy(np.ascontiguousarray(a))
            if pin:
                t = t.pin_memory()
            return t.to(dev, non_blocking=pin)

        return DeviceCOO(list(self.dims), [up(i.view(np.int32)) for i in self.indices],
                         up(self.values.astype(np.float32, copy=False)),
                         None if self.sort_order is None else list(self.sort_order),
                         self.coalesced)


@dataclass
class DeviceCOO:
    """Device-resident COO (SoA, u32 indices as int32 bit patterns, fp32 values)."""

    dims: list
    indices: list  # list of torch.int32 CUDA tensors
    values: torch.Tensor  # torch.float32 CUDA tensor
    sort_order: Optional[list] = None
    coalesced: bool = False
    _desc: Optional[_lib.SptCoo] = field(default=None, repr=False, compare=False)

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    @property
    def device(self) -> torch.device:
        return self.values.device

    @staticmethod
    def empty(dims: Sequence[int], nnz: int, device: torch.device | int = 0) -> "DeviceCOO":
        dev = torch.device("cuda", device) if isinstance(device, int) else device
        return DeviceCOO(list(dims), [torch.empty(nnz, dtype=torch.int32, device=dev)
                                      for _ in dims],
                         torch.empty(nnz, dtype=torch.float32, device=dev))

    def nbytes(self) -> int:
        return self.nnz * 4 * (self.order + 1)

    def descriptor(self) -> _lib.SptCoo:
        d = _lib.SptCoo()
        d.order = self.order
        d.nnz = self.nnz
        for m, e in enumerate(self.dims):
            d.dims[m] = int(e)
        for m, ix in enumerate(self.indices):
            d.idx[m] = ix.data_ptr() if ix.numel() else None
        d.val = self.values.data_ptr() if self.values.numel() else None
        if self.sort_order is not None:
            d.has_sort_order = 1
            for k, m in enumerate(self.sort_order):
                d.sort_order[k] = int(m)
        d.coalesced = 1 if self.coalesced else 0
        return d

    def adopt(self, d: _lib.SptCoo, nnz: Optional[int] = None) -> "DeviceCOO":
        """Take metadata written by the library into descriptor d."""
        self.dims = [int(d.dims[m]) for m in range(d.order)]
        self.sort_order = ([int(d.sort_order[k]) for k in range(d.order)]
                           if d.has_sort_order else None)
        self.coalesced = bool(d.coalesced)
        if nnz is not None and nnz != self.nnz:
            self.indices = [ix[:nnz] for ix in self.indices]
            self.values = self.values[:nnz]
        return self

    def to_host(self) -> HostCOO:
        return HostCOO(list(self.dims),
                       [ix.cpu().numpy().view(np.uint32).copy() for ix in self.indices],
                       self.values.cpu().numpy().copy(),
                       None if self.sort_order is None else list(self.sort_order),
                       self.coalesced)

    def clone(self) -> "DeviceCOO":
        return DeviceCOO(list(self.dims), [i.clone() for i in self.indices], self.values.clone(),
                         None if self.sort_order is None else list(self.sort_order),
                         self.coalesced)


@dataclass
class FiberIndex:
    """Mirror of spten::FiberIndex (P/include/spten/tensor.hpp:88-92) with
    device u32 offsets (fptr[0]==0, fptr[nfibs]==nnz)."""

    mode: int
    nfibs: int
    fptr: torch.Tensor  # int32 CUDA tensor, nfibs+1 entries (u32 bit patterns)


def ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None or t.numel() == 0 else t.data_ptr()


def byref(d: _lib.SptCoo):
    return ctypes.byref(d)
