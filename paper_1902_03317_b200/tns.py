"""`.tns` text ingest on the device: spten::read_tns<float>(path, dims)
(P/include/spten/io.hpp:14-23, P/src/io.cpp:42-120).

The file's bytes are read into pinned host memory (parallel preads, each
8 MB slice copied up as soon as it lands), and split, classified and parsed
on the GPU (spt_tns_scan / spt_tns_parse,
paper_1902_03317_b200/csrc/tns.cu). Same result as the reference (entries in
file order, dims = per-mode max + 1 unless overridden, unsorted and
uncoalesced) and the same errors: std::runtime_error with "path:line: msg"
becomes DeviceRuntimeError (a RuntimeError) with the same text; an empty
dims override is InvalidArgument (std::invalid_argument).
"""
from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor, as_completed
from typing import Optional, Sequence

import torch

from . import _lib
from .coo import DeviceCOO

__all__ = ["read_tns", "read_tns_bytes"]


_SLICE = 8 << 20  # bytes per read / copy slice


def _unpin():
    """A new thread inherits its creator's CPU mask: a caller whose OpenMP
    runtime pinned the main thread (OMP_PROC_BIND) would put every reader on
    that one core."""
    try:
        os.sched_setaffinity(0, range(os.cpu_count() or 1))
    except (OSError, AttributeError):
        pass


def _pool():
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1),
                                   thread_name_prefix="spt_tns_read", initializer=_unpin)
    return _POOL


_POOL = None


def _upload_file(path: str, dev: torch.device) -> torch.Tensor:
    """The file's bytes on `dev`: parallel preads into a pinned buffer, each
    8 MB slice copied up on a side stream as soon as it is read."""
    try:
        fd = os.open(path, os.O_RDONLY)
    except OSError:
        raise _lib.DeviceRuntimeError(f"read_tns: cannot open {path}") from None
    try:
        size = os.fstat(fd).st_size
        host = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        out = torch.empty(size, dtype=torch.uint8, device=dev)
        if not size:
            return out
        view = memoryview(host.numpy())

        def read(lo):
            hi = min(size, lo + _SLICE)
            got = lo
            while got < hi:
                n = os.preadv(fd, [view[got:hi]], got)
                if n <= 0:
                    return None
                got += n
            return lo

        copy = torch.cuda.Stream(dev)
        futs = [_pool().submit(read, lo) for lo in range(0, size, _SLICE)]
        with torch.cuda.stream(copy):
            for f in as_completed(futs):
                lo = f.result()
                if lo is None:
                    raise _lib.DeviceRuntimeError(f"read_tns: I/O error reading {path}")
                hi = min(size, lo + _SLICE)
                out[lo:hi].copy_(host[lo:hi], non_blocking=True)
        # out was allocated on the current stream, which now waits for the
        # copies; the pinned block's reuse is fenced by the copies' events
        torch.cuda.current_stream(dev).wait_stream(copy)
        return out
    finally:
        os.close(fd)


def read_tns_bytes(text: torch.Tensor, dims: Optional[Sequence[int]] = None,
                   device: int | torch.device = 0, name: str = "<text>") -> DeviceCOO:
    """Parse .tns text already in a uint8 tensor (host -- ideally pinned -- or
    on `device`); `name` stands in for the path in error messages."""
    dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
    if dev.type != "cuda":
        raise _lib.InvalidArgument("read_tns: needs a CUDA device (no CPU fallback)")
    if dims is not None and len(dims) == 0:
        raise _lib.InvalidArgument("read_tns: dims override must not be empty")
    ctx = _lib.Context.get(dev.index if dev.index is not None else 0)
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        d_text = text.to(dev, non_blocking=True) if text.device != dev else text
        d_text = d_text.contiguous()
        ov = None
        if dims is not None:
            ov = (ctypes.c_uint32 * len(dims))(*[int(e) for e in dims])
        scan = ctypes.c_void_p()
        order = ctypes.c_uint32()
        nnz = ctypes.c_uint64()
        line = ctypes.c_uint64()

        def fail(status):
            msg = lib.spt_last_error().decode("latin-1")
            exc = _lib._EXC.get(status, _lib.DeviceRuntimeError)
            if line.value:
                raise exc(f"{name}:{line.value}: {msg}")
            if status == _lib.SPT_ERUNTIME and "order is unknown" in msg:
                raise exc(f"read_tns: {name} {msg}")
            raise exc(msg)

        st = lib.spt_tns_scan(ctx.handle, d_text.data_ptr() if d_text.numel() else None,
                              d_text.numel(), ov, len(dims) if dims is not None else 0,
                              ctypes.byref(scan), ctypes.byref(order), ctypes.byref(nnz),
                              ctypes.byref(line), stream.cuda_stream)
        if st != _lib.SPT_OK:
            fail(st)
        try:
            n = int(nnz.value)
            z = DeviceCOO([0] * int(order.value),
                          [torch.empty(n, dtype=torch.int32, device=dev)
                           for _ in range(order.value)],
                          torch.empty(n, dtype=torch.float32, device=dev))
            d = z.descriptor()
            st = lib.spt_tns_parse(ctx.handle, scan, ctypes.byref(d), ctypes.byref(line),
                                   stream.cuda_stream)
            if st != _lib.SPT_OK:
                fail(st)
        finally:
            lib.spt_tns_destroy(scan)
        z.dims = [int(d.dims[m]) for m in range(d.order)]
        z.sort_order = None
        z.coalesced = False
        del d_text  # the parse synchronised the stream: the upload is consumed
    return z


def read_tns(path: str, dims: Optional[Sequence[int]] = None,
             device: int | torch.device = 0) -> DeviceCOO:
    """spten::read_tns<float>(path, dims) onto `device` (P/src/io.cpp:42-120)."""
    dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
    if dev.type != "cuda":
        raise _lib.InvalidArgument("read_tns: needs a CUDA device (no CPU fallback)")
    with torch.cuda.device(dev):
        text = _upload_file(path, dev)
    return read_tns_bytes(text, dims, dev, path)
