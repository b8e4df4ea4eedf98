"""Host-side mirror of the reference's kernel entry points, on device tensors.

Same names, argument meaning and error behaviour as `spten::seq` / `spten::par`
(P/include/spten/kernels_seq.hpp:18-61, P/include/spten/kernels_par.hpp:35-72)
and the tensor helpers (P/include/spten/tensor.hpp:147-165); every call goes
through the C-ABI (include/spten_b200.h) to the sm_100a kernels. There is no
CPU path: without the built extension these functions raise.

Flop accounting mirrors spten::flops (P/src/flop_counter.cpp:8-15): each op
records the sequential reference's count (P/src/kernels_seq.cpp:37, 51, 65,
99, 144, 172).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import (ADD, DIV, MUL, SUB, SCALAR_ADD, SCALAR_MUL, MTTKRP_AUTO, MTTKRP_ATOMIC,
                   MTTKRP_SEGMENTED_CTA, MTTKRP_SEGMENTED_WARP,
                   MTTKRP_SEGMENTED, InvalidArgument, check)
from .coo import DeviceCOO, FiberIndex, ptr

__all__ = [
    "ADD", "SUB", "MUL", "DIV", "SCALAR_ADD", "SCALAR_MUL", "MTTKRP_AUTO", "MTTKRP_ATOMIC",
    "MTTKRP_SEGMENTED", "MTTKRP_SEGMENTED_CTA", "MTTKRP_SEGMENTED_WARP", "flops",
    "ascending_order", "mode_last_order", "check_deferred", "ts", "tew_eq", "tew", "ttv",
    "ttm", "mttkrp", "mttkrp_plan", "MttkrpPlan", "sort_lexicographic", "coalesce", "build_fiber_index",
]


class _Flops:
    """spten::flops::{reset,count,record} (P/include/spten/flop_counter.hpp:8-14)."""

    def __init__(self):
        self._n = 0

    def reset(self) -> None:
        self._n = 0

    def count(self) -> int:
        return self._n

    def record(self, n: int) -> None:
        self._n += int(n)


flops = _Flops()


def ascending_order(n: int) -> list:
    """P/src/tensor.cpp:11-15"""
    return list(range(n))


def mode_last_order(n: int, mode: int) -> list:
    """P/src/tensor.cpp:17-24"""
    return [d for d in range(n) if d != mode] + [mode]


def _ctx(t: DeviceCOO | torch.Tensor):
    dev = t.device if isinstance(t, DeviceCOO) else t.device
    if dev.type != "cuda":
        raise InvalidArgument("spten_b200 ops need CUDA tensors (no CPU fallback)")
    return _lib.Context.get(dev.index if dev.index is not None else 0)


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _check_vec(t: torch.Tensor, device, who: str, name: str, ndim: int) -> None:
    """Dense operands handed to the C-ABI as raw pointers: contiguous float32
    on the tensor's device with the expected rank."""
    if (not isinstance(t, torch.Tensor) or t.dim() != ndim or t.dtype != torch.float32
            or not t.is_contiguous() or t.device != device):
        raise InvalidArgument(f"{who}: {name} must be a contiguous {ndim}-D float32 tensor on "
                              f"{device}")


def _check_out_coo(z: DeviceCOO, order: int, nnz: int, device, who: str) -> None:
    """A caller-provided output COO must hold `nnz` entries of `order` modes on
    the device (the C side writes through its raw pointers)."""
    if z.order != order or z.nnz < nnz or z.device != device or any(
            ix.numel() < nnz or ix.dtype != torch.int32 or not ix.is_contiguous()
            for ix in z.indices) or z.values.dtype != torch.float32 \
            or not z.values.is_contiguous():
        raise InvalidArgument(f"{who}: out must be an order-{order} DeviceCOO with room for "
                              f"{nnz} entries on {device}")


def _flags(sync: bool) -> int:
    return 0 if sync else _lib.SPT_FLAG_ASYNC


def check_deferred(device: int | torch.device = 0) -> None:
    """Raise the first data-dependent error of earlier sync=False calls on this
    device (synchronises torch's current stream; spt_ctx_check)."""
    dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
    ctx = _lib.Context.get(dev.index if dev.index is not None else 0)
    check(_lib.load().spt_ctx_check(ctx.handle, _stream(dev)))


# ---------------------------------------------------------------------------
# TS (P/src/kernels_seq.cpp:55-67)


def ts(x: DeviceCOO, s: float, op: int, out: Optional[DeviceCOO] = None,
       sync: bool = True) -> DeviceCOO:
    ctx = _ctx(x)
    if out is not None:
        _check_out_coo(out, x.order, x.nnz, x.device, "ts")
    z = out if out is not None else DeviceCOO.empty(x.dims, x.nnz, x.device)
    xd, zd = x.descriptor(), z.descriptor()
    check(_lib.load().spt_ts_f32(ctx.handle, ctypes.byref(xd), float(s), int(op),
                                 ctypes.byref(zd), _flags(sync), _stream(x.device)))
    z.adopt(zd)
    flops.record(x.nnz)
    return z


# ---------------------------------------------------------------------------
# TEW-eq (P/src/kernels_seq.cpp:11-39)


def tew_eq(x: DeviceCOO, y: DeviceCOO, op: int, out: Optional[DeviceCOO] = None,
           sync: bool = True) -> DeviceCOO:
    ctx = _ctx(x)
    if out is not None:
        _check_out_coo(out, x.order, x.nnz, x.device, "tew_eq")
    z = out if out is not None else DeviceCOO.empty(x.dims, x.nnz, x.device)
    xd, yd, zd = x.descriptor(), y.descriptor(), z.descriptor()
    check(_lib.load().spt_tew_eq_f32(ctx.handle, ctypes.byref(xd), ctypes.byref(yd), int(op),
                                     ctypes.byref(zd), _flags(sync), _stream(x.device)))
    z.adopt(zd)
    flops.record(x.nnz)
    return z


# ---------------------------------------------------------------------------
# Preprocessing (P/src/tensor.cpp:54-120)


def sort_lexicographic(t: DeviceCOO, mode_order: Sequence[int], sync: bool = True) -> None:
    """In-place stable lexicographic sort; sets t.sort_order (P/src/tensor.cpp:54-64)."""
    ctx = _ctx(t)
    mo = list(mode_order)
    if len(mo) != t.order:
        raise InvalidArgument("sort_lexicographic: mode order has wrong length")
    if sorted(mo) != list(range(t.order)):
        raise InvalidArgument("sort_lexicographic: mode order is not a permutation")
    arr = (ctypes.c_uint32 * t.order)(*mo)
    d = t.descriptor()
    check(_lib.load().spt_sort_f32(ctx.handle, ctypes.byref(d), arr, _flags(sync),
                                   _stream(t.device)))
    t.sort_order = mo


def coalesce(t: DeviceCOO) -> DeviceCOO:
    """Merge duplicate tuples by summation in storage order (P/src/tensor.cpp:66-90).
    Like the reference, an unsorted input is sorted (on a copy) ascending first."""
    ctx = _ctx(t)
    src = t
    if t.sort_order is None:
        src = t.clone()
        sort_lexicographic(src, ascending_order(t.order))
    z = DeviceCOO.empty(t.dims, t.nnz, t.device)
    sd, zd = src.descriptor(), z.descriptor()
    n = ctypes.c_uint64(0)
    check(_lib.load().spt_coalesce_f32(ctx.handle, ctypes.byref(sd), ctypes.byref(zd),
                                       ctypes.byref(n), None, 0, _stream(t.device)))
    return z.adopt(zd, int(n.value))


def build_fiber_index(t: DeviceCOO, mode: int) -> FiberIndex:
    """P/src/tensor.cpp:92-120; fptr as device u32 offsets."""
    ctx = _ctx(t)
    if mode >= t.order:
        raise InvalidArgument("build_fiber_index: mode out of range")
    if t.sort_order is None or t.sort_order[-1] != mode:
        raise InvalidArgument(
            "build_fiber_index: tensor must be sorted with the target mode as the last key")
    fptr = torch.empty(t.nnz + 1, dtype=torch.int32, device=t.device)
    n = ctypes.c_uint64(0)
    d = t.descriptor()
    check(_lib.load().spt_fiber_index(ctx.handle, ctypes.byref(d), int(mode), fptr.data_ptr(),
                                      ctypes.byref(n), None, 0, _stream(t.device)))
    nf = int(n.value)
    return FiberIndex(mode, nf, fptr[: nf + 1])


# ---------------------------------------------------------------------------
# TEW (P/src/kernels_seq.cpp:41-53, P/src/kernel_detail.hpp:36-102)


def tew_device(x: DeviceCOO, y: DeviceCOO, op: int, out: DeviceCOO,
               d_count: torch.Tensor) -> DeviceCOO:
    """Stream-ordered TEW for the device-resident path: x and y must already
    share a sort order; `out` has capacity nnz_x+nnz_y (mul: min); the output
    count lands in d_count (int64 CUDA scalar) without a host sync."""
    ctx = _ctx(x)
    cap = out.nnz
    xd, yd, zd = x.descriptor(), y.descriptor(), out.descriptor()
    check(_lib.load().spt_tew_f32(ctx.handle, ctypes.byref(xd), ctypes.byref(yd), int(op),
                                  ctypes.byref(zd), cap, None, d_count.data_ptr(),
                                  _lib.SPT_FLAG_ASYNC, _stream(x.device)))
    out.adopt(zd)
    return out


def tew(x: DeviceCOO, y: DeviceCOO, op: int, out: Optional[DeviceCOO] = None) -> DeviceCOO:
    """General elementwise op by sorted merge. Like the reference, sorts both
    operands ascending *in place* unless they already share a sort order."""
    ctx = _ctx(x)
    if op == DIV:
        raise InvalidArgument(
            "tew: div is not defined for mismatched patterns (unmatched entries divide by zero)")
    if x.order != y.order:
        raise InvalidArgument("tew: tensors must have the same order")
    if not (x.coalesced and y.coalesced):
        raise InvalidArgument("tew: both inputs must be coalesced")
    if not (x.sort_order is not None and y.sort_order is not None
            and list(x.sort_order) == list(y.sort_order)):
        order = ascending_order(x.order)
        sort_lexicographic(x, order)
        sort_lexicographic(y, order)
    cap = x.nnz + y.nnz if op != MUL else min(x.nnz, y.nnz)
    dims = [max(a, b) for a, b in zip(x.dims, y.dims)]
    if out is not None:
        _check_out_coo(out, x.order, cap, x.device, "tew")
    z = out if out is not None else DeviceCOO.empty(dims, max(cap, 0), x.device)
    xd, yd, zd = x.descriptor(), y.descriptor(), z.descriptor()
    n = ctypes.c_uint64(0)
    check(_lib.load().spt_tew_f32(ctx.handle, ctypes.byref(xd), ctypes.byref(yd), int(op),
                                  ctypes.byref(zd), cap, ctypes.byref(n), None, 0,
                                  _stream(x.device)))
    nz = int(n.value)
    z.adopt(zd, nz)
    # matches + sub negations (P/src/kernel_detail.hpp:55-83)
    flops.record({ADD: x.nnz + y.nnz - nz, SUB: y.nnz, MUL: nz}[op])
    return z


# ---------------------------------------------------------------------------
# TTV / TTM (P/src/kernels_seq.cpp:69-151)


def _precheck(x: DeviceCOO, mode: int, kernel: str) -> None:
    # P/src/kernel_detail.hpp:110-115
    if x.order < 2:
        raise InvalidArgument(f"{kernel}: input must have order >= 2")
    if mode >= x.order:
        raise InvalidArgument(f"{kernel}: mode out of range")
    if not x.coalesced:
        raise InvalidArgument(f"{kernel}: tensor must be coalesced")
    if x.sort_order is None or x.sort_order[-1] != mode:
        raise InvalidArgument(f"{kernel}: tensor must be sorted with the target mode last")


def _fiber_checks(x: DeviceCOO, mode: int, fib: FiberIndex, kernel: str) -> None:
    # P/src/kernel_detail.hpp:106-119
    _precheck(x, mode, kernel)
    if fib.mode != mode or fib.fptr.numel() != fib.nfibs + 1:
        raise InvalidArgument(f"{kernel}: fiber index does not match the tensor")


def ttv(x: DeviceCOO, v: torch.Tensor, mode: int, fib: Optional[FiberIndex] = None,
        out: Optional[DeviceCOO] = None) -> DeviceCOO:
    ctx = _ctx(x)
    if fib is None:
        _precheck(x, mode, "ttv")
        fib = build_fiber_index(x, mode)
    _fiber_checks(x, mode, fib, "ttv")
    _check_vec(v, x.device, "ttv", "v", 1)
    dims = [e for d, e in enumerate(x.dims) if d != mode]
    if out is not None:
        _check_out_coo(out, x.order - 1, fib.nfibs, x.device, "ttv")
    z = out if out is not None else DeviceCOO.empty(dims, fib.nfibs, x.device)
    xd, zd = x.descriptor(), z.descriptor()
    check(_lib.load().spt_ttv_f32(ctx.handle, ctypes.byref(xd), ptr(v), v.numel(), int(mode),
                                  fib.fptr.data_ptr(), fib.nfibs, ctypes.byref(zd), 0,
                                  _stream(x.device)))
    z.adopt(zd)
    flops.record(2 * x.nnz)
    return z


def ttm(x: DeviceCOO, u: torch.Tensor, mode: int, fib: Optional[FiberIndex] = None,
        out: Optional[DeviceCOO] = None) -> DeviceCOO:
    ctx = _ctx(x)
    _check_vec(u, x.device, "ttm", "u", 2)
    if fib is None:
        _precheck(x, mode, "ttm")
        fib = build_fiber_index(x, mode)
    _fiber_checks(x, mode, fib, "ttm")
    R = int(u.shape[1])
    dims = list(x.dims)
    dims[mode] = R
    if out is not None:
        _check_out_coo(out, x.order, fib.nfibs * R, x.device, "ttm")
    z = out if out is not None else DeviceCOO.empty(dims, fib.nfibs * R, x.device)
    xd, zd = x.descriptor(), z.descriptor()
    check(_lib.load().spt_ttm_f32(ctx.handle, ctypes.byref(xd), ptr(u), int(u.shape[0]), R,
                                  int(mode), fib.fptr.data_ptr(), fib.nfibs, ctypes.byref(zd), 0,
                                  _stream(x.device)))
    z.adopt(zd)
    flops.record(2 * R * x.nnz)
    return z


# ---------------------------------------------------------------------------
# MTTKRP (P/src/kernels_seq.cpp:153-174, P/src/kernels_par.cpp:275-337)


def _check_factors(x: DeviceCOO, factors, mode: int, who: str = "mttkrp"):
    """Factor matrices for the C-ABI: contiguous 2-D float32 on x's device
    (P/src/kernel_detail.hpp:163-173 checks the shapes; the C side checks
    them again)."""
    N = x.order
    if len(factors) != N:
        raise InvalidArgument(f"{who}: need one factor matrix per mode")
    fp = (ctypes.c_void_p * N)()
    rows = (ctypes.c_uint64 * N)()
    cols = (ctypes.c_uint64 * N)()
    R = 0
    for d, f in enumerate(factors):
        if d == mode or f is None:
            continue
        if (f.dim() != 2 or f.dtype != torch.float32 or not f.is_contiguous()
                or f.device != x.device):
            raise InvalidArgument(f"{who}: factors must be contiguous 2-D float32 tensors on "
                                  f"{x.device}")
        fp[d] = ptr(f)
        rows[d] = int(f.shape[0])
        cols[d] = int(f.shape[1])
        R = R or int(f.shape[1])
    return fp, rows, cols, R


def _check_out(out: torch.Tensor, shape, device, who: str) -> None:
    if (tuple(out.shape) != tuple(shape) or out.dtype != torch.float32
            or not out.is_contiguous() or out.device != device):
        raise InvalidArgument(f"{who}: out must be a contiguous float32 {tuple(shape)} tensor "
                              f"on {device}")


class MttkrpPlan:
    """Preprocessed MTTKRP input (spt_mttkrp_plan_create): a copy of x sorted
    with `mode` leading and the other modes by decreasing extent, whose most
    gathered factor rows are served from shared memory. Built once (timed as
    preprocessing, like the reference's sort_s, P/src/bench.cpp:363-368);
    `mttkrp(plan, factors, mode)` then runs it with any factor values."""

    def __init__(self, x: DeviceCOO, mode: int, R: int, hot: bool = True):
        ctx = _ctx(x)
        self.device, self.mode, self.R, self.dims, self.order = x.device, mode, R, list(x.dims), x.order
        self.nnz = x.nnz
        flags = 0 if hot else _lib.SPT_PLAN_NO_HOT
        h = ctypes.c_void_p()
        d = x.descriptor()
        check(_lib.load().spt_mttkrp_plan_create(ctx.handle, ctypes.byref(d), int(mode), int(R),
                                                 flags, ctypes.byref(h), _stream(x.device)))
        self.handle = h
        lm = (ctypes.c_uint32 * max(x.order - 1, 1))()
        hp = (ctypes.c_uint32 * max(x.order - 1, 1))()
        nh = ctypes.c_uint32()
        check(_lib.load().spt_mttkrp_plan_info(h, lm, hp, ctypes.byref(nh)))
        self.level_modes = list(lm)[: x.order - 1]
        self.hot_per_level = list(hp)[: x.order - 1]
        self.nhot = int(nh.value)

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.load().spt_mttkrp_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mttkrp_plan(x: DeviceCOO, mode: int, R: int, hot: bool = True) -> MttkrpPlan:
    return MttkrpPlan(x, mode, R, hot=hot)


def mttkrp(x, factors: Sequence[Optional[torch.Tensor]], mode: int,
           strategy: int = MTTKRP_AUTO, out: Optional[torch.Tensor] = None,
           sync: bool = True) -> torch.Tensor:
    """Returns the dims[mode] x R row-major fp32 result on the device.
    factors[mode] is ignored (may be None), as in the reference. x is a
    DeviceCOO (any order: AUTO plans a sorted copy, P/src/kernels_seq.cpp:
    153-174 accepts any order) or an MttkrpPlan."""
    if isinstance(x, MttkrpPlan):
        return _mttkrp_plan_exec(x, factors, mode, out, sync)
    ctx = _ctx(x)
    N = x.order
    if N < 2:
        raise InvalidArgument("mttkrp: input must have order >= 2")
    if mode >= N:
        raise InvalidArgument("mttkrp: mode out of range")
    fp, rows, cols, R = _check_factors(x, factors, mode)
    I = x.dims[mode]
    if out is None:
        out = torch.empty((I, max(R, 1) if R else 0), dtype=torch.float32, device=x.device)
    else:
        _check_out(out, (I, R), x.device, "mttkrp")
    xd = x.descriptor()
    check(_lib.load().spt_mttkrp_f32(ctx.handle, ctypes.byref(xd), fp, rows, cols, int(mode),
                                     ptr(out), int(strategy), _flags(sync), _stream(x.device)))
    flops.record(x.nnz * N * R)
    return out


def _mttkrp_plan_exec(plan: MttkrpPlan, factors, mode: int, out, sync: bool) -> torch.Tensor:
    if mode != plan.mode:
        raise InvalidArgument(f"mttkrp: plan was built for mode {plan.mode}, not {mode}")
    ctx = _lib.Context.get(plan.device.index if plan.device.index is not None else 0)

    class _X:  # shape/device stand-in for _check_factors
        order, device = plan.order, plan.device
    fp, rows, cols, R = _check_factors(_X, factors, mode)
    I = plan.dims[mode]
    if out is None:
        out = torch.empty((I, plan.R), dtype=torch.float32, device=plan.device)
    else:
        _check_out(out, (I, plan.R), plan.device, "mttkrp")
    check(_lib.load().spt_mttkrp_plan_exec(ctx.handle, plan.handle, fp, rows, cols, ptr(out),
                                           _flags(sync), _stream(plan.device)))
    flops.record(plan.nnz * plan.order * plan.R)
    return out
