"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the B200 kernels.

Two layers, both off the product path (only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs import this module):

* `Oracle`: ctypes wrapper of liboracle.so, the plain-C restatement of the
  reference's algorithms (oracle/spten_oracle.c, each function citing the
  reference file:line it follows). Bit-identical to spten::seq for
  ts/tew_eq/tew/sort/coalesce/fiber-index; returns fp64 recomputations for
  ttv/ttm/mttkrp.
* `Ref`: ctypes wrapper of oracle/_ref/libspten_ref.so, the *real* reference
  library compiled from /root/reference/proj/src (oracle/Makefile) behind
  oracle/ref_shim.cpp. Used to pin the restatement (tests/golden) and as the
  timed CPU baseline.

Parity status: pinned -- tests/test_oracle.py checks Oracle against golden
vectors produced by the reference itself (tests/golden/make_golden.py) and,
where _ref is present, against the live reference.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspten_ref.so")

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_P = ctypes.c_void_p


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


def _arr_ptrs(arrs):
    a = (_P * max(1, len(arrs)))()
    for i, x in enumerate(arrs):
        a[i] = x.ctypes.data
    return a


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class HostTensor:
    """Minimal host COO (same fields as the reference's SparseTensorCOO)."""

    def __init__(self, dims, indices, values, sort_order=None, coalesced=False):
        self.dims = [int(d) for d in dims]
        self.indices = [_u32(i) for i in indices]
        self.values = _f32(values)
        self.sort_order = None if sort_order is None else [int(s) for s in sort_order]
        self.coalesced = bool(coalesced)

    @property
    def order(self):
        return len(self.dims)

    @property
    def nnz(self):
        return int(self.values.shape[0])

    def copy(self):
        return HostTensor(self.dims, [i.copy() for i in self.indices], self.values.copy(),
                          self.sort_order, self.coalesced)

    @staticmethod
    def like(t):
        return HostTensor(t.dims, t.indices, t.values, t.sort_order, t.coalesced)


class ReferenceError_(Exception):
    pass


def _raise(code: int, msg: str):
    if code == 1:
        raise ValueError(msg)  # std::invalid_argument
    if code == 2:
        raise ArithmeticError(msg)  # std::domain_error
    if code == 3:
        raise OverflowError(msg)
    if code == 4:
        raise MemoryError(msg)
    raise RuntimeError(msg)


# ---------------------------------------------------------------------------


class Oracle:
    """The plain-C restatement (oracle/spten_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            build()
        self.lib = ctypes.CDLL(ORACLE_SO)

    # seq::ts
    def ts(self, x: HostTensor, s: float, op: int) -> HostTensor:
        zi = [np.empty(x.nnz, np.uint32) for _ in range(x.order)]
        zv = np.empty(x.nnz, np.float32)
        self.lib.or_ts(ctypes.c_uint64(x.nnz), x.order, _arr_ptrs(x.indices),
                       x.values.ctypes.data_as(_f32p), ctypes.c_float(s), op, _arr_ptrs(zi),
                       zv.ctypes.data_as(_f32p))
        return HostTensor(x.dims, zi, zv, x.sort_order, x.coalesced)

    # seq::tew_eq
    def tew_eq(self, x: HostTensor, y: HostTensor, op: int) -> HostTensor:
        if x.order != y.order or x.dims != y.dims:
            raise ValueError("tew_eq: tensors must have identical dimensions")
        if x.nnz != y.nnz:
            raise ValueError("tew_eq: tensors must have identical nonzero counts")
        zi = [np.empty(x.nnz, np.uint32) for _ in range(x.order)]
        zv = np.empty(x.nnz, np.float32)
        err = ctypes.c_uint64(0)
        rc = self.lib.or_tew_eq(ctypes.c_uint64(x.nnz), x.order, _arr_ptrs(x.indices),
                                x.values.ctypes.data_as(_f32p), _arr_ptrs(y.indices),
                                y.values.ctypes.data_as(_f32p), op, _arr_ptrs(zi),
                                zv.ctypes.data_as(_f32p), ctypes.byref(err))
        if rc == 1:
            raise ValueError(f"tew_eq: nonzero patterns differ at entry {err.value}")
        if rc == 2:
            raise ArithmeticError(f"tew_eq: division by a stored zero at entry {err.value}")
        return HostTensor(x.dims, zi, zv, x.sort_order, x.coalesced)

    # sort_lexicographic (in place)
    def sort_perm(self, x: HostTensor, mode_order: Sequence[int]) -> np.ndarray:
        mo = _u32(mode_order)
        perm = np.empty(x.nnz, np.uint64)
        self.lib.or_sort_perm(ctypes.c_uint64(x.nnz), x.order, _arr_ptrs(x.indices),
                              mo.ctypes.data_as(_u32p), perm.ctypes.data_as(_u64p))
        return perm

    def sort_lexicographic(self, x: HostTensor, mode_order: Sequence[int]) -> None:
        perm = self.sort_perm(x, mode_order)
        for d in range(x.order):
            x.indices[d] = x.indices[d][perm]
        x.values = x.values[perm]
        x.sort_order = [int(m) for m in mode_order]

    # coalesce
    def coalesce(self, x: HostTensor) -> HostTensor:
        s = x.copy()
        if s.sort_order is None:
            self.sort_lexicographic(s, list(range(x.order)))
        zi = [np.empty(x.nnz, np.uint32) for _ in range(x.order)]
        zv = np.empty(x.nnz, np.float32)
        mo = _u32(s.sort_order)
        n = self.lib.or_coalesce_sorted
        n.restype = ctypes.c_uint64
        k = n(ctypes.c_uint64(s.nnz), s.order, _arr_ptrs(s.indices), s.values.ctypes.data_as(_f32p),
              mo.ctypes.data_as(_u32p), _arr_ptrs(zi), zv.ctypes.data_as(_f32p))
        return HostTensor(x.dims, [a[:k].copy() for a in zi], zv[:k].copy(), s.sort_order, True)

    # build_fiber_index -> fptr (uint64, nfibs+1)
    def build_fiber_index(self, x: HostTensor, mode: int) -> np.ndarray:
        if mode >= x.order:
            raise ValueError("build_fiber_index: mode out of range")
        if x.sort_order is None or x.sort_order[-1] != mode:
            raise ValueError("build_fiber_index: tensor must be sorted with the target mode as "
                             "the last key")
        fptr = np.empty(x.nnz + 1, np.uint64)
        f = self.lib.or_fiber_index
        f.restype = ctypes.c_uint64
        nf = f(ctypes.c_uint64(x.nnz), x.order, _arr_ptrs(x.indices), mode,
               fptr.ctypes.data_as(_u64p))
        return fptr[: nf + 1].copy()

    # seq::tew (sorts its operands in place unless they share a sort order)
    def tew(self, x: HostTensor, y: HostTensor, op: int) -> tuple:
        if op == 3:
            raise ValueError("tew: div is not defined for mismatched patterns")
        if x.order != y.order:
            raise ValueError("tew: tensors must have the same order")
        if not (x.coalesced and y.coalesced):
            raise ValueError("tew: both inputs must be coalesced")
        if not (x.sort_order and y.sort_order and x.sort_order == y.sort_order):
            self.sort_lexicographic(x, list(range(x.order)))
            self.sort_lexicographic(y, list(range(y.order)))
        cap = x.nnz + y.nnz
        zi = [np.empty(cap, np.uint32) for _ in range(x.order)]
        zv = np.empty(cap, np.float32)
        fl = ctypes.c_uint64(0)
        f = self.lib.or_tew_merge
        f.restype = ctypes.c_uint64
        mo = _u32(x.sort_order)
        k = f(x.order, ctypes.c_uint64(x.nnz), _arr_ptrs(x.indices), x.values.ctypes.data_as(_f32p),
              ctypes.c_uint64(y.nnz), _arr_ptrs(y.indices), y.values.ctypes.data_as(_f32p),
              mo.ctypes.data_as(_u32p), op, _arr_ptrs(zi), zv.ctypes.data_as(_f32p),
              ctypes.byref(fl))
        dims = [max(a, b) for a, b in zip(x.dims, y.dims)]
        return HostTensor(dims, [a[:k].copy() for a in zi], zv[:k].copy(), x.sort_order,
                          True), int(fl.value)

    def ttv(self, x: HostTensor, v: np.ndarray, mode: int, fptr: Optional[np.ndarray] = None):
        if fptr is None:
            fptr = self.build_fiber_index(x, mode)
        fptr = np.ascontiguousarray(fptr, dtype=np.uint64)
        nf = fptr.shape[0] - 1
        zi = [np.empty(nf, np.uint32) for _ in range(x.order - 1)]
        zv = np.empty(nf, np.float32)
        z64 = np.empty(nf, np.float64)
        zab = np.empty(nf, np.float64)
        v = _f32(v)
        self.lib.or_ttv(x.order, ctypes.c_uint64(x.nnz), _arr_ptrs(x.indices),
                        x.values.ctypes.data_as(_f32p), v.ctypes.data_as(_f32p), mode,
                        fptr.ctypes.data_as(_u64p), ctypes.c_uint64(nf), _arr_ptrs(zi),
                        zv.ctypes.data_as(_f32p), z64.ctypes.data_as(_f64p),
                        zab.ctypes.data_as(_f64p))
        dims = [e for d, e in enumerate(x.dims) if d != mode]
        so = [d if d < mode else d - 1 for d in x.sort_order if d != mode]
        return HostTensor(dims, zi, zv, so, True), z64, zab

    def ttm(self, x: HostTensor, u: np.ndarray, mode: int, fptr: Optional[np.ndarray] = None):
        if fptr is None:
            fptr = self.build_fiber_index(x, mode)
        fptr = np.ascontiguousarray(fptr, dtype=np.uint64)
        nf = fptr.shape[0] - 1
        u = _f32(u)
        R = u.shape[1]
        zi = [np.empty(nf * R, np.uint32) for _ in range(x.order)]
        zv = np.empty(nf * R, np.float32)
        z64 = np.empty(nf * R, np.float64)
        zab = np.empty(nf * R, np.float64)
        self.lib.or_ttm(x.order, ctypes.c_uint64(x.nnz), _arr_ptrs(x.indices),
                        x.values.ctypes.data_as(_f32p), u.ctypes.data_as(_f32p),
                        ctypes.c_uint64(R), mode, fptr.ctypes.data_as(_u64p), ctypes.c_uint64(nf),
                        _arr_ptrs(zi), zv.ctypes.data_as(_f32p), z64.ctypes.data_as(_f64p),
                        zab.ctypes.data_as(_f64p))
        dims = list(x.dims)
        dims[mode] = R
        return HostTensor(dims, zi, zv, x.sort_order, True), z64, zab

    def mttkrp(self, x: HostTensor, factors: Sequence[Optional[np.ndarray]], mode: int,
               want64: bool = True):
        R = next(f.shape[1] for d, f in enumerate(factors) if d != mode)
        rows = x.dims[mode]
        fs = [(_f32(f) if (f is not None and d != mode) else np.zeros((1, R), np.float32))
              for d, f in enumerate(factors)]
        out = np.empty((rows, R), np.float32)
        o64 = np.empty((rows, R), np.float64) if want64 else None
        oab = np.empty((rows, R), np.float64) if want64 else None
        self.lib.or_mttkrp(x.order, ctypes.c_uint64(x.nnz), _arr_ptrs(x.indices),
                           x.values.ctypes.data_as(_f32p), _arr_ptrs(fs), ctypes.c_uint64(R),
                           mode, ctypes.c_uint64(rows), out.ctypes.data_as(_f32p),
                           None if o64 is None else o64.ctypes.data_as(_f64p),
                           None if oab is None else oab.ctypes.data_as(_f64p))
        return out, o64, oab


# ---------------------------------------------------------------------------


class Ref:
    """The real reference library (oracle/_ref/libspten_ref.so)."""

    SEQ, PAR = 0, 1

    def __init__(self):
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (reference sources absent)")
        lib = ctypes.CDLL(REF_SO)
        for name in ("ref_coo_new", "ref_gen_synthetic", "ref_fiber_new", "ref_vector_new",
                     "ref_matrix_new", "ref_factors_new"):
            getattr(lib, name).restype = _P
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_flops_count.restype = ctypes.c_uint64
        lib.ref_coo_nnz.restype = ctypes.c_uint64
        lib.ref_coo_new.argtypes = [ctypes.c_uint32, _u32p, ctypes.c_uint64, _P, _P,
                                    ctypes.POINTER(ctypes.c_int32), ctypes.c_int, ctypes.c_int]
        lib.ref_gen_synthetic.argtypes = [ctypes.c_uint32, _u32p, ctypes.c_uint64, ctypes.c_uint64]
        lib.ref_ts.argtypes = [_P, ctypes.c_float, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(_P)]
        for n in ("ref_tew_eq", "ref_tew"):
            getattr(lib, n).argtypes = [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(_P)]
        lib.ref_coo_free.argtypes = [_P]
        lib.ref_coo_order.argtypes = [_P]
        lib.ref_coo_nnz.argtypes = [_P]
        lib.ref_coo_read.argtypes = [_P, _u32p, _P, _f32p, ctypes.POINTER(ctypes.c_int32)]
        lib.ref_sort.argtypes = [_P, _u32p]
        lib.ref_coalesce.argtypes = [_P, ctypes.POINTER(_P)]
        lib.ref_fiber_index.argtypes = [_P, ctypes.c_uint32, _u64p, _u64p]
        lib.ref_fiber_new.argtypes = [_P, ctypes.c_uint32]
        lib.ref_fiber_free.argtypes = [_P]
        lib.ref_vector_new.argtypes = [_f32p, ctypes.c_uint64]
        lib.ref_vector_free.argtypes = [_P]
        lib.ref_matrix_new.argtypes = [_f32p, ctypes.c_uint64, ctypes.c_uint64]
        lib.ref_matrix_free.argtypes = [_P]
        lib.ref_matrix_read.argtypes = [_P, _f32p]
        lib.ref_ttv_fib.argtypes = [_P, _P, ctypes.c_uint32, _P, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(_P)]
        lib.ref_ttm_fib.argtypes = [_P, _P, ctypes.c_uint32, _P, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(_P)]
        lib.ref_mttkrp.argtypes = [_P, _P, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.POINTER(_P)]
        lib.ref_factors_new.argtypes = [_P, _P]
        lib.ref_factors_free.argtypes = [_P]
        lib.ref_mttkrp_fv.argtypes = [_P, _P, ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.POINTER(_P)]
        lib.ref_read_tns.argtypes = [ctypes.c_char_p, _u32p, ctypes.c_uint32, ctypes.POINTER(_P)]
        lib.ref_write_tns.argtypes = [_P, ctypes.c_char_p]
        self.lib = lib

    def read_tns(self, path: str, dims=None) -> HostTensor:
        """spten::read_tns<float> (P/src/io.cpp:42-120)."""
        h = _P()
        d = _u32(dims) if dims is not None else None
        self._check(self.lib.ref_read_tns(path.encode(), d.ctypes.data_as(_u32p) if d is not None
                                          else None, len(dims) if dims is not None else 0,
                                          ctypes.byref(h)))
        return self.read(h.value)

    def write_tns(self, x: HostTensor, path: str) -> None:
        """spten::write_tns<float> (P/src/io.cpp:122-)."""
        h = self.coo(x)
        try:
            self._check(self.lib.ref_write_tns(h, path.encode()))
        finally:
            self.free(h)

    def max_threads(self) -> int:
        return int(self.lib.ref_max_threads())

    def _check(self, rc):
        if rc:
            _raise(rc, self.lib.ref_last_error().decode("latin-1"))

    # handles ------------------------------------------------------------------
    def coo(self, t: HostTensor) -> int:
        dims = _u32(t.dims)
        so = (ctypes.c_int32 * max(1, t.order))(*(t.sort_order or [0] * t.order))
        return self.lib.ref_coo_new(t.order, dims.ctypes.data_as(_u32p), t.nnz,
                                    _arr_ptrs(t.indices), t.values.ctypes.data, so,
                                    1 if t.sort_order is not None else 0, 1 if t.coalesced else 0)

    def read(self, h: int, free: bool = True) -> HostTensor:
        order = self.lib.ref_coo_order(h)
        n = self.lib.ref_coo_nnz(h)
        dims = np.empty(order, np.uint32)
        idx = [np.empty(n, np.uint32) for _ in range(order)]
        vals = np.empty(n, np.float32)
        so = (ctypes.c_int32 * max(1, order))()
        flags = self.lib.ref_coo_read(h, dims.ctypes.data_as(_u32p), _arr_ptrs(idx),
                                      vals.ctypes.data_as(_f32p), so)
        if free:
            self.lib.ref_coo_free(h)
        return HostTensor(dims.tolist(), idx, vals, list(so)[:order] if flags & 1 else None,
                          bool(flags & 2))

    def free(self, h: int) -> None:
        self.lib.ref_coo_free(h)

    # generators / ops ---------------------------------------------------------
    def gen_synthetic(self, dims, nnz: int, seed: int) -> HostTensor:
        d = _u32(dims)
        h = self.lib.ref_gen_synthetic(len(dims), d.ctypes.data_as(_u32p), nnz, seed)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode("latin-1"))
        return self.read(h)

    def ts(self, x: HostTensor, s: float, op: int, variant=0, nthreads=0) -> HostTensor:
        hx = self.coo(x)
        out = _P()
        try:
            self._check(self.lib.ref_ts(hx, s, op, variant, nthreads, ctypes.byref(out)))
        finally:
            self.free(hx)
        return self.read(out.value)

    def tew_eq(self, x, y, op, variant=0, nthreads=0) -> HostTensor:
        hx, hy = self.coo(x), self.coo(y)
        out = _P()
        try:
            self._check(self.lib.ref_tew_eq(hx, hy, op, variant, nthreads, ctypes.byref(out)))
        finally:
            self.free(hx)
            self.free(hy)
        return self.read(out.value)

    def tew(self, x, y, op, variant=0, nthreads=0):
        """Returns (z, x_after, y_after): tew sorts its operands in place."""
        hx, hy = self.coo(x), self.coo(y)
        out = _P()
        try:
            self.lib.ref_flops_reset()
            self._check(self.lib.ref_tew(hx, hy, op, variant, nthreads, ctypes.byref(out)))
            fl = int(self.lib.ref_flops_count())
        except Exception:
            self.free(hx)
            self.free(hy)
            raise
        return self.read(out.value), self.read(hx), self.read(hy), fl

    def sort_lexicographic(self, x: HostTensor, mode_order) -> HostTensor:
        hx = self.coo(x)
        try:
            self._check(self.lib.ref_sort(hx, _u32(mode_order).ctypes.data_as(_u32p)))
        except Exception:
            self.free(hx)
            raise
        return self.read(hx)

    def coalesce(self, x: HostTensor) -> HostTensor:
        hx = self.coo(x)
        out = _P()
        try:
            self._check(self.lib.ref_coalesce(hx, ctypes.byref(out)))
        finally:
            self.free(hx)
        return self.read(out.value)

    def build_fiber_index(self, x: HostTensor, mode: int) -> np.ndarray:
        hx = self.coo(x)
        fptr = np.empty(x.nnz + 1, np.uint64)
        nf = ctypes.c_uint64(0)
        try:
            self._check(self.lib.ref_fiber_index(hx, mode, fptr.ctypes.data_as(_u64p),
                                                 ctypes.byref(nf)))
        finally:
            self.free(hx)
        return fptr[: nf.value + 1].copy()

    def ttv(self, x, v, mode, variant=0, nthreads=0) -> HostTensor:
        hx = self.coo(x)
        v = _f32(v)
        hv = self.lib.ref_vector_new(v.ctypes.data_as(_f32p), v.shape[0])
        hf = self.lib.ref_fiber_new(hx, mode)
        out = _P()
        try:
            if not hf:
                _raise(1, self.lib.ref_last_error().decode("latin-1"))
            self._check(self.lib.ref_ttv_fib(hx, hv, mode, hf, variant, nthreads,
                                             ctypes.byref(out)))
        finally:
            self.free(hx)
            self.lib.ref_vector_free(hv)
            if hf:
                self.lib.ref_fiber_free(hf)
        return self.read(out.value)

    def ttm(self, x, u, mode, variant=0, nthreads=0) -> HostTensor:
        hx = self.coo(x)
        u = _f32(u)
        hu = self.lib.ref_matrix_new(u.ctypes.data_as(_f32p), u.shape[0], u.shape[1])
        out = _P()
        try:
            self._check(self.lib.ref_ttm_fib(hx, hu, mode, None, variant, nthreads,
                                             ctypes.byref(out)))
        finally:
            self.free(hx)
            self.lib.ref_matrix_free(hu)
        return self.read(out.value)

    def mttkrp(self, x, factors, mode, variant=0, nthreads=0, strategy=0) -> np.ndarray:
        hx = self.coo(x)
        hs = (_P * x.order)()
        R = 0
        for d, f in enumerate(factors):
            if f is None:
                continue
            f = _f32(f)
            hs[d] = self.lib.ref_matrix_new(f.ctypes.data_as(_f32p), f.shape[0], f.shape[1])
            if d != mode:
                R = f.shape[1]
        out = _P()
        try:
            self._check(self.lib.ref_mttkrp(hx, hs, mode, variant, nthreads, strategy,
                                            ctypes.byref(out)))
        finally:
            self.free(hx)
            for d in range(x.order):
                if hs[d]:
                    self.lib.ref_matrix_free(hs[d])
        res = np.empty((x.dims[mode], R), np.float32)
        self.lib.ref_matrix_read(out.value, res.ctypes.data_as(_f32p))
        self.lib.ref_matrix_free(out.value)
        return res


# ---------------------------------------------------------------------------
# .tns ingest: a pure-Python restatement of spten::read_tns<float>
# (P/src/io.cpp:42-120; split_ws / fail_at at io.cpp:17-39), for small files.
# Pinned against the live reference (Ref.read_tns) by tests/test_tns_oracle.py.

import re  # noqa: E402
from fractions import Fraction  # noqa: E402

_TNS_NUM = re.compile(rb"-?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?\Z")
_TNS_WORD = re.compile(rb"-?(?:inf|infinity|nan(?:\([A-Za-z0-9_]*\))?)\Z", re.I)
_FLT_MAX = float(np.finfo(np.float32).max)


def _f32_bits_of(q: Fraction) -> Optional[int]:
    """Correctly rounded (ties to even) float32 bits of q > 0; None when the
    result is out of range (rounds to infinity, or a nonzero q rounds to 0),
    std::from_chars' result_out_of_range."""
    c = np.float32(min(float(q), _FLT_MAX)).view(np.uint32).item()
    # the candidates around c: bits c-2 .. c+2 (bit 0x7F800000 stands for
    # "rounds to infinity", 0 for "rounds to zero")
    best, best_err = None, None
    for b in range(max(0, c - 2), min(0x7F800000, c + 2) + 1):
        v = Fraction(2 ** 128) if b == 0x7F800000 else Fraction(
            float(np.uint32(b).view(np.float32)))
        err = abs(q - v)
        if best is None or err < best_err or (err == best_err and b % 2 == 0):
            best, best_err = b, err
    if best in (0, 0x7F800000):
        return None
    return best


def _tns_value(tok: bytes) -> Optional[int]:
    """std::from_chars(float) over the whole token -> float32 bits or None."""
    if _TNS_WORD.match(tok):
        neg = tok.startswith(b"-")
        w = tok.lstrip(b"-").lower()
        bits = 0x7F800000 if w.startswith(b"inf") else 0x7FC00000
        return bits | (0x80000000 if neg else 0)
    if not _TNS_NUM.match(tok):
        return None
    neg = tok.startswith(b"-")
    body = tok.lstrip(b"-")
    mant, _, exp = body.lower().partition(b"e")
    ip, _, fp = mant.partition(b".")
    digits = (ip + fp).lstrip(b"0")
    if not digits:
        return 0x80000000 if neg else 0
    E = (int(exp) if exp else 0) - len(fp)
    mag = len(digits) - 1 + E
    if mag > 38 or mag < -46:
        return None
    q = Fraction(int(digits)) * (Fraction(10) ** E)
    b = _f32_bits_of(q)
    if b is None:
        return None
    return b | (0x80000000 if neg else 0)


def read_tns_py(data: bytes, dims: Optional[Sequence[int]] = None, name: str = "<text>"):
    """read_tns<float> over the bytes of a file: returns (dims, [idx u32 arrays],
    values f32) or raises RuntimeError("name:line: msg") / ValueError like the
    reference (P/src/io.cpp:42-120)."""
    def fail(lineno, msg):
        raise RuntimeError(f"{name}:{lineno}: {msg}")

    N = 0
    have_order = False
    if dims is not None:
        N = len(dims)
        if N == 0:
            raise ValueError("read_tns: dims override must not be empty")
        have_order = True
    idx: list = [[] for _ in range(N)]
    vals: list = []
    maxidx = [0] * N
    lines = data.split(b"\n")
    if lines and lines[-1] == b"":
        lines.pop()  # std::getline: a final '\n' ends the last line
    for lineno, line in enumerate(lines, 1):
        if line.endswith(b"\r"):
            line = line[:-1]
        s = line.lstrip(b" \t")
        if not s or s.startswith(b"#"):
            continue
        tok = [t for t in re.split(rb"[ \t]+", line) if t]
        if not have_order:
            if len(tok) < 2:
                fail(lineno, "need at least one index and a value per entry")
            N = len(tok) - 1
            have_order = True
            idx = [[] for _ in range(N)]
            maxidx = [0] * N
        elif len(tok) != N + 1:
            fail(lineno, f"expected {N + 1} tokens, got {len(tok)}")
        for d in range(N):
            t = tok[d]
            if not re.fullmatch(rb"[0-9]+", t) or int(t) >= 1 << 64:
                fail(lineno, f"non-numeric index token '{t.decode('latin-1')}'")
            raw = int(t)
            if raw < 1:
                fail(lineno, "indices are 1-based; got 0")
            if raw > 0xFFFFFFFF:
                fail(lineno, f"index {raw} out of range")
            if dims is not None:
                if raw - 1 >= dims[d]:
                    fail(lineno, f"index {raw} exceeds declared dimension {dims[d]} of mode {d}")
            else:
                maxidx[d] = max(maxidx[d], raw - 1)
            idx[d].append(raw - 1)
        b = _tns_value(tok[N])
        if b is None:
            fail(lineno, f"unparsable value '{tok[N].decode('latin-1')}'")
        vals.append(b)
    if not have_order:
        raise RuntimeError(f"read_tns: {name} has no entries and no dims override; "
                           "order is unknown")
    nnz = len(vals)
    out_dims = list(dims) if dims is not None else [(m + 1) if nnz else 0 for m in maxidx]
    return (out_dims, [np.array(i, np.uint32) for i in idx],
            np.array(vals, np.uint32).view(np.float32))
