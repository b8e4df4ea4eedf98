"""ctypes binding of the C-ABI in include/spten_b200.h (libspten_b200.so).

This is the Python-side FFI a reference maintainer would add; the same
symbols are what the C++ drop-in layer (include/spten/gpu.hpp) calls. The
product path has no fallback: if the shared library is missing the import of
any op raises immediately.
"""
from __future__ import annotations

import ctypes
import os
import threading

MAX_ORDER = 8
# SPT_LIB_PATH selects an alternative build of the same library (tuning
# experiments); it is never a different implementation.
LIB_PATH = os.environ.get(
    "SPT_LIB_PATH",
    os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspten_b200.so"))

# spt_status -> reference exception types (P/src/kernel_detail.hpp:38-44,
# P/src/kernels_seq.cpp:32-34). Named after the C++ exceptions.
SPT_OK, SPT_EINVAL, SPT_EDOMAIN, SPT_EOVERFLOW, SPT_ENOMEM, SPT_ERUNTIME = range(6)
SPT_FLAG_ASYNC = 1
SPT_PLAN_NO_HOT = 2  # spt_mttkrp_plan_create flag

# spten::ElemOp / ScalarOp / MttkrpStrategy enumerator values (P/include/spten/ops.hpp:5-7)
ADD, SUB, MUL, DIV = 0, 1, 2, 3
SCALAR_ADD, SCALAR_MUL = 0, 1
MTTKRP_AUTO, MTTKRP_SEGMENTED, MTTKRP_ATOMIC = -1, 0, 1
MTTKRP_SEGMENTED_CTA, MTTKRP_SEGMENTED_WARP = 2, 3  # forced tile shape (tuning/tests)


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DomainError(ArithmeticError):
    """std::domain_error"""


class IndexOverflow(OverflowError):
    """std::overflow_error"""


class DeviceOutOfMemory(MemoryError):
    """std::bad_alloc"""


class DeviceRuntimeError(RuntimeError):
    """std::runtime_error"""


_EXC = {
    SPT_EINVAL: InvalidArgument,
    SPT_EDOMAIN: DomainError,
    SPT_EOVERFLOW: IndexOverflow,
    SPT_ENOMEM: DeviceOutOfMemory,
    SPT_ERUNTIME: DeviceRuntimeError,
}


class SptCoo(ctypes.Structure):
    """struct spt_coo (include/spten_b200.h)."""

    _fields_ = [
        ("order", ctypes.c_uint32),
        ("_pad0", ctypes.c_uint32),
        ("nnz", ctypes.c_uint64),
        ("dims", ctypes.c_uint32 * MAX_ORDER),
        ("idx", ctypes.c_void_p * MAX_ORDER),
        ("val", ctypes.c_void_p),
        ("sort_order", ctypes.c_int32 * MAX_ORDER),
        ("has_sort_order", ctypes.c_int32),
        ("coalesced", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_U32 = ctypes.c_uint32
_I = ctypes.c_int
_PCOO = ctypes.POINTER(SptCoo)
_PU64 = ctypes.POINTER(ctypes.c_uint64)

_SIGNATURES = {
    "spt_abi_version": ([], _I),
    "spt_last_error": ([], ctypes.c_char_p),
    "spt_ctx_create": ([_I, ctypes.POINTER(_P)], _I),
    "spt_ctx_destroy": ([_P], None),
    "spt_ctx_trim": ([_P], _I),
    "spt_ctx_launches": ([_P], _U64),
    "spt_ctx_check": ([_P, _P], _I),
    "spt_ts_f32": ([_P, _PCOO, ctypes.c_float, _I, _PCOO, ctypes.c_uint, _P], _I),
    "spt_tew_eq_f32": ([_P, _PCOO, _PCOO, _I, _PCOO, ctypes.c_uint, _P], _I),
    "spt_tew_f32": ([_P, _PCOO, _PCOO, _I, _PCOO, _U64, _PU64, _P, ctypes.c_uint, _P], _I),
    "spt_sort_f32": ([_P, _PCOO, ctypes.POINTER(_U32), ctypes.c_uint, _P], _I),
    "spt_coalesce_f32": ([_P, _PCOO, _PCOO, _PU64, _P, ctypes.c_uint, _P], _I),
    "spt_fiber_index": ([_P, _PCOO, _U32, _P, _PU64, _P, ctypes.c_uint, _P], _I),
    "spt_ttv_f32": ([_P, _PCOO, _P, _U64, _U32, _P, _U64, _PCOO, ctypes.c_uint, _P], _I),
    "spt_ttm_f32": ([_P, _PCOO, _P, _U64, _U64, _U32, _P, _U64, _PCOO, ctypes.c_uint, _P], _I),
    "spt_mttkrp_f32": ([_P, _PCOO, ctypes.POINTER(_P), _PU64, _PU64, _U32, _P, _I,
                        ctypes.c_uint, _P], _I),
    "spt_mttkrp_plan_create": ([_P, _PCOO, _U32, _U64, ctypes.c_uint, ctypes.POINTER(_P), _P],
                               _I),
    "spt_mttkrp_plan_exec": ([_P, _P, ctypes.POINTER(_P), _PU64, _PU64, _P, ctypes.c_uint, _P],
                             _I),
    "spt_mttkrp_plan_info": ([_P, ctypes.POINTER(_U32), ctypes.POINTER(_U32),
                              ctypes.POINTER(_U32)], _I),
    "spt_mttkrp_plan_destroy": ([_P], None),
    "spt_row_aligned_cuts": ([_P, _PCOO, _U32, _U32, _PU64, ctypes.POINTER(_U32), _P], _I),
    "spt_mttkrp_f32_multi": ([_I, ctypes.POINTER(_P), _PCOO, ctypes.POINTER(_U32),
                              ctypes.POINTER(_P), _PU64, _PU64, _U32, ctypes.POINTER(_P),
                              ctypes.POINTER(_P)], _I),
    "spt_tns_scan": ([_P, _P, _U64, ctypes.POINTER(_U32), _U32, ctypes.POINTER(_P),
                      ctypes.POINTER(_U32), _PU64, _PU64, _P], _I),
    "spt_tns_parse": ([_P, _P, _PCOO, _PU64, _P], _I),
    "spt_tns_destroy": ([_P], None),
    "spt_gen_coo_f32": ([_P, _PCOO, _U64, ctypes.POINTER(ctypes.c_double), ctypes.c_float,
                         ctypes.c_float, ctypes.POINTER(_U32), _P], _I),
    "spt_gen_uniform_f32": ([_P, _P, _U64, _U64, _U64, ctypes.c_float, ctypes.c_float, _P], _I),
    "spt_l2_flush": ([_P, _P], _I),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load libspten_b200.so once; raise (never fall back) when it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: the CUDA extension is not built "
                    "(run `python -c 'import __graft_entry__ as g; g.build()'`). "
                    "There is no CPU fallback.")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGNATURES.items():
                fn = getattr(lib, name, None)
                if fn is None:  # reported by missing_symbols(); calling it raises
                    continue
                fn.argtypes = args
                fn.restype = res
            _lib = lib
    return _lib


def missing_symbols() -> list[str]:
    lib = load()
    return [n for n in _SIGNATURES if not hasattr(lib, n)]


def check(status: int) -> None:
    if status != SPT_OK:
        msg = load().spt_last_error().decode(errors="replace")
        raise _EXC.get(status, DeviceRuntimeError)(msg)


class Context:
    """One spt_ctx per (device); calls are issued on torch's current stream."""

    _per_device: dict[int, "Context"] = {}

    def __init__(self, device: int):
        lib = load()
        h = ctypes.c_void_p()
        check(lib.spt_ctx_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device

    @classmethod
    def get(cls, device: int) -> "Context":
        with _lock:
            c = cls._per_device.get(device)
        if c is None:
            c = Context(device)
            with _lock:
                cls._per_device[device] = c
        return c

    def launches(self) -> int:
        return int(load().spt_ctx_launches(self.handle))

    def trim(self) -> None:
        """Release the context's cached device memory (spt_ctx_trim)."""
        check(load().spt_ctx_trim(self.handle))
