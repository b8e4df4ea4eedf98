"""The C-ABI boundary, checked without a GPU: the library loads, exports every
symbol include/*.h declares, the ctypes mirror of struct spt_coo matches the C
layout, errors map onto the reference's exception types, and there is no CPU
fallback."""
import ctypes
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "spten_b200.h")


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(r"SPT_API\s+[\w\s\*]+?\b(spt_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1902_03317_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 17
    missing = [s for s in syms if not hasattr(lib, s)]
    assert missing == []
    assert set(syms) == set(_lib.EXPORTED)  # the ctypes table covers the header exactly
    assert lib.spt_abi_version() == 1


def test_nm_shows_only_the_c_abi():
    so = os.path.join(ROOT, "paper_1902_03317_b200", "libspten_b200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True,
                         check=True).stdout
    exported = sorted(l.split()[-1] for l in out.splitlines() if l.split()[-1].startswith("spt_"))
    assert exported == declared_symbols()


def test_struct_layout_matches_c():
    from paper_1902_03317_b200._lib import SptCoo
    src = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "spten_b200.h"
    int main(void) {
      printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(spt_coo), offsetof(spt_coo, nnz),
             offsetof(spt_coo, dims), offsetof(spt_coo, idx), offsetof(spt_coo, val),
             offsetof(spt_coo, sort_order), offsetof(spt_coo, has_sort_order),
             offsetof(spt_coo, coalesced));
      return 0;
    }"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", "-I", os.path.dirname(HDR), c, "-o", exe], check=True)
        got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True,
                                              check=True).stdout.split()]
    want = [ctypes.sizeof(SptCoo), SptCoo.nnz.offset, SptCoo.dims.offset, SptCoo.idx.offset,
            SptCoo.val.offset, SptCoo.sort_order.offset, SptCoo.has_sort_order.offset,
            SptCoo.coalesced.offset]
    assert got == want


def test_status_codes_map_to_reference_exceptions():
    from paper_1902_03317_b200 import _lib
    assert issubclass(_lib.InvalidArgument, ValueError)  # std::invalid_argument
    assert issubclass(_lib.DomainError, ArithmeticError)  # std::domain_error
    assert issubclass(_lib.IndexOverflow, OverflowError)  # std::overflow_error
    assert issubclass(_lib.DeviceOutOfMemory, MemoryError)  # std::bad_alloc
    assert issubclass(_lib.DeviceRuntimeError, RuntimeError)  # std::runtime_error
    with pytest.raises(ValueError):
        _lib.check(_lib.SPT_EINVAL)
    with pytest.raises(ArithmeticError):
        _lib.check(_lib.SPT_EDOMAIN)


def test_null_and_contract_errors_without_gpu():
    """Argument validation happens on the host before any CUDA call."""
    from paper_1902_03317_b200 import _lib
    lib = _lib.load()
    assert lib.spt_ts_f32(None, None, 1.0, 0, None, 0, None) == _lib.SPT_EINVAL
    x = _lib.SptCoo()
    x.order = 9
    assert lib.spt_sort_f32(None, ctypes.byref(x), None, 0, None) == _lib.SPT_EINVAL


def test_no_cpu_fallback():
    """Ops on host tensors raise instead of computing on the CPU."""
    import torch
    from paper_1902_03317_b200 import ops
    from paper_1902_03317_b200.coo import DeviceCOO
    t = DeviceCOO([2, 2], [torch.zeros(1, dtype=torch.int32)] * 2, torch.ones(1), None, True)
    with pytest.raises(ValueError, match="no CPU fallback"):
        ops.ts(t, 2.0, ops.SCALAR_MUL)
    if not torch.cuda.is_available():
        from paper_1902_03317_b200 import _lib
        h = ctypes.c_void_p()
        assert lib_create_fails(_lib, h)


def lib_create_fails(_lib, h):
    return _lib.load().spt_ctx_create(0, ctypes.byref(h)) in (_lib.SPT_ERUNTIME, _lib.SPT_ENOMEM)
