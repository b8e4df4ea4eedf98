"""Seeded synthetic inputs for the BASELINE.json configurations, built on the
device by the library's own generator (spt_gen_coo_f32, csrc/gen.cu).

The reference's gen_synthetic (P/src/io.cpp:151-244) cannot express these
configs (fixed U[1,2) values, no Zipf modes, u64 linearisation overflow for
C4/C5, P/src/io.cpp:157-166); this keeps its contract (exactly nnz distinct
tuples, duplicates rejected in draw order) with the configs' distributions.
The public datasets of the paper (FROSTT/HaTen2) are not available offline;
these seeded tensors stand in for them with the configs' shapes and value
distributions.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from . import _lib
from .coo import DeviceCOO


def _ctx_stream(device: int):
    return _lib.Context.get(device), torch.cuda.current_stream(device).cuda_stream


def coo(dims: Sequence[int], nnz: int, seed: int, zipf: Optional[Sequence[float]] = None,
        lo: float = 0.0, hi: float = 1.0, sort_order: Optional[Sequence[int]] = None,
        device: int = 0) -> DeviceCOO:
    """nnz distinct tuples; mode d uniform (zipf[d] == 0) or Zipf(zipf[d]) over a
    seeded permutation of the ids; values U[lo, hi); optionally sorted."""
    ctx, st = _ctx_stream(device)
    t = DeviceCOO.empty(dims, nnz, device)
    d = t.descriptor()
    zs = (ctypes.c_double * len(dims))(*(zipf if zipf is not None else [0.0] * len(dims)))
    so = (ctypes.c_uint32 * len(dims))(*sort_order) if sort_order is not None else None
    _lib.check(_lib.load().spt_gen_coo_f32(ctx.handle, ctypes.byref(d), seed, zs, lo, hi, so, st))
    t.adopt(d)
    return t


def uniform(shape, seed: int, stream_id: int, lo: float, hi: float,
            device: int = 0) -> torch.Tensor:
    ctx, st = _ctx_stream(device)
    out = torch.empty(shape, dtype=torch.float32, device=f"cuda:{device}")
    _lib.check(_lib.load().spt_gen_uniform_f32(ctx.handle, out.data_ptr() if out.numel() else None,
                                               out.numel(), seed, stream_id, lo, hi, st))
    return out


# ---------------------------------------------------------------------------
# BASELINE.json configs.

CONFIGS = {
    # C1: MTTKRP mode 0 (R=16) + TS add/mul by 2.5
    "c1": dict(dims=[1000, 1000, 1000], nnz=1_000_000, zipf=[0, 0, 0], lo=0.0, hi=1.0, R=16),
    # C2: TEW-eq add/sub/mul/div (shared pattern) + TEW add/mul (independent pattern)
    "c2": dict(dims=[10000, 10000, 10000], nnz=10_000_000, zipf=[0, 0, 0], lo=0.5, hi=1.5),
    # C3: TTV / TTM (R=16) along every mode; mode-0 slices Zipf(1.1)
    "c3": dict(dims=[50000, 20000, 100000], nnz=50_000_000, zipf=[1.1, 0, 0], lo=0.0, hi=1.0,
               R=16),
    # C4: MTTKRP all modes, R=32, 4th order, every mode Zipf(1.2)
    "c4": dict(dims=[2_000_000, 500_000, 100_000, 1000], nnz=100_000_000,
               zipf=[1.2, 1.2, 1.2, 1.2], lo=0.0, hi=1.0, R=32),
    # C5: multi-GPU MTTKRP modes 0-2 (R=32) + TEW-eq mul, 1B nnz, Zipf(1.1)
    "c5": dict(dims=[10_000_000] * 3, nnz=1_000_000_000, zipf=[1.1, 1.1, 1.1], lo=0.0, hi=1.0,
               R=32),
}


def config_tensor(name: str, seed: int = 1, sort_order=None, device: int = 0,
                  nnz: Optional[int] = None) -> DeviceCOO:
    c = CONFIGS[name]
    return coo(c["dims"], nnz or c["nnz"], seed, c["zipf"], c["lo"], c["hi"], sort_order, device)


def tns_text(x: DeviceCOO, decimals: int = 6) -> torch.Tensor:
    """The .tns text of x (P/include/spten/io.hpp:14-20: 1-based indices, then
    the value, single spaces, '\\n' endings) as a uint8 tensor on x's device,
    built with tensor ops: bench / test input for the ingest path, not a
    product path. Values are written in fixed notation with `decimals`
    fractional digits (so they parse to the nearest float of that decimal,
    not necessarily to x's values)."""
    dev = x.device
    n = x.nnz
    chars, masks = [], []

    def digits(v: torch.Tensor, width: int, keep_one: bool = True):
        p = torch.tensor([10 ** k for k in range(width - 1, -1, -1)], dtype=torch.int64,
                         device=dev)
        d = (v[:, None] // p[None, :]) % 10
        nd = (v[:, None] >= p[None, :]).sum(1)
        if keep_one:
            nd = nd.clamp(min=1)
        mask = torch.arange(width, device=dev)[None, :] >= (width - nd)[:, None]
        return (d + 48).to(torch.uint8), mask

    def const(c: str):
        chars.append(torch.full((n, 1), ord(c), dtype=torch.uint8, device=dev))
        masks.append(torch.ones((n, 1), dtype=torch.bool, device=dev))

    for d in range(x.order):
        v = (x.indices[d].to(torch.int64) & 0xFFFFFFFF) + 1
        c, m = digits(v, len(str(int(x.dims[d]))))
        chars.append(c)
        masks.append(m)
        const(" ")
    val = x.values.to(torch.float64)
    chars.append(torch.full((n, 1), ord("-"), dtype=torch.uint8, device=dev))
    masks.append((val < 0)[:, None])
    q = torch.round(val.abs() * 10 ** decimals).to(torch.int64)
    ip, fp = q // 10 ** decimals, q % 10 ** decimals
    c, m = digits(ip, max(1, len(str(int(ip.max().item()))) if n else 1))
    chars.append(c)
    masks.append(m)
    if decimals:
        const(".")
        c, _ = digits(fp, decimals, keep_one=False)
        chars.append(c)
        masks.append(torch.ones_like(c, dtype=torch.bool))
    const("\n")
    return torch.cat(chars, 1)[torch.cat(masks, 1)]
