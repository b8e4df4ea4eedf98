"""B200-native COO sparse-tensor kernels (PASTA / spten hot path) behind a C-ABI.

See DESIGN.md. Public surface: `ops` (the reference-named entry points on
device tensors), `coo` (DeviceCOO / HostCOO / FiberIndex), `generate`
(seeded synthetic inputs), `parallel` (multi-GPU sharding).
"""
from . import _lib  # noqa: F401

__all__ = ["ops", "coo", "generate", "parallel"]
