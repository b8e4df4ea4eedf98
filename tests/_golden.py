"""Load the reference-generated golden fixtures (tests/golden/*.npz)."""
import os

import numpy as np

from oracle.oracle import HostTensor

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def tensor(z, key):
    dims = [int(d) for d in z[f"{key}.dims"]]
    idx = [z[f"{key}.idx{d}"] for d in range(len(dims))]
    so = z[f"{key}.sort"]
    return HostTensor(dims, idx, z[f"{key}.val"], None if so.size == 0 else so.tolist(),
                      bool(z[f"{key}.coal"][0]))


def same(a, b, check_meta=True):
    """bit_identical (P/include/spten/tensor.hpp:117-123) plus metadata."""
    ok = (list(a.dims) == list(b.dims) and len(a.indices) == len(b.indices)
          and all(np.array_equal(np.asarray(p, np.uint32), np.asarray(q, np.uint32))
                  for p, q in zip(a.indices, b.indices))
          and np.array_equal(np.asarray(a.values, np.float32).view(np.uint32),
                             np.asarray(b.values, np.float32).view(np.uint32)))
    if check_meta:
        ok = ok and (a.sort_order == b.sort_order) and (bool(a.coalesced) == bool(b.coalesced))
    return ok
