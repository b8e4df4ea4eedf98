"""The single-process multi-GPU MTTKRP of the C-ABI (spt_row_aligned_cuts,
spt_mttkrp_f32_multi) on the one GPU this box has: the
device-side row-aligned cuts equal parallel.row_aligned_ranges / row_blocks
(the torch.distributed path), and a one-device run equals the single-GPU
kernel bit for bit. More devices: correct by construction (each row computed
whole on one device, NCCL broadcasts of owned row blocks)."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_1902_03317_b200 import _lib, generate, ops, parallel
    return _lib, generate, ops, parallel


def test_row_aligned_cuts_match_host_split(mods):
    _lib, generate, ops, parallel = mods
    x = generate.coo([5000, 300, 200], 400_000, 9, [1.3, 0, 0], 0.0, 1.0, [0, 1, 2])
    ctx = _lib.Context.get(0)
    for G in (1, 2, 3, 4, 8, 16):
        cuts = (ctypes.c_uint64 * (G + 1))()
        rlo = (ctypes.c_uint32 * (G + 1))()
        d = x.descriptor()
        _lib.check(_lib.load().spt_row_aligned_cuts(ctx.handle, ctypes.byref(d), 0, G, cuts, rlo,
                                                    torch.cuda.current_stream().cuda_stream))
        rr = parallel.row_aligned_ranges(x.indices[0], G)
        bl = parallel.row_blocks(x.indices[0], rr, x.dims[0])
        assert [int(c) for c in cuts] == [lo for lo, _ in rr] + [x.nnz], G
        # owned blocks: the same partition of the rows (empty shards own empty blocks)
        got = [(int(rlo[k]), int(rlo[k + 1])) for k in range(G)]
        assert [b for b in got if b[1] > b[0]] == [b for b in bl if b[1] > b[0]], G


def test_mttkrp_multi_one_device_equals_single(mods):
    _lib, generate, ops, parallel = mods
    x = generate.coo([3000, 400, 500], 300_000, 4, [1.1, 1.1, 0], 0.0, 1.0, [1, 0, 2])
    fs = [generate.uniform((d, 32), 4, 10 + k, 0.0, 1.0) for k, d in enumerate(x.dims)]
    want = ops.mttkrp(x, fs, 1, ops.MTTKRP_SEGMENTED)
    got = parallel.mttkrp_multi(x, [fs], 1, 32)
    assert len(got) == 1 and torch.equal(got[0], want)


def test_mttkrp_multi_rejects_a_device_twice(mods):
    _lib, generate, ops, parallel = mods
    x = generate.coo([300, 40, 50], 3000, 4, [0, 0, 0], 0.0, 1.0, [0, 1, 2])
    fs = [generate.uniform((d, 16), 4, 10 + k, 0.0, 1.0) for k, d in enumerate(x.dims)]
    with pytest.raises(_lib.InvalidArgument):
        parallel.mttkrp_multi(x, [fs, fs], 0, 16)


def test_tew_shards_device_equals_host(mods):
    """The key-range split of two TEW operands searched on the device (only
    the splitter tuples leave it) equals the packed-key split on the host,
    with unequal dims and with shared and unshared tuples."""
    _lib, generate, ops, parallel = mods
    x = generate.coo([400, 300, 50], 200_000, 21, [1.2, 0, 0], 0.5, 1.5, [2, 0, 1])
    y = generate.coo([380, 310, 64], 150_000, 22, [0, 0, 0], 0.5, 1.5, [2, 0, 1])
    hx, hy = x.to_host(), y.to_host()
    for world in (1, 2, 3, 8):
        dev = parallel.tew_shards(x, y, [2, 0, 1], world)
        host = parallel.tew_shards(hx, hy, [2, 0, 1], world)
        assert dev == host
    # x against itself: every cut tuple exists in y, lower bound = same position
    assert all(a == b for a, b in parallel.tew_shards(x, x, [2, 0, 1], 5))
