"""The pipelined host-buffer path bench.py times as `e2e` (pinned uploads in
chunks, kernels and downloads on separate streams) returns exactly what the
oracle computes from the same host inputs."""
import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.oracle import HostTensor, Oracle
from tests._golden import same

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _ht(h):
    return HostTensor(list(h.dims), [np.asarray(i, np.uint32).copy() for i in h.indices],
                      np.asarray(h.values, np.float32).copy(), h.sort_order, h.coalesced)


@pytest.mark.parametrize("scale", [0.0005, 0.0123])
def test_c2_pipelined_e2e_matches_oracle(scale):
    import bench
    wl = bench.C2(20190210, 0, scale)
    host = wl.e2e_host(0)
    for _ in range(2):  # second pass reuses every buffer
        for o in host["out_eq"] + host["out_tew"]:
            o.val.fill_(np.nan)
            o.nnz = 0
        h2d, d2h = wl.e2e_step(host)
        torch.cuda.synchronize()
    hx, hy, hy2 = (_ht(h) for h in wl.host_inputs())
    assert h2d == 3 * wl.nnz * 16
    O = Oracle()
    for k, op in enumerate(range(4)):
        got = host["out_eq"][k].to_host()
        assert same(_ht(got), O.tew_eq(hx, hy, op)), op
    n_out = 0
    for k, op in enumerate((0, 2)):
        ref, _ = O.tew(hx.copy(), hy2.copy(), op)
        got = host["out_tew"][k].to_host()
        assert same(_ht(got), ref), op
        n_out += ref.nnz
    assert d2h == (4 * wl.nnz + n_out) * 16


@pytest.mark.parametrize("scale", [0.01, 1.0])
def test_c1_pipelined_e2e_matches_oracle(scale):
    """C1's host-buffer path (chunked x upload, TS per chunk, MTTKRP on the
    whole tensor) returns what the oracle computes from the same host data."""
    import bench
    wl = bench.C1(20190210, 0, scale)
    host = wl.e2e_host(0)
    for _ in range(2):
        for o in host["out_ts"]:
            o.val.fill_(np.nan)
            o.nnz = 0
        host["out_m"].fill_(np.nan)
        h2d, d2h = wl.e2e_step(host)
        torch.cuda.synchronize()
    n = wl.nnz
    assert h2d == n * 16 + sum(f.numel() * 4 for f in wl.f)
    assert d2h == 2 * n * 16 + host["out_m"].numel() * 4
    hx = _ht(wl.x.to_host())
    O = Oracle()
    for k, op in enumerate((0, 1)):
        assert same(_ht(host["out_ts"][k].to_host()), O.ts(hx, 2.5, op)), op
    _, y64, yab = O.mttkrp(hx, [f.cpu().numpy() for f in wl.f], 0)
    got = host["out_m"].numpy()
    assert np.all(np.abs(got - y64) <= 1e-5 * np.maximum(np.abs(y64), yab))


def test_c5_e2e_small_matches_fp64():
    """C5's host-buffer path (uploads, one plan per mode built and run, the
    I x R results and the TEW-eq output downloaded) at 1/1000 of the nnz."""
    import bench
    wl = bench.C5(20190210, 0, 0.001)
    hx = wl.x.to_host()
    hyv = wl.y.values.cpu().numpy()
    fs = [f.clone() for f in wl.f]
    host = wl.e2e_host(0)
    h2d, d2h = wl.e2e_step(host)
    torch.cuda.synchronize()
    n = wl.nnz
    assert h2d == 2 * n * 16 + sum(f.numel() * 4 for f in fs)
    assert d2h == sum(o.numel() * 4 for o in host["out_m"]) + n * 16
    idx = [torch.from_numpy(a.astype(np.int64)).cuda() for a in hx.indices]
    val = torch.from_numpy(hx.values).cuda().to(torch.float64)
    for m in range(3):
        t = val[:, None].expand(-1, wl.R).clone()
        for d in range(3):
            if d != m:
                t *= fs[d][idx[d]].to(torch.float64)
        want = torch.zeros((wl.dims[m], wl.R), dtype=torch.float64, device="cuda")
        want.index_add_(0, idx[m], t)
        got = host["out_m"][m].cuda().to(torch.float64)
        assert bool(((got - want).abs() <= 1e-5 * want.abs()).all()), m
    z = host["out_eq"].to_host()
    assert np.array_equal(z.values.view(np.uint32), (hx.values * hyv).view(np.uint32))
    assert all(np.array_equal(a, b) for a, b in zip(z.indices, hx.indices))


def test_c4_e2e_small_matches_fp64():
    """C4's host-buffer path (x in draw order uploaded, one plan per mode built
    from the unsorted tensor and run, the I x R results downloaded) at 1/100
    of the nnz."""
    import bench
    wl = bench.C4(20190210, 0, 0.01)
    hx = wl.host_x
    fs = [f.clone() for f in wl.f]
    host = wl.e2e_host(0)
    for _ in range(2):
        for o in host["out_m"]:
            o.fill_(np.nan)
        h2d, d2h = wl.e2e_step(host)
        torch.cuda.synchronize()
    n = wl.nnz
    assert h2d == n * 20 + sum(f.numel() * 4 for f in fs)
    assert d2h == sum(o.numel() * 4 for o in host["out_m"])
    idx = [torch.from_numpy(a.astype(np.int64)).cuda() for a in hx.indices]
    val = torch.from_numpy(hx.values).cuda().to(torch.float64)
    for m in range(4):
        t = val[:, None].expand(-1, wl.R).clone()
        for d in range(4):
            if d != m:
                t *= fs[d][idx[d]].to(torch.float64)
        want = torch.zeros((wl.dims[m], wl.R), dtype=torch.float64, device="cuda")
        want.index_add_(0, idx[m], t)
        got = host["out_m"][m].cuda().to(torch.float64)
        assert bool(((got - want).abs() <= 1e-5 * want.abs()).all()), m


def test_c3_e2e_small_matches_device_ops():
    """C3's host-buffer path (x in draw order uploaded, sorted mode-last and
    indexed on the device per mode, TTV and TTM outputs downloaded) at 1/100
    of the nnz: the last mode's downloaded outputs equal the ops run directly."""
    import bench
    from paper_1902_03317_b200 import ops
    wl = bench.C3(20190210, 0, 0.01)
    xs2, fib2 = wl.xs[2], wl.fib[2]
    zv = ops.ttv(xs2, wl.v[2], 2, fib2)
    zm = ops.ttm(xs2, wl.u[2], 2, fib2)
    want_v, want_m = zv.to_host(), zm.to_host()
    host = wl.e2e_host(0)
    h2d, d2h = wl.e2e_step(host)
    torch.cuda.synchronize()
    got_v, got_m = host["out_v"].to_host(), host["out_m"].to_host()
    nf = fib2.nfibs
    assert all(np.array_equal(a[:nf], b) for a, b in zip(got_v.indices, want_v.indices))
    assert np.array_equal(got_v.values[:nf].view(np.uint32), want_v.values.view(np.uint32))
    assert all(np.array_equal(a[:nf * wl.R], b) for a, b in zip(got_m.indices, want_m.indices))
    assert np.array_equal(got_m.values[:nf * wl.R].view(np.uint32), want_m.values.view(np.uint32))
    assert h2d == wl.nnz * 16 + sum(v.numel() * 4 for v in host["pv"] + host["pu"])
