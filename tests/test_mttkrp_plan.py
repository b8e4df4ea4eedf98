"""GPU parity of the plan MTTKRP (spt_mttkrp_plan_create / _exec,
csrc/mttkrp_plan.cu) against the CPU oracle (P/src/kernels_seq.cpp:153-174).

Tolerance (BASELINE.json north_star): every output entry within 1e-5 of the
fp64 recomputation, |y - y64| <= 1e-5 * max(|y64|, sum|terms|). Empty rows
must be exact zeros. The plan kernel is deterministic: two runs are
bit-identical.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.oracle import HostTensor, Oracle
from tests.test_gpu_parity import dev, rand_tensor, within_tol

pytestmark = pytest.mark.gpu
O = Oracle()


@pytest.fixture(scope="module")
def ops():
    from paper_1902_03317_b200 import _lib, ops
    assert _lib.missing_symbols() == []
    return ops


def up(x: HostTensor):
    from paper_1902_03317_b200.coo import HostCOO
    return dev((None, HostCOO, None), x)


def _factors(rng, dims, R, lo=0.0, hi=1.0):
    return [rng.uniform(lo, hi, (d, R)).astype(np.float32) for d in dims]


def _check(ops, x: HostTensor, fs, mode, **plan_kw):
    _, o64, oab = O.mttkrp(x, fs, mode)
    dx = up(x)
    if plan_kw.pop("presorted", False):  # input already in some mode-leading order
        xs = x.copy()
        O.sort_lexicographic(xs, [mode] + [d for d in range(len(x.dims)) if d != mode])
        dx = up(xs)
    plan = ops.mttkrp_plan(dx, mode, fs[0].shape[1], **plan_kw)
    tf = [torch.from_numpy(f).cuda() for f in fs]
    out = ops.mttkrp(plan, tf, mode).cpu().numpy()
    ok, worst = within_tol(out, o64, oab)
    assert ok, (mode, plan_kw, worst)
    assert np.all(out[oab == 0] == 0.0), "empty rows must be zero"
    again = ops.mttkrp(plan, tf, mode).cpu().numpy()
    assert np.array_equal(out.view(np.uint32), again.view(np.uint32)), "not deterministic"
    return plan, out


@pytest.mark.parametrize("R", [16, 32, 48, 64])
@pytest.mark.parametrize("order", [2, 3, 4])
@pytest.mark.parametrize("hot", ["0", "100000"])
def test_plan_shapes(ops, R, order, hot, monkeypatch):
    """SPT_PLAN_HOT_MAX > 0 also serves the most gathered rows from shared
    memory (the kernel's HOT instantiation)."""
    monkeypatch.setenv("SPT_PLAN_HOT_MAX", hot)
    rng = np.random.default_rng(100 * R + order)
    dims = {2: [3000, 700], 3: [600, 500, 400], 4: [90, 80, 70, 60]}[order]
    x = rand_tensor(rng, dims, 60_000)
    fs = _factors(rng, dims, R)
    for mode in range(order):
        for kw in ({}, {"hot": False}, {"presorted": True}):
            _check(ops, x, fs, mode, **kw)


def test_plan_zipf_hot_rows(ops, monkeypatch):
    """Zipf modes: hot rows are chosen, long rows cross many lane groups and
    CTAs (CTA fold and the last-CTA grid fold)."""
    monkeypatch.setenv("SPT_PLAN_HOT_MAX", "100000")
    from paper_1902_03317_b200 import generate
    g = generate.coo([20000, 8000, 3000], 2_000_000, 5, [1.1, 1.1, 1.1], 0.0, 1.0)
    x = HostTensor(*[getattr(g.to_host(), k) for k in ("dims", "indices", "values",
                                                       "sort_order", "coalesced")])
    rng = np.random.default_rng(5)
    fs = _factors(rng, x.dims, 32)
    for mode in range(3):
        plan, _ = _check(ops, x, fs, mode)
        assert plan.nhot > 0 and sum(plan.hot_per_level) == plan.nhot
        # levels: the other modes by decreasing extent
        others = [d for d in range(3) if d != mode]
        assert plan.level_modes == sorted(others, key=lambda d: -x.dims[d])


def test_plan_heavy_row_and_gaps(ops):
    """One row holding 1M entries (spans ~100 lane groups and several CTAs),
    scattered light rows and long runs of empty rows, 4th order."""
    rng = np.random.default_rng(7)
    n_heavy = 1_000_000
    rows = np.concatenate([np.full(n_heavy, 7, np.uint32),
                           rng.choice(np.arange(10, 50000, 7), 30000).astype(np.uint32)])
    j = rng.integers(0, 300, rows.shape[0]).astype(np.uint32)
    k = rng.integers(0, 300, rows.shape[0]).astype(np.uint32)
    m = rng.integers(0, 50, rows.shape[0]).astype(np.uint32)
    lin = ((rows.astype(np.int64) * 300 + j) * 300 + k) * 50 + m
    _, first = np.unique(lin, return_index=True)
    x = HostTensor([50003, 300, 300, 50], [rows[first], j[first], k[first], m[first]],
                   rng.uniform(0, 1, first.shape[0]).astype(np.float32), None, True)
    fs = _factors(rng, x.dims, 32)
    _check(ops, x, fs, 0)
    _check(ops, x, fs, 3)


@pytest.mark.parametrize("nnz", [1, 3, 5, 17, 100, 4099])
def test_plan_tiny_and_ragged(ops, nnz):
    """Fewer entries than lane groups (most groups empty), ranges that are
    not multiples of 4, and a large output of mostly empty rows."""
    rng = np.random.default_rng(nnz)
    x = rand_tensor(rng, [20000, 30, 40], nnz)
    fs = _factors(rng, x.dims, 16)
    for mode in range(3):
        _check(ops, x, fs, mode)


def test_plan_signed_factors_and_reuse(ops):
    """Signed factors (cancellation: the sum|terms| bound) and one plan run
    with two different factor sets."""
    rng = np.random.default_rng(3)
    x = rand_tensor(rng, [400, 300, 200], 200_000, -1, 1)
    fs = _factors(rng, x.dims, 32, -1, 1)
    plan, out1 = _check(ops, x, fs, 1)
    fs2 = _factors(rng, x.dims, 32, -1, 1)
    _, o64, oab = O.mttkrp(x, fs2, 1)
    out2 = ops.mttkrp(plan, [torch.from_numpy(f).cuda() for f in fs2], 1).cpu().numpy()
    assert within_tol(out2, o64, oab)[0]
    assert not np.array_equal(out1, out2)


def test_plan_errors(ops):
    from paper_1902_03317_b200._lib import InvalidArgument
    rng = np.random.default_rng(1)
    x = rand_tensor(rng, [50, 40, 30], 1000)
    dx = up(x)
    with pytest.raises(InvalidArgument):
        ops.mttkrp_plan(dx, 0, 12)  # R not a multiple of 16: use ops.mttkrp
    with pytest.raises(InvalidArgument):
        ops.mttkrp_plan(dx, 3, 16)
    plan = ops.mttkrp_plan(dx, 0, 16)
    fs = [torch.rand(d, 32, device="cuda") for d in x.dims]
    with pytest.raises(InvalidArgument):
        ops.mttkrp(plan, fs, 0)  # R differs from the plan's
    with pytest.raises(InvalidArgument):
        ops.mttkrp(plan, [torch.rand(d, 16, device="cuda") for d in x.dims], 1)  # other mode
    with pytest.raises(InvalidArgument):
        ops.mttkrp(plan, [torch.rand(d, 16, device="cuda") for d in x.dims], 0,
                   out=torch.empty(49, 16, device="cuda"))
