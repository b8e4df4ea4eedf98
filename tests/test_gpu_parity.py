"""GPU parity: the sm_100a kernels (through the C-ABI) against the oracle and
the reference-generated golden fixtures.

Bar (BASELINE.json north_star): indices, patterns, sort/coalesce/fiber index,
TS, TEW-eq and TEW values bit-exact; TTV/TTM/MTTKRP values within a relative
tolerance of 1e-5 per output entry against an fp64 recomputation:

    |y - y64| <= TOL * max(|y64|, sum|terms|),   TOL = 1e-5

(the sum-of-|terms| form only matters where signed terms cancel, see
SURVEY.md section 7; MTTKRP inputs are all-positive so it is plain relative).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.oracle import HostTensor, Oracle
from tests._golden import load, same, tensor

pytestmark = pytest.mark.gpu
TOL = 1e-5
O = Oracle()


@pytest.fixture(scope="module")
def sp():
    from paper_1902_03317_b200 import _lib, ops
    from paper_1902_03317_b200.coo import HostCOO
    assert _lib.missing_symbols() == []
    return ops, HostCOO, _lib


def dev(sp, t: HostTensor, offset=0):
    """Upload; offset>0 places every array at a non-16B-aligned address."""
    ops, HostCOO, _ = sp
    if offset == 0:
        return HostCOO(t.dims, t.indices, t.values, t.sort_order, t.coalesced).to_device(0)
    from paper_1902_03317_b200.coo import DeviceCOO

    def up(a, dt):
        buf = torch.empty(a.shape[0] + offset, dtype=dt, device="cuda")
        v = buf[offset:]
        v.copy_(torch.from_numpy(np.ascontiguousarray(a)).to(dt))
        return v

    return DeviceCOO(list(t.dims), [up(i.view(np.int32), torch.int32) for i in t.indices],
                     up(t.values, torch.float32), t.sort_order, t.coalesced)


def host(d) -> HostTensor:
    h = d.to_host()
    return HostTensor(h.dims, h.indices, h.values, h.sort_order, h.coalesced)


def within_tol(got, y64, yabs, tol=TOL):
    got = np.asarray(got, np.float64)
    bound = tol * np.maximum(np.abs(y64), yabs)
    bad = np.abs(got - y64) > bound + 1e-300
    return not bad.any(), float(np.max(np.abs(got - y64) / np.maximum(bound / tol, 1e-300)))


def rand_tensor(rng, dims, nnz, lo=0.0, hi=1.0, sort=None):
    cap = int(np.prod([float(d) for d in dims]))
    if cap < 16 * nnz:
        lin = rng.choice(cap, size=nnz, replace=False)
    else:
        lin = np.unique(np.concatenate([
            rng.integers(0, cap, size=nnz + nnz // 8 + 16)]))
        rng.shuffle(lin)
        lin = lin[:nnz]
    idx = []
    for d in reversed(dims):
        idx.append((lin % d).astype(np.uint32))
        lin = lin // d
    t = HostTensor(dims, idx[::-1], rng.uniform(lo, hi, len(idx[0])).astype(np.float32), None,
                   True)
    if sort is not None:
        O.sort_lexicographic(t, sort)
    return t


# ---------------------------------------------------------------------------
# golden fixtures (outputs of the reference itself)


def test_ts_tew_eq_golden(sp):
    ops = sp[0]
    z = load("elementwise.npz")
    for i in range(int(z["n_ew"])):
        x, y = tensor(z, f"ew{i}.x"), tensor(z, f"ew{i}.y")
        dx, dy = dev(sp, x), dev(sp, y)
        for op, sc in ((0, 2.5), (1, 2.5), (1, 1.0), (0, 0.0)):
            got = host(ops.ts(dx, sc, op))
            assert same(got, HostTensor(x.dims, x.indices, z[f"ew{i}.ts{op}_{sc}"], x.sort_order,
                                        x.coalesced))
        for op in range(4):
            if str(z[f"ew{i}.tew_eq{op}.expect"]) == "ok":
                got = host(ops.tew_eq(dx, dy, op))
                assert same(got, HostTensor(x.dims, x.indices, z[f"ew{i}.tew_eq{op}"],
                                            x.sort_order, x.coalesced)), (i, op)
            else:
                with pytest.raises(ArithmeticError) as e:
                    ops.tew_eq(dx, dy, op)
                assert str(e.value) == str(z[f"ew{i}.tew_eq{op}.msg"])


def test_tew_golden(sp):
    ops = sp[0]
    z = load("elementwise.npz")
    for j in range(int(z["n_tew"])):
        for op in range(3):
            k = f"tew{j}_{op}"
            x, y = tensor(z, f"{k}.x"), tensor(z, f"{k}.y")
            dx, dy = dev(sp, x), dev(sp, y)
            ops.flops.reset()
            got = host(ops.tew(dx, dy, op))
            assert same(got, tensor(z, f"{k}.z")), k
            assert ops.flops.count() == int(z[f"{k}.flops"]), k
            assert dx.sort_order == z[f"{k}.xa_sort"].tolist()  # operands sorted in place


def test_preprocess_golden(sp):
    ops = sp[0]
    z = load("preprocess.npz")
    for j in range(int(z["n_pre"])):
        k = f"pre{j}"
        x = tensor(z, f"{k}.x")
        mo = z[f"{k}.mo"].tolist()
        dx = dev(sp, x)
        ops.sort_lexicographic(dx, mo)
        assert same(host(dx), tensor(z, f"{k}.sorted")), k
        c = ops.coalesce(dx)
        assert same(host(c), tensor(z, f"{k}.coalesced")), k
        fib = ops.build_fiber_index(c, mo[-1])
        assert fib.nfibs == z[f"{k}.fptr"].shape[0] - 1
        assert np.array_equal(fib.fptr.cpu().numpy().view(np.uint32).astype(np.uint64),
                              z[f"{k}.fptr"]), k


def test_reductions_golden(sp):
    ops = sp[0]
    z = load("reductions.npz")
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    got = host(ops.ttv(dev(sp, tensor(z, "kat_ttv.x")), cu(z["kat_ttv.v"]), 2))
    assert same(got, tensor(z, "kat_ttv.z"))  # {(0,0):50, (1,1):30}
    got = host(ops.ttm(dev(sp, tensor(z, "kat_ttm.x")), cu(z["kat_ttm.u"]), 2))
    assert same(got, tensor(z, "kat_ttm.z"))  # 7, 10
    out = ops.mttkrp(dev(sp, tensor(z, "kat_mttkrp.x")),
                     [None, cu(z["kat_mttkrp.f1"]), cu(z["kat_mttkrp.f2"])], 0).cpu().numpy()
    assert out.tolist() == [[0.0, 0.0], [12.0, 30.0]]
    for n in range(int(z["n_red"])):
        k = f"red{n}"
        x = tensor(z, f"{k}.x")
        mode = int(z[f"{k}.mode"])
        dx = dev(sp, x)
        ref_ttv = tensor(z, f"{k}.ttv")
        _, y64, yab = O.ttv(x, z[f"{k}.v"], mode)
        g = host(ops.ttv(dx, cu(z[f"{k}.v"]), mode))
        assert same(HostTensor(g.dims, g.indices, ref_ttv.values, g.sort_order, g.coalesced),
                    ref_ttv), k
        assert within_tol(g.values, y64, yab)[0], k
        ref_ttm = tensor(z, f"{k}.ttm")
        _, y64, yab = O.ttm(x, z[f"{k}.u"], mode)
        g = host(ops.ttm(dx, cu(z[f"{k}.u"]), mode))
        assert same(HostTensor(g.dims, g.indices, ref_ttm.values, g.sort_order, g.coalesced),
                    ref_ttm), k
        assert within_tol(g.values, y64, yab)[0], k
        xu = tensor(z, f"{k}.xu")
        fs = [z[f"{k}.f{d}"] for d in range(x.order)]
        _, o64, oab = O.mttkrp(xu, fs, mode)
        for strategy, t in ((ops.MTTKRP_ATOMIC, xu), (ops.MTTKRP_SEGMENTED, None)):
            if t is None:  # segmented needs the output mode leading
                t = xu.copy()
                O.sort_lexicographic(t, [mode] + [d for d in range(x.order) if d != mode])
            out = ops.mttkrp(dev(sp, t), [cu(f) for f in fs], mode, strategy).cpu().numpy()
            assert within_tol(out, o64, oab)[0], (k, strategy)


# ---------------------------------------------------------------------------
# edge cases the reference tests exercise (empty, ragged tails, errors, shapes)


def test_empty_tensors(sp):
    ops = sp[0]
    e = HostTensor([3, 4, 5], [np.zeros(0, np.uint32)] * 3, np.zeros(0, np.float32), [0, 1, 2],
                   True)
    de = dev(sp, e)
    assert ops.ts(de, 2.0, 1).nnz == 0
    assert ops.tew_eq(de, dev(sp, e), 0).nnz == 0
    fib = ops.build_fiber_index(de, 2)
    assert fib.nfibs == 0 and fib.fptr.cpu().tolist() == [0]  # test_tensor.cpp:157-164
    out = ops.mttkrp(de, [None, torch.ones(4, 8, device="cuda"), torch.ones(5, 8, device="cuda")], 0)
    assert out.shape == (3, 8) and float(out.abs().sum()) == 0.0
    x = rand_tensor(np.random.default_rng(1), [3, 4, 5], 7, sort=[0, 1, 2])
    z = ops.tew(dev(sp, x), de, 0)
    assert same(host(z), x)
    assert ops.tew(dev(sp, x), de, 2).nnz == 0


def test_errors_map_to_reference_exceptions(sp):
    ops, _, lib = sp
    rng = np.random.default_rng(3)
    x = rand_tensor(rng, [4, 4, 4], 20, sort=[0, 1, 2])
    y = x.copy()
    y.indices[1] = y.indices[1].copy()
    y.indices[1][11] = (y.indices[1][11] + 1) % 4
    y.values = y.values.copy()
    y.values[5] = 0.0
    # first failing entry decides; entry 5 (zero divisor) precedes entry 11 (mismatch)
    with pytest.raises(ArithmeticError, match="entry 5"):
        ops.tew_eq(dev(sp, x), dev(sp, y), ops.DIV)
    with pytest.raises(lib.InvalidArgument, match="entry 11"):
        ops.tew_eq(dev(sp, x), dev(sp, y), ops.ADD)
    with pytest.raises(ValueError):
        ops.tew_eq(dev(sp, x), dev(sp, rand_tensor(rng, [4, 4, 5], 20)), ops.ADD)
    with pytest.raises(ValueError):
        ops.tew(dev(sp, x), dev(sp, x), ops.DIV)
    with pytest.raises(ValueError):
        ops.ttv(dev(sp, x), torch.ones(4, device="cuda"), 0)  # sorted for mode 2, not 0
    with pytest.raises(ValueError):
        ops.ttv(dev(sp, x), torch.ones(3, device="cuda"), 2)  # wrong vector length
    with pytest.raises(ValueError):
        ops.ttm(dev(sp, x), torch.ones(4, 0, device="cuda"), 2)  # R = 0
    f = [torch.ones(4, 4, device="cuda") for _ in range(3)]
    with pytest.raises(ValueError):
        ops.mttkrp(dev(sp, x), [f[0], torch.ones(5, 4, device="cuda"), f[2]], 0)
    with pytest.raises(ValueError):
        ops.mttkrp(dev(sp, x), [f[0], torch.ones(4, 3, device="cuda"), f[2]], 0)
    ops.mttkrp(dev(sp, x), [torch.ones(1, 1, device="cuda"), f[1], f[2]], 0)  # factors[mode] ignored
    # segmented strategy on an input not sorted by the output mode is reported
    xs = x.copy()
    O.sort_lexicographic(xs, [1, 0, 2])
    with pytest.raises(ValueError, match="sorted by the output mode"):
        ops.mttkrp(dev(sp, xs), f, 0, ops.MTTKRP_SEGMENTED)


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("nnz", [1, 3, 4, 5, 2047, 2048, 2049, 12345])
def test_streaming_tails_and_alignment(sp, nnz, offset):
    ops = sp[0]
    rng = np.random.default_rng(nnz)
    x = rand_tensor(rng, [40, 50, 60], nnz, 0.5, 1.5, sort=[0, 1, 2])
    y = x.copy()
    y.values = rng.uniform(0.5, 1.5, nnz).astype(np.float32)
    dx, dy = dev(sp, x, offset), dev(sp, y, offset)
    for op in range(2):
        assert same(host(ops.ts(dx, 2.5, op)), O.ts(x, 2.5, op))
    for op in range(4):
        assert same(host(ops.tew_eq(dx, dy, op)), O.tew_eq(x, y, op))


@pytest.mark.parametrize("R", [1, 3, 8, 12, 16, 32, 64, 100, 128, 200])
@pytest.mark.parametrize("order", [2, 3, 5])
def test_mttkrp_shapes(sp, R, order):
    ops = sp[0]
    rng = np.random.default_rng(R * 10 + order)
    dims = {2: [300, 70], 3: [60, 50, 40], 5: [9, 8, 7, 6, 5]}[order]
    x = rand_tensor(rng, dims, 9000)
    fs = [rng.uniform(0, 1, (d, R)).astype(np.float32) for d in dims]
    for mode in range(order):
        _, o64, oab = O.mttkrp(x, fs, mode)
        xs = x.copy()
        O.sort_lexicographic(xs, [mode] + [d for d in range(order) if d != mode])
        # AUTO on an unsorted input: a temporary plan (R % 16 == 0) or a sorted
        # copy, held to the same 1e-5 as the segmented paths; only an explicit
        # ATOMIC request gets fp32 atomics (1e-4)
        for strat, t in ((ops.MTTKRP_SEGMENTED_CTA, xs), (ops.MTTKRP_SEGMENTED_WARP, xs),
                         (ops.MTTKRP_AUTO, xs), (ops.MTTKRP_AUTO, x), (ops.MTTKRP_ATOMIC, x)):
            out = ops.mttkrp(dev(sp, t), [torch.from_numpy(f).cuda() for f in fs], mode,
                             strat).cpu().numpy()
            ok, worst = within_tol(out, o64, oab, 1e-5 if strat != ops.MTTKRP_ATOMIC else 1e-4)
            assert ok, (mode, strat, worst)


def test_mttkrp_heavy_rows_and_gaps(sp):
    """Look-back chains: one row spanning ~500 tiles, rows with no entries
    (zero-fill), a tail row, and fp64 accumulation accuracy on the long row."""
    ops = sp[0]
    rng = np.random.default_rng(11)
    n_heavy = 1_000_000
    rows = np.concatenate([np.full(n_heavy, 7, np.uint32),
                           rng.choice(np.arange(10, 5000, 3), 20000).astype(np.uint32)])
    j = rng.integers(0, 3000, rows.shape[0]).astype(np.uint32)
    k = rng.integers(0, 3000, rows.shape[0]).astype(np.uint32)
    lin = (rows.astype(np.int64) * 3000 + j) * 3000 + k
    _, first = np.unique(lin, return_index=True)
    first.sort()
    x = HostTensor([5003, 3000, 3000], [rows[first], j[first], k[first]],
                   rng.uniform(0, 1, first.shape[0]).astype(np.float32), None, True)
    O.sort_lexicographic(x, [0, 1, 2])
    fs = [rng.uniform(0, 1, (d, 32)).astype(np.float32) for d in x.dims]
    _, o64, oab = O.mttkrp(x, fs, 0)
    for strat in (ops.MTTKRP_SEGMENTED_CTA, ops.MTTKRP_SEGMENTED_WARP):
        out = ops.mttkrp(dev(sp, x), [torch.from_numpy(f).cuda() for f in fs], 0,
                         strat).cpu().numpy()
        ok, worst = within_tol(out, o64, oab)
        assert ok, (strat, worst)
        assert np.all(out[o64 == 0] == 0)


@pytest.mark.parametrize("R", [1, 5, 16, 32])
def test_ttv_ttm_long_fibers(sp, R):
    """Fibers much longer than a tile plus many length-1 fibers."""
    ops = sp[0]
    rng = np.random.default_rng(R)
    x = rand_tensor(rng, [4, 6, 200000], 300000, -1, 1)
    extra = rand_tensor(rng, [300, 300, 40], 100000, -1, 1)
    for mode in range(3):
        for t in (x, extra):
            xs = t.copy()
            O.sort_lexicographic(xs, [d for d in range(3) if d != mode] + [mode])
            v = rng.uniform(-1, 1, t.dims[mode]).astype(np.float32)
            u = rng.uniform(-1, 1, (t.dims[mode], R)).astype(np.float32)
            dx = dev(sp, xs)
            zt, y64, yab = O.ttv(xs, v, mode)
            g = host(ops.ttv(dx, torch.from_numpy(v).cuda(), mode))
            assert same(HostTensor(g.dims, g.indices, zt.values, g.sort_order, g.coalesced), zt)
            assert within_tol(g.values, y64, yab)[0]
            zm, y64, yab = O.ttm(xs, u, mode)
            g = host(ops.ttm(dx, torch.from_numpy(u).cuda(), mode))
            assert same(HostTensor(g.dims, g.indices, zm.values, g.sort_order, g.coalesced), zm)
            assert within_tol(g.values, y64, yab)[0]


def test_sort_wide_keys_and_stability(sp):
    """Keys wider than 64 bits (C4: 67 bits) and duplicate tuples."""
    ops = sp[0]
    rng = np.random.default_rng(5)
    dims = [2_000_000, 500_000, 100_000, 1000]
    n = 200_000
    idx = [rng.integers(0, d, n).astype(np.uint32) for d in dims]
    for a in idx:
        a[n // 2:n // 2 + 1000] = a[:1000]  # duplicates, distinct values
    x = HostTensor(dims, idx, rng.uniform(-1, 1, n).astype(np.float32), None, False)
    for mo in ([0, 1, 2, 3], [3, 1, 0, 2], [2, 3, 1, 0]):
        dx = dev(sp, x)
        ops.sort_lexicographic(dx, mo)
        ox = x.copy()
        O.sort_lexicographic(ox, mo)
        assert same(host(dx), ox)
        assert same(host(ops.coalesce(dx)), O.coalesce(ox))


@pytest.mark.parametrize("dims,n", [
    ([2, 1, 2], 5000),            # 2-bit key: two passes of one bit
    ([1, 1, 1], 300),             # no significant bit at all
    ([1, 2, 1], 4609),            # one-bit key, one entry past a u32-key tile
    ([300, 200, 100], 6144),      # u32 key (25 bits), exactly one tile
    ([300, 200, 100], 6145),
    ([300, 200, 100], 100_003),
    ([70000, 70000, 3], 4608),    # u64 key (36 bits), exactly one tile
    ([70000, 70000, 3], 4607),
    ([70000, 70000, 3], 150_001),
    ([4, 3, 2], 120_000),         # 24 distinct tuples: long duplicate runs, stability
    ([1 << 20, 1 << 20, 1 << 20, 16], 50_000),  # 64-bit key exactly
    ([3, 2], 1), ([3, 2], 2), ([3, 2], 3),
])
def test_sort_radix_edges(sp, dims, n):
    """The hand-written radix passes at their edges: key widths 0..64 bits,
    tile boundaries, duplicate runs (stability), sorted and reversed inputs."""
    ops = sp[0]
    rng = np.random.default_rng(len(dims) * 1000 + n)
    idx = [rng.integers(0, d, n).astype(np.uint32) for d in dims]
    x = HostTensor(dims, idx, rng.uniform(-1, 1, n).astype(np.float32), None, False)
    N = len(dims)
    orders = [list(range(N)), list(range(N))[::-1], [(k + 1) % N for k in range(N)]]
    for mo in orders:
        dx = dev(sp, x)
        ops.sort_lexicographic(dx, mo)
        ox = x.copy()
        O.sort_lexicographic(ox, mo)
        assert same(host(dx), ox), (dims, n, mo)
        # sorted input (every warp's digits agree in the high passes) and a
        # second order from it
        mo2 = mo[::-1]
        ops.sort_lexicographic(dx, mo2)
        O.sort_lexicographic(ox, mo2)
        assert same(host(dx), ox), (dims, n, mo, "resort")


def test_tew_merge_large(sp):
    ops = sp[0]
    rng = np.random.default_rng(9)
    x = rand_tensor(rng, [200, 200, 200], 400_000, 0.5, 1.5)
    y = rand_tensor(rng, [250, 200, 190], 300_000, 0.5, 1.5)
    for op in range(3):
        dx, dy = dev(sp, x), dev(sp, y)
        ops.flops.reset()
        got = host(ops.tew(dx, dy, op))
        want, fl = O.tew(x.copy(), y.copy(), op)
        assert same(got, want), op
        assert ops.flops.count() == fl
    # already sorted under a shared non-ascending order: no re-sort
    xs, ys = x.copy(), y.copy()
    O.sort_lexicographic(xs, [2, 0, 1])
    O.sort_lexicographic(ys, [2, 0, 1])
    got = host(ops.tew(dev(sp, xs), dev(sp, ys), 0))
    want, _ = O.tew(xs, ys, 0)
    assert same(got, want) and got.sort_order == [2, 0, 1]


def test_generator_contract(sp):
    from paper_1902_03317_b200 import generate
    t = generate.coo([1000, 800, 600], 200_000, seed=5, zipf=[1.2, 0.0, 1.1], lo=0.5, hi=1.5)
    h = host(t)
    lin = (h.indices[0].astype(np.int64) * 800 + h.indices[1]) * 600 + h.indices[2]
    assert np.unique(lin).shape[0] == 200_000  # distinct tuples
    assert h.indices[0].max() < 1000 and h.indices[2].max() < 600
    assert h.values.min() >= 0.5 and h.values.max() < 1.5
    t2 = generate.coo([1000, 800, 600], 200_000, seed=5, zipf=[1.2, 0.0, 1.1], lo=0.5, hi=1.5)
    assert same(host(t2), h)  # seeded
    # Zipf mode 0 is heavy-headed, mode 1 is flat
    c0 = np.bincount(h.indices[0], minlength=1000)
    c1 = np.bincount(h.indices[1], minlength=800)
    assert c0.max() > 20 * c0.mean() and c1.max() < 3 * c1.mean()


def _wide_tensor(rng, dims, nnz, lo=0.5, hi=1.5):
    """Distinct tuples drawn mode by mode (index spaces beyond 2^63)."""
    idx = np.stack([rng.integers(0, d, size=nnz + nnz // 4, dtype=np.uint64) for d in dims], 1)
    idx = np.unique(idx, axis=0)
    rng.shuffle(idx)
    idx = idx[:nnz]
    return HostTensor(list(dims), [idx[:, d].astype(np.uint32).copy() for d in range(len(dims))],
                      rng.uniform(lo, hi, idx.shape[0]).astype(np.float32), None, True)


@pytest.mark.parametrize("dims", [
    [1 << 30, 1 << 30, 1 << 30],            # 90-bit keys: generic N-word merge
    [40000, 40000, 40000, 40000, 40000],    # 80 bits: generic
    [256] * 8,                              # exactly 64 bits, order 8: packed
    [3, 5, 7, 11],                          # tiny widths, many duplicates across x and y
])
def test_tew_key_widths(sp, dims):
    ops = sp[0]
    rng = np.random.default_rng(len(dims) * 7 + dims[0] % 97)
    cap = float(np.prod([float(d) for d in dims]))
    n = int(min(60_000, cap // 3))
    x = _wide_tensor(rng, dims, n)
    y = _wide_tensor(rng, dims, n)
    for op in range(3):
        got = host(ops.tew(dev(sp, x), dev(sp, y), op))
        want, _ = O.tew(x.copy(), y.copy(), op)
        assert same(got, want), (dims, op)


@pytest.mark.parametrize("nnz", [2047, 2048, 4096 + 5, 50_000])
def test_tew_matches_at_tile_edges(sp, nnz):
    """x and y share most tuples, so matched pairs straddle every merge tile
    boundary (the pair is split between two tiles' x and y runs)."""
    ops = sp[0]
    rng = np.random.default_rng(nnz)
    base = rand_tensor(rng, [300, 300, 300], nnz + nnz // 3, 0.5, 1.5)
    keep_x = rng.random(base.nnz) < 0.8
    keep_y = rng.random(base.nnz) < 0.8
    sub = lambda m: HostTensor(base.dims, [a[m].copy() for a in base.indices],
                               rng.uniform(0.5, 1.5, int(m.sum())).astype(np.float32), None, True)
    x, y = sub(keep_x), sub(keep_y)
    for op in range(3):
        got = host(ops.tew(dev(sp, x), dev(sp, y), op))
        want, _ = O.tew(x.copy(), y.copy(), op)
        assert same(got, want), (nnz, op)
    # identical patterns: every item of x matches
    y2 = HostTensor(x.dims, [a.copy() for a in x.indices], (x.values * 2).astype(np.float32),
                    None, True)
    for op in range(3):
        got = host(ops.tew(dev(sp, x), dev(sp, y2), op))
        want, _ = O.tew(x.copy(), y2.copy(), op)
        assert same(got, want), ("identical", nnz, op)


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("strat", ["cta", "warp"])
def test_mttkrp_tile_shapes_and_alignment(sp, offset, strat):
    """The persistent CTA-tile kernel (aligned inputs), its per-CTA fallback
    (unaligned views) and the warp-tile kernel, on partial tiles, rows that
    cross many tiles and 4th-order Zipf-like rows."""
    ops = sp[0]
    s = {"cta": ops.MTTKRP_SEGMENTED_CTA, "warp": ops.MTTKRP_SEGMENTED_WARP}[strat]
    rng = np.random.default_rng(17 + offset)
    for dims, nnz, R in (([50, 40, 30, 20], 70_001, 32), ([7, 3000, 3000], 123_457, 12),
                         ([2, 500, 400], 99_999, 16)):
        x = rand_tensor(rng, dims, nnz)
        fs = [rng.uniform(0, 1, (d, R)).astype(np.float32) for d in dims]
        for mode in (0, len(dims) - 1):
            xs = x.copy()
            O.sort_lexicographic(xs, [mode] + [d for d in range(len(dims)) if d != mode])
            _, o64, oab = O.mttkrp(xs, fs, mode)
            out = ops.mttkrp(dev(sp, xs, offset), [torch.from_numpy(f).cuda() for f in fs], mode,
                             s).cpu().numpy()
            ok, worst = within_tol(out, o64, oab)
            assert ok, (dims, mode, worst)


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("R", [3, 8, 20, 64])
def test_ttv_ttm_warp_tiles_orders(sp, R, offset):
    """Warp-tile TTV/TTM at orders 2-4, ragged warp tiles, fibers of every
    length from 1 to thousands, R that is not a multiple of 4, and unaligned
    index/value views (scalar staging and head-flag paths)."""
    ops = sp[0]
    rng = np.random.default_rng(R + 101)
    for dims, nnz in (([3000, 40], 50_003), ([30, 40, 2000], 77_777), ([9, 8, 7, 600], 123_001)):
        x = rand_tensor(rng, dims, nnz, -1, 1)
        N = len(dims)
        for mode in range(N):
            xs = x.copy()
            O.sort_lexicographic(xs, [d for d in range(N) if d != mode] + [mode])
            dx = dev(sp, xs, offset)
            v = rng.uniform(-1, 1, dims[mode]).astype(np.float32)
            zt, y64, yab = O.ttv(xs, v, mode)
            g = host(ops.ttv(dx, torch.from_numpy(v).cuda(), mode))
            assert same(HostTensor(g.dims, g.indices, zt.values, g.sort_order, g.coalesced), zt)
            assert within_tol(g.values, y64, yab)[0], (dims, mode)
            u = rng.uniform(-1, 1, (dims[mode], R)).astype(np.float32)
            zm, y64, yab = O.ttm(xs, u, mode)
            g = host(ops.ttm(dx, torch.from_numpy(u).cuda(), mode))
            assert same(HostTensor(g.dims, g.indices, zm.values, g.sort_order, g.coalesced), zm)
            assert within_tol(g.values, y64, yab)[0], (dims, mode, R)


@pytest.mark.parametrize("R", [130, 200])
def test_ttm_mttkrp_many_column_blocks(sp, R):
    """R beyond one launch's column block (float4 lanes: 128 columns, scalar
    lanes: 32): several launches, each emitting its own column slice of the
    values and of the TTM index rows."""
    ops = sp[0]
    rng = np.random.default_rng(R)
    x = rand_tensor(rng, [50, 40, 300], 20_000, -1, 1)
    for mode in range(3):
        xs = x.copy()
        O.sort_lexicographic(xs, [d for d in range(3) if d != mode] + [mode])
        u = rng.uniform(-1, 1, (x.dims[mode], R)).astype(np.float32)
        zm, y64, yab = O.ttm(xs, u, mode)
        g = host(ops.ttm(dev(sp, xs), torch.from_numpy(u).cuda(), mode))
        assert same(HostTensor(g.dims, g.indices, zm.values, g.sort_order, g.coalesced), zm)
        assert within_tol(g.values, y64, yab)[0], (R, mode)
    xs = x.copy()
    O.sort_lexicographic(xs, [0, 1, 2])
    fs = [rng.uniform(0, 1, (d, R)).astype(np.float32) for d in x.dims]
    _, o64, oab = O.mttkrp(xs, fs, 0)
    out = ops.mttkrp(dev(sp, xs), [torch.from_numpy(f).cuda() for f in fs], 0).cpu().numpy()
    assert np.all(np.abs(out - o64) <= TOL * np.maximum(np.abs(o64), oab) + 1e-30)
