"""Parity at BASELINE.json's full sizes (the oracle-sized cases live in
test_gpu_parity.py). Too large for the CPU oracle, so each check is a
size-independent property or an on-device recomputation:

* TS, TEW-eq: bit-exact against one IEEE fp32 torch op per stored value
  (the reference's apply_scalar / apply_elem, P/src/kernel_detail.hpp:19-32),
  indices identical to x's;
* TEW merge (C2b, 10M + 10M independent patterns): output keys strictly
  increasing (sorted, coalesced), the key set equals the union (add) /
  intersection (mul) of the input key sets, matched values bit-exact x op y,
  unmatched values copied bit-exactly;
* sort: non-decreasing keys and the same multiset of tuples (sorted keys equal);
* MTTKRP (C4, 100M nnz, R=32, every mode; C5, 1B nnz, R=32, modes 0-2, the
  plan kernel the bench runs and the segmented kernel), TTV and TTM (C3, 50M,
  every mode): per output entry within TOL = 1e-5 of an fp64 recomputation
  (chunked torch index_add over the same fp32 inputs),
  |y - y64| <= TOL * max(|y64|, sum|terms|); rows without entries exactly 0;
* C5 TEW-eq mul (1B nnz): bit-exact against one IEEE fp32 multiply per value;
* the C5 row-aligned sharding of bench.py --gpus G (G = 2, 4, 8) emulated on
  one GPU: each shard's plan run in turn, the owned row blocks assembled, the
  result within the same 1e-5 rule and every row written by its owner only.
"""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
TOL = 1e-5
CHUNK = 4_000_000


@pytest.fixture(scope="module")
def lib():
    from paper_1902_03317_b200 import _lib, generate, ops
    assert _lib.missing_symbols() == []
    return ops, generate


def u32(t):
    return t.to(torch.int64) & 0xFFFFFFFF


def keys(t, order=None):
    """Linearised tuples (int64; the configs' index spaces fit 63 bits)."""
    order = order if order is not None else list(range(len(t.dims)))
    k = torch.zeros(t.nnz, dtype=torch.int64, device=t.values.device)
    for d in order:
        k = k * int(t.dims[d]) + u32(t.indices[d][: t.nnz])
    return k


def bits(v):
    return v.contiguous().view(torch.int32)


def test_c1_ts_full(lib):
    ops, gen = lib
    x = gen.config_tensor("c1", seed=11, sort_order=[0, 1, 2])
    s = torch.tensor(2.5, dtype=torch.float32, device="cuda")
    for op, ref in ((ops.SCALAR_ADD, x.values + s), (ops.SCALAR_MUL, x.values * s)):
        z = ops.ts(x, 2.5, op)
        assert torch.equal(bits(z.values), bits(ref))
        assert all(torch.equal(a, b) for a, b in zip(z.indices, x.indices))


def test_c2_tew_eq_full(lib):
    ops, gen = lib
    x = gen.config_tensor("c2", seed=21, sort_order=[0, 1, 2])
    y = x.clone()
    y.values = gen.uniform(x.nnz, 22, 7, 0.5, 1.5)
    for op, f in ((ops.ADD, torch.add), (ops.SUB, torch.sub), (ops.MUL, torch.mul),
                  (ops.DIV, torch.div)):
        z = ops.tew_eq(x, y, op)
        assert torch.equal(bits(z.values), bits(f(x.values, y.values))), op
        assert all(torch.equal(a, b) for a, b in zip(z.indices, x.indices))


def test_c2_tew_merge_full(lib):
    ops, gen = lib
    x = gen.config_tensor("c2", seed=31, sort_order=[0, 1, 2])
    y = gen.config_tensor("c2", seed=32, sort_order=[0, 1, 2])
    kx, ky = keys(x), keys(y)  # independent patterns: ~100 tuples match by chance
    for op in (ops.ADD, ops.MUL):
        z = ops.tew(x, y, op)
        kz = keys(z)
        assert bool((kz[1:] > kz[:-1]).all()), "output keys strictly increasing"
        inter = kx[torch.isin(kx, ky)]
        if op == ops.ADD:
            assert z.nnz == x.nnz + y.nnz - inter.numel()
        else:
            assert z.nnz == inter.numel() and torch.equal(kz, inter)
        # values: locate each output key in x and y
        ix = torch.searchsorted(kx, kz).clamp(max=x.nnz - 1)
        iy = torch.searchsorted(ky, kz).clamp(max=y.nnz - 1)
        inx, iny = kx[ix] == kz, ky[iy] == kz
        assert bool((inx | iny).all())
        xv, yv = x.values[ix], y.values[iy]
        both = inx & iny
        want = torch.where(both, xv + yv if op == ops.ADD else xv * yv,
                           torch.where(inx, xv, yv))
        assert torch.equal(bits(z.values[: z.nnz]), bits(want)), op


def test_c2_sort_full(lib):
    ops, gen = lib
    x = gen.config_tensor("c2", seed=41)  # draw order
    k0 = keys(x)
    ops.sort_lexicographic(x, [2, 0, 1])
    k = keys(x, [2, 0, 1])
    assert bool((k[1:] >= k[:-1]).all())
    k0p = keys(x)  # the same multiset of tuples as before the sort
    assert int(k0.sum()) == int(k0p.sum())
    assert torch.equal(torch.sort(k0).values, torch.sort(k0p).values)


def _mttkrp64(x, fs, mode):
    """fp64 out(i, :) += val * prod_{d != mode} F_d(i_d, :), in chunks; also
    the sum of |terms| (equal to out for these all-positive inputs)."""
    R = fs[0].shape[1]
    out = torch.zeros((x.dims[mode], R), dtype=torch.float64, device="cuda")
    for a in range(0, x.nnz, CHUNK):
        b = min(x.nnz, a + CHUNK)
        t = x.values[a:b].to(torch.float64)[:, None].expand(-1, R).clone()
        for d in range(len(x.dims)):
            if d != mode:
                t *= fs[d][u32(x.indices[d][a:b])].to(torch.float64)
        out.index_add_(0, u32(x.indices[mode][a:b]), t)
    return out


def _check_mttkrp(got, want):
    got = got.to(torch.float64)
    assert bool(((got - want).abs() <= TOL * want.abs()).all())
    assert bool((got[want == 0] == 0).all())  # rows without entries are exact zeros


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_c4_mttkrp_full(lib, mode):
    ops, gen = lib
    c = gen.CONFIGS["c4"]
    x = gen.config_tensor("c4", seed=51, sort_order=[mode] + [d for d in range(4) if d != mode])
    fs = [gen.uniform((d, c["R"]), 51, 100 + k, 0.0, 1.0) for k, d in enumerate(c["dims"])]
    want = _mttkrp64(x, fs, mode)
    _check_mttkrp(ops.mttkrp(x, fs, mode, ops.MTTKRP_SEGMENTED), want)
    plan = ops.mttkrp_plan(x, mode, c["R"])
    _check_mttkrp(ops.mttkrp(plan, fs, mode), want)


@pytest.mark.parametrize("dims,nnz,R,zipf", [
    ([1000, 1000, 1000], 1_000_000, 16, [0, 0, 0]),        # C1: one staged chunk per share
    ([5000, 3000, 700], 2_500_003, 16, [1.1, 0, 0]),        # several chunks per share, heavy rows
    ([200_000, 900, 800], 700_001, 32, [0, 0, 0]),          # ~3.5 entries per row, empty rows
    ([3, 50_000, 40_000], 1_200_000, 64, [0, 0, 0]),        # three rows spanning every share
    ([40_000, 600, 500, 30], 900_000, 8, [1.1, 0, 0, 0]),   # order 4, R = 8
    ([1000, 1000], 3000, 128, [0, 0]),                      # short rows: the tiled kernel's case
    ([50, 2000], 3000, 128, [0, 0]),                        # fewer entries than shares x 4
    ([2000, 5000, 3000], 8_000_000, 16, [1.1, 0, 0]),       # a heavy row over hundreds of shares
    ([300, 4000, 3000], 6_000_000, 64, [1.3, 0, 0]),        # the same with two warps per slot
])
def test_mttkrp_onewave(lib, dims, nnz, R, zipf):
    """The one-wave small-input MTTKRP (default segmented path up to 3M
    entries) against the fp64 recomputation and the tiled kernel."""
    ops, gen = lib
    N = len(dims)
    for mode in (0, N - 1):
        order = [mode] + [d for d in range(N) if d != mode]
        x = gen.coo(dims, nnz, 77, zipf, 0.0, 1.0, order)
        fs = [gen.uniform((d, R), 77, 300 + k, 0.0, 1.0) for k, d in enumerate(dims)]
        want = _mttkrp64(x, fs, mode)
        got = ops.mttkrp(x, fs, mode, ops.MTTKRP_SEGMENTED)
        _check_mttkrp(got, want)
        again = ops.mttkrp(x, fs, mode, ops.MTTKRP_SEGMENTED)
        assert torch.equal(got, again)  # fixed shares and summation orders
        _check_mttkrp(ops.mttkrp(x, fs, mode, ops.MTTKRP_SEGMENTED_CTA), want)


def test_mttkrp_onewave_unsorted(lib):
    ops, gen = lib
    x = gen.coo([500, 400, 300], 200_000, 5, [0, 0, 0], 0.0, 1.0, [0, 1, 2])
    fs = [gen.uniform((d, 16), 5, 10 + k, 0.0, 1.0) for k, d in enumerate(x.dims)]
    i0 = x.indices[0]
    i0[100_000], i0[100_001] = i0[100_001].clone() + 3, i0[100_000].clone()
    x.sort_order = [0, 1, 2]
    with pytest.raises(Exception, match="sorted by the output mode"):
        ops.mttkrp(x, fs, 0, ops.MTTKRP_SEGMENTED)


@pytest.fixture(scope="module")
def c5(lib):
    ops, gen = lib
    c = gen.CONFIGS["c5"]
    x = gen.config_tensor("c5", seed=81, sort_order=[0, 1, 2])
    fs = [gen.uniform((d, c["R"]), 81, 100 + k, 0.0, 1.0) for k, d in enumerate(c["dims"])]
    return x, fs, c["R"]


def test_c5_tew_eq_mul_full(lib, c5):
    ops, gen = lib
    x, _, _ = c5
    y = type(x)(list(x.dims), x.indices, gen.uniform(x.nnz, 81, 77, 0.5, 1.5), list(x.sort_order),
                True)
    z = ops.tew_eq(x, y, ops.MUL)
    assert torch.equal(bits(z.values), bits(x.values * y.values))
    assert all(torch.equal(a, b) for a, b in zip(z.indices, x.indices))


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_c5_mttkrp_full(lib, c5, mode):
    """1B entries, 10M-row Zipf(1.1) outputs: rows spanning many CTAs (the
    grid fold), u32 offsets near 2^30."""
    ops, gen = lib
    x, fs, R = c5
    want = _mttkrp64(x, fs, mode)
    plan = ops.mttkrp_plan(x, mode, R)
    _check_mttkrp(ops.mttkrp(plan, fs, mode), want)
    del plan
    torch.cuda.empty_cache()
    if mode == 0:  # the segmented kernel on the mode-leading input it needs
        _check_mttkrp(ops.mttkrp(x, fs, 0, ops.MTTKRP_SEGMENTED), want)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_c5_row_aligned_shards(lib, c5, G):
    """bench.py's C5 strong-scaling split (parallel.row_aligned_ranges /
    row_blocks, one plan per shard) run shard by shard on one GPU."""
    from paper_1902_03317_b200 import parallel
    ops, gen = lib
    x, fs, R = c5
    mode = 0
    want = _mttkrp64(x, fs, mode)
    rr = parallel.row_aligned_ranges(x.indices[mode], G)
    blocks = parallel.row_blocks(x.indices[mode], rr, x.dims[mode])
    assert rr[0][0] == 0 and rr[-1][1] == x.nnz
    assert all(a[1] == b[0] for a, b in zip(rr[:-1], rr[1:]))
    assert blocks[0][0] == 0 and blocks[-1][1] == x.dims[mode]
    out = torch.full((x.dims[mode], R), float("nan"), device="cuda")
    for (lo, hi), (a, b) in zip(rr, blocks):
        if hi == lo:
            continue
        shard = parallel.slice_coo(x, lo, hi).clone()
        plan = ops.mttkrp_plan(shard, mode, R)
        part = ops.mttkrp(plan, fs, mode)
        # a shard's rows are exact; everything outside its block is zero
        assert bool((part[:a] == 0).all()) and bool((part[b:] == 0).all())
        out[a:b] = part[a:b]
        del plan, shard, part
        torch.cuda.empty_cache()
    _check_mttkrp(out, want)


def _fiber_ids(x, fib):
    f = torch.arange(fib.nfibs, device="cuda", dtype=torch.int64)
    fptr = u32(fib.fptr)
    return torch.repeat_interleave(f, fptr[1:] - fptr[:-1], output_size=x.nnz)


def test_c3_ttv_full(lib):
    ops, gen = lib
    c = gen.CONFIGS["c3"]
    base = gen.config_tensor("c3", seed=61)
    for mode in range(3):
        x = base.clone()
        ops.sort_lexicographic(x, ops.mode_last_order(3, mode))
        fib = ops.build_fiber_index(x, mode)
        v = gen.uniform(c["dims"][mode], 61, 200 + mode, -1.0, 1.0)
        z = ops.ttv(x, v, mode, fib)
        fid = _fiber_ids(x, fib)
        term = x.values.to(torch.float64) * v[u32(x.indices[mode])].to(torch.float64)
        y64 = torch.zeros(fib.nfibs, dtype=torch.float64, device="cuda").index_add_(0, fid, term)
        yab = torch.zeros_like(y64).index_add_(0, fid, term.abs())
        err = (z.values[: fib.nfibs].to(torch.float64) - y64).abs()
        assert bool((err <= TOL * torch.maximum(y64.abs(), yab)).all()), mode
        heads = u32(fib.fptr[:-1])
        others = [d for d in range(3) if d != mode]
        for j, d in enumerate(others):  # output tuple = the fiber head's non-mode indices
            assert torch.equal(z.indices[j][: fib.nfibs], x.indices[d][heads]), (mode, d)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_c3_ttm_full(lib, mode):
    ops, gen = lib
    c = gen.CONFIGS["c3"]
    R = c["R"]
    x = gen.config_tensor("c3", seed=71)
    ops.sort_lexicographic(x, ops.mode_last_order(3, mode))
    fib = ops.build_fiber_index(x, mode)
    u = gen.uniform((c["dims"][mode], R), 71, 300, -1.0, 1.0)
    z = ops.ttm(x, u, mode, fib)
    fid = _fiber_ids(x, fib)
    y64 = torch.zeros((fib.nfibs, R), dtype=torch.float64, device="cuda")
    yab = torch.zeros_like(y64)
    for a in range(0, x.nnz, CHUNK):
        b = min(x.nnz, a + CHUNK)
        t = x.values[a:b].to(torch.float64)[:, None] * u[u32(x.indices[mode][a:b])].to(torch.float64)
        y64.index_add_(0, fid[a:b], t)
        yab.index_add_(0, fid[a:b], t.abs())
    got = z.values[: fib.nfibs * R].view(fib.nfibs, R).to(torch.float64)
    assert bool(((got - y64).abs() <= TOL * torch.maximum(y64.abs(), yab)).all())
    r = torch.arange(R, device="cuda", dtype=torch.int32).repeat(fib.nfibs)
    assert torch.equal(z.indices[mode][: fib.nfibs * R], r)  # mode index = column
    heads = u32(fib.fptr[:-1])
    for d in range(3):  # other index rows: the fiber head's index, repeated R times
        if d != mode:
            want = x.indices[d][heads].repeat_interleave(R)
            assert torch.equal(z.indices[d][: fib.nfibs * R], want), (mode, d)
