import numpy as np, sys
sys.path.insert(0, '.')
from oracle.oracle import Oracle, Ref, HostTensor
O, R = Oracle(), Ref()
print("threads", R.max_threads())
def same(a, b):
    return a.dims == b.dims and all((p == q).all() for p, q in zip(a.indices, b.indices)) and (a.values.view(np.uint32) == b.values.view(np.uint32)).all() and a.sort_order == b.sort_order and a.coalesced == b.coalesced
rng = np.random.default_rng(0)
for seed in range(30):
    N = 3 + seed % 2
    dims = list(rng.integers(2, 16, N))
    cap = int(np.prod(dims)); nnz = max(1, int(cap * rng.uniform(0.05, 0.5)))
    x = R.gen_synthetic(dims, nnz, seed); y = x.copy(); y.values = rng.uniform(1, 2, nnz).astype(np.float32)
    for op in range(2): assert same(O.ts(x, 2.5, op), R.ts(x, 2.5, op))
    for op in range(4): assert same(O.tew_eq(x, y, op), R.tew_eq(x, y, op)), op
    y2 = R.gen_synthetic(dims, nnz, seed + 1000)
    for op in range(3):
        zr, xr, yr, flr = R.tew(x.copy(), y2.copy(), op)
        xo, yo = x.copy(), y2.copy(); zo, flo = O.tew(xo, yo, op)
        assert same(zo, zr) and same(xo, xr) and same(yo, yr) and flo == flr, (seed, op)
    for mode in range(N):
        mo = [d for d in range(N) if d != mode] + [mode]
        xs = R.sort_lexicographic(x, mo); xo = x.copy(); O.sort_lexicographic(xo, mo); assert same(xs, xo)
        assert (R.build_fiber_index(xs, mode) == O.build_fiber_index(xo, mode)).all()
        v = rng.uniform(-1, 1, dims[mode]).astype(np.float32)
        assert same(R.ttv(xs, v, mode), O.ttv(xo, v, mode)[0])
        u = rng.uniform(-1, 1, (dims[mode], 5)).astype(np.float32)
        assert same(R.ttm(xs, u, mode), O.ttm(xo, u, mode)[0])
        F = [rng.uniform(0, 1, (dims[d], 7)).astype(np.float32) for d in range(N)]
        a = R.mttkrp(x, F, mode); b = O.mttkrp(x, F, mode)[0]
        assert (a.view(np.uint32) == b.view(np.uint32)).all()
    # coalesce with duplicates
    xd = x.copy(); k = min(5, nnz); 
    xd = HostTensor(dims, [np.concatenate([i, i[:k]]) for i in x.indices], np.concatenate([x.values, x.values[:k]]), None, False)
    assert same(R.coalesce(xd), O.coalesce(xd))
print("oracle == reference on 30 random instances")
