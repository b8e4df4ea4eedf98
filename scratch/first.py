import numpy as np, torch, time
from paper_1902_03317_b200 import ops
from paper_1902_03317_b200.coo import HostCOO
rng = np.random.default_rng(1)
def rand_coo(dims, nnz):
    lin = rng.choice(int(np.prod(dims)), size=nnz, replace=False)
    idx = []
    for d in reversed(dims):
        idx.append((lin % d).astype(np.uint32)); lin //= d
    idx = idx[::-1]
    return HostCOO(list(dims), idx, rng.random(nnz, dtype=np.float32), None, True)
x = rand_coo([50, 60, 70], 20001)
dx = x.to_device(0)
z = ops.ts(dx, 2.5, ops.SCALAR_MUL).to_host()
assert all((a == b).all() for a, b in zip(z.indices, x.indices)); assert (z.values == x.values * np.float32(2.5)).all()
y = x.copy(); y.values = rng.random(x.nnz, dtype=np.float32) + np.float32(0.5)
for op in range(4):
    z = ops.tew_eq(dx, y.to_device(0), op).to_host()
    want = [x.values + y.values, x.values - y.values, x.values * y.values, x.values / y.values][op]
    assert (z.values.view(np.uint32) == want.view(np.uint32)).all(), op
y2 = y.copy(); y2.indices[1] = y2.indices[1].copy(); y2.indices[1][777] ^= 1
try:
    ops.tew_eq(dx, y2.to_device(0), 0); raise SystemExit("no error")
except ValueError as e: print("ok mismatch:", e)
y3 = y.copy(); y3.values[555] = 0; y3.values[900] = 0
try:
    ops.tew_eq(dx, y3.to_device(0), 3); raise SystemExit("no error")
except ArithmeticError as e: print("ok divzero:", e)
print("ts/tew_eq OK")
# mttkrp: sort host-side by mode
for N, dims, R in [(3, [50, 60, 70], 16), (3, [50, 60, 70], 32), (4, [40, 30, 20, 10], 8), (3, [7, 1000, 1000], 32), (3, [3000, 10, 10], 5)]:
    x = rand_coo(dims, min(200000, int(np.prod(dims)) // 3))
    F = [rng.random((d, R), dtype=np.float32) for d in dims]
    for mode in range(N):
        perm = np.lexsort([x.indices[d] for d in reversed([mode] + [d for d in range(N) if d != mode])])
        xs = HostCOO(dims, [i[perm] for i in x.indices], x.values[perm], [mode] + [d for d in range(N) if d != mode], True)
        want = np.zeros((dims[mode], R))
        prod = xs.values.astype(np.float64)[:, None] * np.ones((1, R))
        for d in range(N):
            if d != mode: prod = prod * F[d][xs.indices[d]].astype(np.float64)
        np.add.at(want, xs.indices[mode], prod)
        dF = [torch.from_numpy(f).cuda() for f in F]
        for strat in (ops.MTTKRP_SEGMENTED, ops.MTTKRP_ATOMIC):
            got = ops.mttkrp(xs.to_device(0), dF, mode, strat).cpu().numpy()
            err = np.abs(got - want).max() / np.abs(want).max()
            print(N, dims, R, mode, strat, "rel err", err)
            assert err < 1e-5
print("mttkrp OK")
