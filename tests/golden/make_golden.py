"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the dev container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
Every expected output below is produced by the reference library itself
(spten::seq::*, sort_lexicographic, coalesce, build_fiber_index compiled from
/root/reference/proj/src by oracle/Makefile), never by code in this repo.

Inputs:
  * the reference unit tests' hand examples (P/tests/test_kernels_seq.cpp,
    P/tests/test_tensor.cpp; line numbers in KATS below);
  * random instances from the reference's own generator gen_synthetic
    (P/src/io.cpp:151-244) in the acceptance envelope of
    P/tests/acceptance.cpp:48-69 (order 3-4, extents 2..16, density
    0.05-0.5, R in {1, 8, 16}), seeds 1000+i as in acceptance criterion 1.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import HostTensor, Ref  # noqa: E402

ADD, SUB, MUL, DIV = 0, 1, 2, 3


def lit(dims, entries, sorted_coalesced=False):
    """make_tensor (P/tests/test_util.hpp:20-31)."""
    N = len(dims)
    idx = [np.array([e[0][d] for e in entries], np.uint32) for d in range(N)]
    vals = np.array([e[1] for e in entries], np.float32)
    return HostTensor(dims, idx, vals, list(range(N)) if sorted_coalesced else None,
                      sorted_coalesced)


class Store:
    def __init__(self):
        self.arrays = {}
        self.n = 0

    def put_tensor(self, key, t: HostTensor):
        self.arrays[f"{key}.dims"] = np.array(t.dims, np.uint32)
        for d, a in enumerate(t.indices):
            self.arrays[f"{key}.idx{d}"] = a
        self.arrays[f"{key}.val"] = t.values
        self.arrays[f"{key}.sort"] = np.array(t.sort_order if t.sort_order is not None else [],
                                              np.int32)
        self.arrays[f"{key}.coal"] = np.array([1 if t.coalesced else 0], np.int32)

    def put(self, key, a):
        self.arrays[key] = np.asarray(a)

    def save(self, name):
        np.savez_compressed(os.path.join(HERE, name), **self.arrays)


def instance(ref: Ref, rng: np.random.Generator, max_dim=16):
    N = 3 + int(rng.integers(0, 2))
    dims = [int(rng.integers(2, max_dim + 1)) for _ in range(N)]
    cap = int(np.prod(dims))
    nnz = min(cap, max(1, int(round(rng.uniform(0.05, 0.5) * cap))))
    return ref.gen_synthetic(dims, nnz, int(rng.integers(0, 2**62)))


def main():
    ref = Ref()
    rng = np.random.default_rng(20190210)

    # ---- elementwise: ts, tew_eq, tew ------------------------------------
    s = Store()
    k = 0
    # KATs: test_kernels_seq.cpp:81-85 (div by stored zero), :87-102 (disjoint),
    # :104-109 (shape unify), :137-144 (sub negation).
    kat_x = lit([2, 2], [((0, 0), 1.0), ((1, 1), 2.0)])
    kat_y = lit([2, 2], [((0, 0), 4.0), ((1, 1), 0.0)])
    s.put_tensor("tew_eq_err0.x", kat_x)
    s.put_tensor("tew_eq_err0.y", kat_y)
    s.put("tew_eq_err0.op", DIV)
    s.put("tew_eq_err0.expect", "domain_error")
    tews = [
        (lit([1, 1, 2], [((0, 0, 0), 1.0)], True), lit([1, 1, 2], [((0, 0, 1), 2.0)], True)),
        (lit([2, 3], [((1, 2), 1.0)], True), lit([4, 2], [((3, 0), 2.0)], True)),
        (lit([2, 2], [((0, 0), 5.0)], True), lit([2, 2], [((0, 0), 2.0), ((1, 1), 3.0)], True)),
    ]
    for i in range(24):
        x = instance(ref, rng, max_dim=12)
        y = x.copy()
        y.values = rng.uniform(1.0, 2.0, x.nnz).astype(np.float32)
        if i % 7 == 3:  # a stored zero divisor in the middle
            y.values[x.nnz // 2] = 0.0
        key = f"ew{i}"
        s.put_tensor(f"{key}.x", x)
        s.put_tensor(f"{key}.y", y)
        for op in (ADD, SUB, MUL, DIV):
            try:
                s.put(f"{key}.tew_eq{op}", ref.tew_eq(x, y, op).values)
                s.put(f"{key}.tew_eq{op}.expect", "ok")
            except ArithmeticError as e:
                s.put(f"{key}.tew_eq{op}.expect", "domain_error")
                s.put(f"{key}.tew_eq{op}.msg", str(e))
        for op, sc in ((0, 2.5), (1, 2.5), (1, 1.0), (0, 0.0)):
            z = ref.ts(x, sc, op)
            assert all((a == b).all() for a, b in zip(z.indices, x.indices))
            s.put(f"{key}.ts{op}_{sc}", z.values)
        # independent pattern over the same space (partial overlap), unsorted
        if i < 12:
            y2 = ref.gen_synthetic(x.dims, x.nnz, int(rng.integers(0, 2**62)))
            tews.append((x, y2))
    s.put("n_ew", 24)
    for j, (x, y) in enumerate(tews):
        for op in (ADD, SUB, MUL):
            key = f"tew{j}_{op}"
            z, xa, ya, fl = ref.tew(x.copy(), y.copy(), op)
            s.put_tensor(f"{key}.x", x)
            s.put_tensor(f"{key}.y", y)
            s.put(f"{key}.op", op)
            s.put_tensor(f"{key}.z", z)
            s.put(f"{key}.xa_sort", np.array(xa.sort_order, np.int32))
            s.put(f"{key}.flops", fl)
    s.put("n_tew", len(tews))
    s.save("elementwise.npz")

    # ---- preprocessing: sort, coalesce, fiber index ------------------------
    s = Store()
    # KATs: test_tensor.cpp:22-33 (sort), :60-65 (stability), :82-89 (coalesce),
    # :120-128 (exact-zero sums kept), :148-155 (fiber index [0,2,3]).
    cases = [
        (lit([2, 2, 2], [((1, 0, 0), 1.0), ((0, 1, 0), 2.0), ((0, 0, 1), 3.0)]), [0, 1, 2]),
        (lit([2, 2], [((1, 1), 1.0), ((0, 0), 2.0), ((1, 1), 3.0), ((0, 0), 4.0)]), [0, 1]),
        (lit([1, 1, 1], [((0, 0, 0), 1.0), ((0, 0, 0), 2.0)]), [0, 1, 2]),
        (lit([2, 2], [((1, 0), 1.0), ((1, 0), -1.0), ((0, 1), 5.0)]), [0, 1]),
        (lit([2, 1, 3], [((0, 0, 0), 1.0), ((0, 0, 2), 2.0), ((1, 0, 1), 3.0)]), [0, 1, 2]),
    ]
    for i in range(40):
        x = instance(ref, rng)
        # scramble storage order, add a few duplicate tuples
        perm = rng.permutation(x.nnz)
        dup = rng.integers(0, x.nnz, size=min(5, x.nnz))
        idx = [np.concatenate([a[perm], a[dup]]) for a in x.indices]
        vals = np.concatenate([x.values[perm], rng.uniform(-1, 1, dup.shape[0]).astype(np.float32)])
        t = HostTensor(x.dims, idx, vals, None, False)
        cases.append((t, [int(m) for m in rng.permutation(x.order)]))
    for j, (t, mo) in enumerate(cases):
        key = f"pre{j}"
        s.put_tensor(f"{key}.x", t)
        s.put(f"{key}.mo", np.array(mo, np.uint32))
        srt = ref.sort_lexicographic(t, mo)
        s.put_tensor(f"{key}.sorted", srt)
        s.put_tensor(f"{key}.coalesced", ref.coalesce(srt))
        c = ref.coalesce(srt)
        last = mo[-1]
        s.put(f"{key}.fptr", ref.build_fiber_index(c, last))
    s.put("n_pre", len(cases))
    s.save("preprocess.npz")

    # ---- reductions: ttv, ttm, mttkrp --------------------------------------
    s = Store()
    # KATs: test_kernels_seq.cpp:188-202 (ttv -> 50, 30), :253-265 (ttm -> 7, 10),
    # :313-330 (mttkrp row 1 = [12, 30]).
    s.put_tensor("kat_ttv.x", lit([2, 2, 2], [((0, 0, 0), 1.0), ((0, 0, 1), 2.0),
                                              ((1, 1, 0), 3.0)], True))
    s.put("kat_ttv.v", np.array([10.0, 20.0], np.float32))
    s.put_tensor("kat_ttm.x", lit([1, 1, 2], [((0, 0, 0), 1.0), ((0, 0, 1), 2.0)], True))
    s.put("kat_ttm.u", np.array([[1.0, 2.0], [3.0, 4.0]], np.float32))
    s.put_tensor("kat_mttkrp.x", lit([2, 3, 1], [((1, 2, 0), 3.0)], True))
    f1 = np.zeros((3, 2), np.float32)
    f1[2] = [1.0, 2.0]
    f2 = np.array([[4.0, 5.0]], np.float32)
    s.put("kat_mttkrp.f0", np.zeros((2, 2), np.float32))
    s.put("kat_mttkrp.f1", f1)
    s.put("kat_mttkrp.f2", f2)
    kx = lit([2, 2, 2], [((0, 0, 0), 1.0), ((0, 0, 1), 2.0), ((1, 1, 0), 3.0)], True)
    s.put_tensor("kat_ttv.z", ref.ttv(kx, np.array([10.0, 20.0], np.float32), 2))
    s.put_tensor("kat_ttm.z", ref.ttm(lit([1, 1, 2], [((0, 0, 0), 1.0), ((0, 0, 1), 2.0)], True),
                                      np.array([[1.0, 2.0], [3.0, 4.0]], np.float32), 2))
    s.put("kat_mttkrp.out", ref.mttkrp(lit([2, 3, 1], [((1, 2, 0), 3.0)], True),
                                       [np.zeros((2, 2), np.float32), f1, f2], 0))
    n = 0
    for i in range(40):
        x = instance(ref, rng)
        N = x.order
        R = [1, 8, 16][i % 3]
        mode = int(rng.integers(0, N))
        key = f"red{n}"
        mo = [d for d in range(N) if d != mode] + [mode]
        xs = ref.sort_lexicographic(x, mo)
        s.put_tensor(f"{key}.x", xs)
        s.put(f"{key}.mode", mode)
        v = rng.uniform(-1, 1, x.dims[mode]).astype(np.float32)
        u = rng.uniform(-1, 1, (x.dims[mode], R)).astype(np.float32)
        s.put(f"{key}.v", v)
        s.put(f"{key}.u", u)
        s.put_tensor(f"{key}.ttv", ref.ttv(xs, v, mode))
        s.put_tensor(f"{key}.ttm", ref.ttm(xs, u, mode))
        fs = [rng.uniform(0.5, 1.5, (x.dims[d], R)).astype(np.float32) for d in range(N)]
        for d in range(N):
            s.put(f"{key}.f{d}", fs[d])
        s.put(f"{key}.mttkrp", ref.mttkrp(x, fs, mode))  # unsorted input, any order works
        s.put_tensor(f"{key}.xu", x)
        n += 1
    s.put("n_red", n)
    s.save("reductions.npz")
    print("golden fixtures written:", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
