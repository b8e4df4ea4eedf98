"""CP-ALS driver (paper_1902_03317_b200/cpals.py) on the GPU kernels, against
a plain numpy CP-ALS that uses the oracle's fp64 MTTKRP, from the same init."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.oracle import HostTensor, Oracle

pytestmark = pytest.mark.gpu


def _np_cpals(x: HostTensor, init, iters):
    O = Oracle()
    N = x.order
    U = [u.astype(np.float64).copy() for u in init]
    lam = None
    for _ in range(iters):
        for n in range(N):
            M = O.mttkrp(x, [u.astype(np.float32) for u in U], n)[1]
            V = np.ones((U[0].shape[1],) * 2)
            for m in range(N):
                if m != n:
                    V *= U[m].T @ U[m]
            Un = M @ np.linalg.pinv(V)
            lam = np.linalg.norm(Un, axis=0)
            lam[lam == 0] = 1
            U[n] = (Un / lam).astype(np.float32).astype(np.float64)
    return lam, U


def test_cpals_matches_numpy_reference():
    from paper_1902_03317_b200.coo import HostCOO
    from paper_1902_03317_b200.cpals import cp_als
    rng = np.random.default_rng(0)
    dims, R, nnz = [40, 30, 20], 4, 6000
    lin = rng.choice(int(np.prod(dims)), nnz, replace=False)
    idx = []
    for d in reversed(dims):
        idx.append((lin % d).astype(np.uint32))
        lin //= d
    idx = idx[::-1]
    vals = rng.uniform(0, 1, nnz).astype(np.float32)
    x = HostTensor(dims, idx, vals, None, True)
    init = [rng.uniform(0, 1, (d, R)).astype(np.float32) for d in dims]
    lam_ref, U_ref = _np_cpals(x, init, 3)
    dx = HostCOO(dims, idx, vals, None, True).to_device(0)
    res = cp_als(dx, R, iters=3, tol=0.0, init=[torch.from_numpy(u) for u in init])
    assert res.iterations == 3
    np.testing.assert_allclose(res.weights.cpu().numpy(), lam_ref, rtol=1e-3)
    for a, b in zip(res.factors, U_ref):
        np.testing.assert_allclose(a.cpu().numpy(), b, rtol=1e-3, atol=1e-4)


def test_cpals_recovers_exact_low_rank_dense_tensor():
    """Every entry stored (dense pattern) of an exact rank-3 tensor: fit -> 1."""
    from paper_1902_03317_b200.coo import HostCOO
    from paper_1902_03317_b200.cpals import cp_als
    rng = np.random.default_rng(1)
    dims, R = [12, 10, 8], 3
    A = [rng.uniform(0.5, 1.5, (d, R)) for d in dims]
    full = np.einsum("ir,jr,kr->ijk", *A).astype(np.float32)
    I, J, K = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
    x = HostCOO(dims, [I.ravel().astype(np.uint32), J.ravel().astype(np.uint32),
                       K.ravel().astype(np.uint32)], full.ravel(), [0, 1, 2], True).to_device(0)
    res = cp_als(x, R, iters=1000, tol=1e-12, seed=3)
    assert res.fits[-1] > 0.999, res.fits[-5:]
