"""CP-ALS driver on the device-resident kernels ("next"
row 3: MTTKRP's caller; the reference leaves it out of scope).

Rank-R CP decomposition X ~ [[lambda; U_0, ..., U_{N-1}]] by alternating least
squares (Kolda & Bader 2009, Alg. CP-ALS): for each mode n

    M   = MTTKRP(X, U, n)                        -- sm_100a segmented kernel
    V   = *_{m != n} (U_m^T U_m)                 -- R x R Hadamard of Grams
    U_n = M V^+ ,  lambda = column norms of U_n,  U_n /= lambda

Factors stay on the device across iterations; MTTKRP consumes one
mode-leading sorted copy per mode built once up front (preprocessing, like
the reference's sort_s). The R x R algebra runs in fp64 (negligible cost).
The fit uses ||X||^2, <X, model> = sum_r lambda_r (M_last * U_last)_r and
||model||^2 = lambda^T (*_m U_m^T U_m) lambda, so it needs no extra pass over X.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import torch

from . import generate, ops
from .coo import DeviceCOO


@dataclass
class CPResult:
    weights: torch.Tensor  # lambda, (R,)
    factors: List[torch.Tensor]  # U_n, (I_n, R) fp32, unit-norm columns
    fits: List[float]  # fit after each iteration
    iterations: int


def cp_als(x: DeviceCOO, rank: int, iters: int = 20, tol: float = 1e-5, seed: int = 0,
           init: Optional[List[torch.Tensor]] = None,
           sorted_copies: Optional[List[DeviceCOO]] = None) -> CPResult:
    N = x.order
    dev = x.device
    if sorted_copies is None:
        sorted_copies = []
        for n in range(N):
            xs = x.clone()
            ops.sort_lexicographic(xs, [n] + [d for d in range(N) if d != n])
            sorted_copies.append(xs)
    if init is None:
        U = [generate.uniform((x.dims[n], rank), seed, 500 + n, 0.0, 1.0,
                              dev.index or 0) for n in range(N)]
    else:
        U = [u.to(dev, torch.float32).contiguous().clone() for u in init]
    grams = [(u.double().T @ u.double()) for u in U]
    normx2 = float((x.values.double() ** 2).sum())
    lam = torch.ones(rank, dtype=torch.float64, device=dev)
    fits: List[float] = []
    it = 0
    for it in range(1, iters + 1):
        for n in range(N):
            M = ops.mttkrp(sorted_copies[n], U, n, ops.MTTKRP_SEGMENTED).double()
            V = torch.ones((rank, rank), dtype=torch.float64, device=dev)
            for m in range(N):
                if m != n:
                    V = V * grams[m]
            Un = M @ torch.linalg.pinv(V)
            lam = torch.linalg.vector_norm(Un, dim=0)
            lam = torch.where(lam > 0, lam, torch.ones_like(lam))
            Un = Un / lam
            U[n] = Un.float().contiguous()
            grams[n] = U[n].double().T @ U[n].double()
        # fit from the last mode's MTTKRP (M computed with the updated others)
        inner = float((lam * (M * U[N - 1].double()).sum(dim=0)).sum())
        H = torch.ones((rank, rank), dtype=torch.float64, device=dev)
        for m in range(N):
            H = H * grams[m]
        model2 = float(lam @ H @ lam)
        resid2 = max(normx2 + model2 - 2.0 * inner, 0.0)
        fit = 1.0 - (resid2 ** 0.5) / (normx2 ** 0.5) if normx2 > 0 else 1.0
        fits.append(fit)
        if len(fits) > 1 and abs(fits[-1] - fits[-2]) < tol:
            break
    return CPResult(lam.float(), U, fits, it)


# ---------------------------------------------------------------------------
# Row-sharded CP-ALS across ranks
#
# Every rank owns, for each mode n, a block of rows [lo, hi) of U_n and the
# entries of X whose mode-n index falls in it (the row-aligned shard of the
# mode-n-sorted tensor, parallel.row_aligned_ranges / row_blocks). Its
# MTTKRP over that shard is exact on the owned rows (no partial sums cross
# ranks), so the only data exchanged per mode update is
#   * an all-reduce of R column sums of squares (lambda) -- R doubles;
#   * an all-gather of the updated owned row blocks of U_n, because the other
#     modes' MTTKRPs gather U_n rows at arbitrary indices: (G-1)/G of
#     I_n x R fp32 received per rank, where the all-reduce of MTTKRP partials
#     (section 8(e)) would move twice that;
# and per iteration one all-reduce of the fit's inner product. The Gram
# matrices come from the full factor replicas every rank holds (identical on
# all ranks, no exchange).

class SimRanks:
    """G ranks driven from one process on one device, for tests and
    single-GPU emulation: a collective combines the per-rank list in rank
    order. No rank ever waits on another (they run one after another)."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def all_reduce(self, xs: List[torch.Tensor]) -> List[torch.Tensor]:
        s = xs[0].clone()
        for t in xs[1:]:
            s += t
        return [s for _ in xs]

    def all_gather_rows(self, parts: List[torch.Tensor], blocks) -> List[torch.Tensor]:
        full = torch.cat(parts, 0)
        assert full.shape[0] == blocks[-1][1]
        return [full for _ in parts]


class DistRanks:
    """This process's rank of a torch.distributed group (NCCL on the GPU box,
    gloo in the CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]

    def all_reduce(self, xs: List[torch.Tensor]) -> List[torch.Tensor]:
        self.dist.all_reduce(xs[0], group=self.group)
        return xs

    def all_gather_rows(self, parts: List[torch.Tensor], blocks) -> List[torch.Tensor]:
        p = parts[0]
        B = max(1, max(hi - lo for lo, hi in blocks))
        send = torch.zeros((B, p.shape[1]), dtype=p.dtype, device=p.device)
        send[: p.shape[0]] = p
        recv = torch.empty((self.world * B, p.shape[1]), dtype=p.dtype, device=p.device)
        self.dist.all_gather_into_tensor(recv, send, group=self.group)
        return [torch.cat([recv[r * B: r * B + (hi - lo)] for r, (lo, hi) in enumerate(blocks)])]


def row_shard(xs, mode: int, world: int, rank: int):
    """Rank `rank`'s row-aligned shard of xs (sorted with `mode` leading) and
    the owned row blocks of every rank (parallel.row_aligned_ranges /
    row_blocks)."""
    from . import parallel
    rows = xs.indices[mode]
    rr = parallel.row_aligned_ranges(rows, world)
    blocks = parallel.row_blocks(rows, rr, xs.dims[mode])
    return parallel.slice_coo(xs, *rr[rank]), blocks


def mode_sorted(x: DeviceCOO, mode: int) -> DeviceCOO:
    """A copy of x sorted with `mode` leading, the others ascending."""
    xs = x.clone()
    ops.sort_lexicographic(xs, [mode] + [d for d in range(x.order) if d != mode])
    return xs


def cp_als_rowsharded(shards, blocks, dims, rank: int, ranks, iters: int = 20,
                      tol: float = 1e-5, init: Optional[List[torch.Tensor]] = None,
                      seed: int = 0, mttkrp_fn=None) -> CPResult:
    """CP-ALS over row-sharded factors. shards[n][j] is local rank j's
    (ranks.ranks[j]) row-aligned shard for mode n, blocks[n] the owned row
    blocks of all ranks; every rank starts from the same init. mttkrp_fn(shard,
    factors, n) returns the full dims[n] x R MTTKRP of the shard (zero outside
    its rows); default: the sm_100a kernel. Returns rank ranks.ranks[0]'s view
    (factors identical on every rank)."""
    N = len(dims)
    L = len(ranks.ranks)
    if mttkrp_fn is None:
        mttkrp_fn = lambda s, f, n: ops.mttkrp(s, f, n, ops.MTTKRP_AUTO)  # noqa: E731
    dev = shards[0][0].values.device if isinstance(shards[0][0], DeviceCOO) else \
        torch.device("cpu")
    if init is None:
        init = [generate.uniform((dims[n], rank), seed, 500 + n, 0.0, 1.0, dev.index or 0)
                for n in range(N)]
    U = [[u.to(dev, torch.float32).contiguous().clone() for u in init] for _ in range(L)]
    grams = [[u.double().T @ u.double() for u in U[j]] for j in range(L)]

    def vals(s):
        v = s.values
        return v.double() if isinstance(v, torch.Tensor) else torch.from_numpy(v).double()
    normx2 = float(ranks.all_reduce([(vals(shards[0][j]) ** 2).sum().reshape(1).to(dev)
                                     for j in range(L)])[0][0])
    lam = torch.ones(rank, dtype=torch.float64, device=dev)
    fits: List[float] = []
    it = 0
    M = [None] * L
    for it in range(1, iters + 1):
        for n in range(N):
            own, colsq = [], []
            for j, g in enumerate(ranks.ranks):
                lo, hi = blocks[n][g]
                Mj = mttkrp_fn(shards[n][j], U[j], n)
                Mj = (Mj if isinstance(Mj, torch.Tensor) else torch.from_numpy(Mj))
                M[j] = Mj.to(dev).double()[lo:hi]
                V = torch.ones((rank, rank), dtype=torch.float64, device=dev)
                for m in range(N):
                    if m != n:
                        V = V * grams[j][m]
                Un = M[j] @ torch.linalg.pinv(V)
                own.append(Un)
                colsq.append((Un * Un).sum(dim=0))
            lam = ranks.all_reduce(colsq)[0].sqrt()
            lam = torch.where(lam > 0, lam, torch.ones_like(lam))
            full = ranks.all_gather_rows([(Un / lam).float().contiguous() for Un in own],
                                         blocks[n])
            for j in range(L):
                U[j][n] = full[j].contiguous()
                grams[j][n] = U[j][n].double().T @ U[j][n].double()
        inner = []
        for j, g in enumerate(ranks.ranks):
            lo, hi = blocks[N - 1][g]
            inner.append((lam * (M[j] * U[j][N - 1][lo:hi].double()).sum(dim=0)).sum()
                         .reshape(1))
        inner = float(ranks.all_reduce(inner)[0][0])
        H = torch.ones((rank, rank), dtype=torch.float64, device=dev)
        for m in range(N):
            H = H * grams[0][m]
        model2 = float(lam @ H @ lam)
        resid2 = max(normx2 + model2 - 2.0 * inner, 0.0)
        fit = 1.0 - (resid2 ** 0.5) / (normx2 ** 0.5) if normx2 > 0 else 1.0
        fits.append(fit)
        if len(fits) > 1 and abs(fits[-1] - fits[-2]) < tol:
            break
    return CPResult(lam.float(), U[0], fits, it)
