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
