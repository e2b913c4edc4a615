"""Conjugate gradient and batched multi-RHS CG — PAPER.md §3.1 (lines 107-108, 124).

PAPER.md:108 solves K u = y by CG; "we adopt a batch CG algorithm ... to
compute all m solves simultaneously"; "terminate our PCG procedure when the
L2 norm of the residual vector is less than 0.01 ... 2,000 as the maximum number of
iterations".  Readings: P3 the residual is that of the transformed (split)
system A x = b with A = R^{-T} K'' R^{-1}, absolute, per column; P4 x_0 = 0; P5 per-column
alpha_j / beta_j, a column freezes (x, r, p stop updating) once ||r_j|| < tol or
r_j^T r_j == 0; P7 explicit split preconditioning.

Textbook CG (Hestenes-Stiefel) per column j, checked at the top of every iteration:
    stop if sqrt(r^T r) < tol   (or r^T r == 0, or k == max_iter)
    q = A p;  alpha = r^T r / p^T q;  x += alpha p;  r -= alpha q
    beta = r'^T r' / r^T r;  p = r' + beta p
Replay mode runs exactly replay[j] iterations for column j (parity protocol).
Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class CGResult:
    X: np.ndarray
    iters: np.ndarray
    alphas: list = field(default_factory=list)   # per column, list of alpha_k
    betas: list = field(default_factory=list)    # per column, list of beta_k
    resid: np.ndarray = None                     # final ||r_j||
    converged: np.ndarray = None


def cg_batched(apply, B, tol=0.01, max_iter=2000, replay=None) -> CGResult:
    B = np.asarray(B, dtype=np.float64)
    if B.ndim == 1:
        B = B[:, None]
    n, c = B.shape
    X = np.zeros((n, c))
    R = B.copy()
    P = R.copy()
    rr = np.einsum("ij,ij->j", R, R)
    iters = np.zeros(c, dtype=np.int64)
    alphas = [[] for _ in range(c)]
    betas = [[] for _ in range(c)]

    def active_cols():
        if replay is not None:
            return iters < np.asarray(replay, dtype=np.int64)
        return (iters < max_iter) & ~(np.sqrt(rr) < tol) & (rr > 0.0)

    act = active_cols()
    while act.any():
        Q = apply(P)
        for j in np.nonzero(act)[0]:
            pq = float(P[:, j] @ Q[:, j])
            alpha = rr[j] / pq
            X[:, j] += alpha * P[:, j]
            R[:, j] -= alpha * Q[:, j]
            rr_new = float(R[:, j] @ R[:, j])
            beta = rr_new / rr[j]
            P[:, j] = R[:, j] + beta * P[:, j]
            rr[j] = rr_new
            iters[j] += 1
            alphas[j].append(alpha)
            betas[j].append(beta)
        act = active_cols()
    resid = np.sqrt(rr)
    conv = ~(resid >= tol) if replay is None else np.ones(c, dtype=bool)
    return CGResult(X=X, iters=iters, alphas=alphas, betas=betas, resid=resid, converged=conv)
