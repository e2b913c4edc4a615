"""Kernel functions — PAPER.md:52-56 (§2, Eq. 2).

Eq. (2) prints k(x,x') = alpha*exp(-||x-x'||_2 / (2 lambda^2)) with the distance NOT
squared.  Reading X3/P1: the default `rbf` squares it (the standard RBF
kernel, which the paper's GPyTorch baseline uses); the printed form is `rbf_as_printed`
(an exponential kernel, also PD).  `matern52` is the textbook Matern-5/2 (config C4).

Squared distances are computed directly as sum_d (x_d - x'_d)^2, never through
||x||^2 + ||x'||^2 - 2 x.x', so k(x,x) == alpha exactly and K(X,X) is bitwise symmetric.
Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

RBF, MATERN52, RBF_AS_PRINTED = "rbf", "matern52", "rbf_as_printed"
KERNEL_IDS = {RBF: 0, MATERN52: 1, RBF_AS_PRINTED: 2}


def sqdist(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Pairwise squared Euclidean distances, sum over dimensions of (a_d - b_d)^2."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    out = np.zeros((A.shape[0], B.shape[0]))
    for dd in range(A.shape[1]):                       # fixed dimension order
        diff = A[:, dd][:, None] - B[:, dd][None, :]
        out += diff * diff
    return out


def kernel_matrix(kind: str, A, B, lengthscale: float, outputscale: float) -> np.ndarray:
    """k(A, B; lambda, alpha) without noise (K_rep and off-diagonal use)."""
    sq = sqdist(A, B)
    lam, alpha = float(lengthscale), float(outputscale)
    if kind == RBF:
        return alpha * np.exp(-sq / (2.0 * lam * lam))
    if kind == RBF_AS_PRINTED:                         # Eq. (2) literally
        return alpha * np.exp(-np.sqrt(sq) / (2.0 * lam * lam))
    if kind == MATERN52:
        rho = np.sqrt(sq)
        s = np.sqrt(5.0) * rho / lam
        return alpha * (1.0 + s + 5.0 * sq / (3.0 * lam * lam)) * np.exp(-s)
    raise ValueError(f"unknown kernel {kind!r}")


def kernel_eval(kind: str, x, xp, lengthscale: float, outputscale: float) -> float:
    return float(kernel_matrix(kind, np.atleast_2d(x), np.atleast_2d(xp), lengthscale, outputscale)[0, 0])
