"""NEXT-1 — the GP posterior with the nuGPR covariance (Eq. (4)-(5); RMSE and
confidence band Eq. (6)-(7)).

    mean = K*^T K''^{-1} y,      var = diag(K** - K*^T K''^{-1} K*)   (+ sigma^2 if requested)

K* = k(X_train, X_test) is the exact kernel (generated on the fly), K** = k(x*, x*) = alpha for the
stationary kernels, and K''^{-1} is applied EXACTLY through the structure of Eq. (28) (reading
P22): with the blocks R, u built at the trained theta, W = R^{-T}E has
disjoint-support columns u_i, d_i = u_i^T u_i, M~ = D^{1/2} M D^{1/2}, C = I + M~ = L_C L_C^T,
    K''^{-1} = K_d^{-1} - K_d^{-1} E M (I + D M)^{-1} E^T K_d^{-1}                (Woodbury)
so that, with c = R^{-T} y, w_j = R^{-T} k*_j (per block), zeta_i = u_i^T c_i / sqrt(d_i) and
p_ij = u_i^T w_ij / sqrt(d_i), and because M~ C^{-1} = I - C^{-1}:
    mean_j = w_j^T c - (p_j^T zeta - (L_C^{-1} p_j)^T (L_C^{-1} zeta))
    var_j  = alpha - (||w_j||^2 - (||p_j||^2 - ||L_C^{-1} p_j||^2)).
RMSE is the standard sqrt(mean((mu - y)^2)) (reading P21); the band is mu +- 2 sqrt(var)
(Eq. (7)).  `dense_posterior` is the plain dense definition (n <= 4096) that pins it.
Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular

from .kernels import kernel_matrix
from .structured import Blocks, dense_Kpp, solve_Rt, theta_tuple


def posterior(blocks: Blocks, y, X_test, add_noise: bool = False):
    """(mean, var) of the structured posterior at the blocks' theta_0 (exact, no CG)."""
    lam, s2, alpha = theta_tuple(blocks.theta0)
    X_test = np.atleast_2d(np.asarray(X_test, dtype=np.float64))
    y = np.asarray(y, dtype=np.float64)
    n_c = blocks.n_c
    d = np.array([float(ui @ ui) for ui in blocks.u])
    sd = np.sqrt(d)
    Mt = sd[:, None] * blocks.M * sd[None, :]
    LC = np.linalg.cholesky(np.eye(n_c) + Mt)
    c = solve_Rt(blocks, y)
    zeta = np.array([blocks.u[i] @ c[blocks.block(i)] for i in range(n_c)]) / sd
    nt = X_test.shape[0]
    wc = np.zeros(nt)
    ww = np.zeros(nt)
    p = np.zeros((n_c, nt))
    for i in range(n_c):
        sl = blocks.block(i)
        Ks = kernel_matrix(blocks.kind, blocks.X[sl], X_test, lam, alpha)          # b_i x nt
        W = solve_triangular(blocks.R[i].T, Ks, lower=True)                          # R_i^{-T} K*_i
        wc += W.T @ c[sl]
        ww += np.sum(W * W, axis=0)
        p[i] = (blocks.u[i] @ W) / sd[i]
    lp = solve_triangular(LC, p, lower=True)
    lz = solve_triangular(LC, zeta, lower=True)
    mean = wc - (p.T @ zeta - lp.T @ lz)
    var = alpha - (ww - (np.sum(p * p, axis=0) - np.sum(lp * lp, axis=0)))
    if add_noise:
        var = var + s2
    return mean, var


def dense_posterior(blocks: Blocks, y, X_test, add_noise: bool = False, K=None):
    """Eq. (4)-(5) by dense linear algebra on K'' (or on a given dense K)."""
    lam, s2, alpha = theta_tuple(blocks.theta0)
    if K is None:
        K = dense_Kpp(blocks, blocks.theta0)
    Ks = kernel_matrix(blocks.kind, blocks.X, np.atleast_2d(X_test), lam, alpha)
    Lk = np.linalg.cholesky(K)
    a = np.linalg.solve(Lk.T, np.linalg.solve(Lk, y))
    V = np.linalg.solve(Lk, Ks)
    mean = Ks.T @ a
    var = alpha - np.sum(V * V, axis=0)
    if add_noise:
        var = var + s2
    return mean, var


def rmse(mean, y_test) -> float:
    """Standard RMSE (reading P21; Eq. (6) prints sqrt(||mu - y||_2))."""
    r = np.asarray(mean) - np.asarray(y_test)
    return float(np.sqrt(np.mean(r * r)))


def confidence_band(mean, var):
    """Eq. (7): mu +- 2 s."""
    s = np.sqrt(np.maximum(var, 0.0))
    return mean - 2.0 * s, mean + 2.0 * s
