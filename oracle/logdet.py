"""Log-determinant estimators — PAPER.md §3.1-§3.2.

Pade/Hutchinson (the paper's estimator):
  Eq. (8)  log|K| = tr log K
  Eq. (9)  tr log K ~ (1/m) sum_i z_i^T log(K) z_i, z_i in {+-1}^n
  Eq. (10) log K ~ P(K) Q(K)^{-1} = (3K^2 - 3I)(K^2 + 4K + I)^{-1}
  PAPER.md:124 "use CG to first solve for Q^{-1} z_i, multiply the result with P, and
           finally compute the dot product against z_i" -> literal t_j = z_j^T(3A(Aw_j) - 3w_j)
           (reading P2)
  Eq. (16) log|K''| = 2 sum log|R_i| + (1/m) sum z^T log(R^{-T}K''R^{-1}) z

SLQ (north_star "Lanczos/SLQ estimate taken from the CG coefficients", reading X1): the CG
run on Q(A) with x_0 = 0 is Lanczos on Q(A) started at z/||z||; its tridiagonal is
  T_11 = 1/alpha_0,  T_kk = 1/alpha_{k-1} + beta_{k-2}/alpha_{k-2},  T_{k,k+1} = sqrt(beta_{k-1})/alpha_{k-1}
(Saad, Iterative Methods §6.7.3).  With Ritz pairs (theta_l, first components tau_l),
z^T f(Q(A)) z ~ ||z||^2 sum_l tau_l^2 f(theta_l); choosing f(mu) = log(-2 + sqrt(3 + mu))
(the inverse of mu = lambda^2 + 4 lambda + 1 on lambda > 0) estimates z^T log(A) z.
Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import eigh_tridiagonal


def pade_r(x):
    """Scalar 2-2 Pade of log at 1: r(x) = 3(x^2 - 1)/(x^2 + 4x + 1)."""
    x = np.asarray(x, dtype=np.float64)
    return 3.0 * (x * x - 1.0) / (x * x + 4.0 * x + 1.0)


def pade_trace_terms(apply, Z, W):
    """t_j = z_j^T (3 A(A w_j) - 3 w_j) for each probe column (Z, W are n x m)."""
    V = apply(W)
    U = apply(V)
    return np.einsum("ij,ij->j", Z, 3.0 * U - 3.0 * W)


def lanczos_tridiag_from_cg(alphas, betas):
    """(diag, offdiag) of the Lanczos tridiagonal implied by CG coefficients."""
    k = len(alphas)
    a = np.asarray(alphas, dtype=np.float64)
    b = np.asarray(betas, dtype=np.float64)
    diag = np.empty(k)
    diag[0] = 1.0 / a[0]
    for t in range(1, k):
        diag[t] = 1.0 / a[t] + b[t - 1] / a[t - 1]
    off = np.array([np.sqrt(b[t]) / a[t] for t in range(k - 1)])
    return diag, off


def slq_term(alphas, betas, znorm2, f=None):
    """||z||^2 sum_l tau_l^2 f(theta_l); default f maps Q(A)'s spectrum to log(A)."""
    if len(alphas) == 0:
        return 0.0
    if f is None:
        f = lambda mu: np.log(-2.0 + np.sqrt(3.0 + mu))
    diag, off = lanczos_tridiag_from_cg(alphas, betas)
    if len(diag) == 1:
        theta, tau = diag, np.ones(1)
    else:
        theta, V = eigh_tridiagonal(diag, off)
        tau = V[0, :]
    return float(znorm2 * np.sum(tau * tau * f(theta)))
