"""Exact oracles that pin the estimator oracle (O-EXACT, O-DENSE).

O-EXACT — the exact structured MLL L(K''(theta)) at any n, O(sum b^3/3 + n_c^3), from the
structure of Eq. (28)-(29): with R, u refactored at theta itself,
W = R^{-T}E has disjoint-support columns u_i, so W^T W = D_u = diag(u_i^T u_i) and, with
M~ = D_u^{1/2} M D_u^{1/2}, mu = eig(M~):
    log|K''| = 2 sum log diag R + sum log(1 + mu)           (matrix determinant lemma)
    y^T K''^{-1} y = c^T c - xi^T M~ (I + M~)^{-1} xi,  xi_i = u_i^T c_i / sqrt(d_i)  (Woodbury)
and at the baseline, for any probe z, with zeta_i = u_i^T z_i / sqrt(d_i):
    z^T f(A) z = f(1) (||z||^2 - ||zeta||^2) + zeta^T f(I + M~) zeta.
O-DENSE — densify K'' (and the true K = k(X,X) + sigma^2 I) and use dense Cholesky; n <= 4096.
Analytic gradient of the exact structured MLL: dL = 1/2 tr(K''^{-1} dK'') - 1/2 a^T dK'' a,
a = K''^{-1} y, dK'' = blockdiag(dK_i) + E (dK_rep - (v0^T dK_rep v0) I) E^T
(Hellmann-Feynman for lambda_0; RBF: dk/dlambda = k ||dx||^2 / lambda^3, dk/dalpha = k/alpha).
Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import math

import numpy as np

from .kernels import RBF, kernel_matrix, sqdist
from .structured import build_blocks, dense_Kpp, solve_Rt, theta_tuple

LOG2PI = math.log(2.0 * math.pi)
DENSE_MAX_N = 4096


def _eig_structure(blocks):
    d = np.array([float(ui @ ui) for ui in blocks.u])
    sd = np.sqrt(d)
    Mt = sd[:, None] * blocks.M * sd[None, :]
    mu, V = np.linalg.eigh(Mt)
    return d, sd, Mt, mu, V


def exact_structured(X, offsets, reps, y, theta, kind=RBF):
    """(L, quad, logdet) of K''(theta) exactly, refactoring at theta (O-EXACT)."""
    b = build_blocks(X, offsets, reps, theta, kind)
    d, sd, Mt, mu, V = _eig_structure(b)
    logdet = b.logdet_R + float(np.sum(np.log1p(mu)))
    c = solve_Rt(b, y)
    xi = np.array([b.u[i] @ c[b.block(i)] for i in range(b.n_c)]) / sd
    quad = float(c @ c) - float(xi @ (Mt @ np.linalg.solve(np.eye(b.n_c) + Mt, xi)))
    n = len(y)
    return 0.5 * (quad + logdet + n * LOG2PI), quad, logdet


def probe_quadform_baseline(blocks, z, f):
    """z^T f(A) z at the baseline A = I + W M W^T, closed form (O-EXACT)."""
    d, sd, Mt, mu, V = _eig_structure(blocks)
    zeta = np.array([blocks.u[i] @ z[blocks.block(i)] for i in range(blocks.n_c)]) / sd
    w = V.T @ zeta
    return float(f(1.0) * (z @ z - zeta @ zeta) + np.sum(w * w * f(1.0 + mu)))


def spectrum_A_baseline(blocks):
    """Eigenvalues of A at the baseline: 1 (multiplicity n - n_c) and 1 + mu."""
    _, _, _, mu, _ = _eig_structure(blocks)
    return np.concatenate([np.ones(blocks.n - blocks.n_c), 1.0 + mu])


def dense_mll(K, y):
    """L = 1/2 (y^T K^{-1} y + log|K| + n log 2 pi) by dense Cholesky (O-DENSE)."""
    n = K.shape[0]
    if n > DENSE_MAX_N:
        raise ValueError("O-DENSE refuses n > 4096 (SPEC.md:517)")
    Lc = np.linalg.cholesky(K)
    a = np.linalg.solve(Lc, y)
    quad = float(a @ a)
    logdet = 2.0 * float(np.sum(np.log(np.diag(Lc))))
    return 0.5 * (quad + logdet + n * LOG2PI), quad, logdet


def dense_structured_mll(X, offsets, reps, y, theta, kind=RBF):
    b = build_blocks(X, offsets, reps, theta, kind)
    return dense_mll(dense_Kpp(b, theta), y)


def dense_true_K(X, theta, kind=RBF):
    lam, s2, alpha = theta_tuple(theta)
    return kernel_matrix(kind, X, X, lam, alpha) + s2 * np.eye(X.shape[0])


def analytic_grad_structured(X, offsets, reps, y, theta):
    """Exact gradient of the structured MLL (RBF only, jitter-free), dense, n <= 4096."""
    lam, s2, alpha = theta_tuple(theta)
    b = build_blocks(X, offsets, reps, theta, RBF)
    if np.any(b.jitter > 0):
        raise ValueError("analytic gradient assumes no jitter")
    K = dense_Kpp(b, theta)
    if K.shape[0] > DENSE_MAX_N:
        raise ValueError("dense gradient refuses n > 4096")
    Kinv = np.linalg.inv(K)
    a = Kinv @ y
    evals, evecs = np.linalg.eigh(b.Krep)
    v0 = evecs[:, 0]
    sqr = sqdist(b.reps, b.reps)
    Krep = b.Krep
    dKrep = {"lam": Krep * sqr / lam ** 3, "alpha": Krep / alpha}
    n = K.shape[0]
    grads = []
    for name in ("lam", "s2", "alpha"):
        dK = np.zeros((n, n))
        for i in range(b.n_c):
            sl = b.block(i)
            Xi = X[sl]
            ki = kernel_matrix(RBF, Xi, Xi, lam, alpha)
            if name == "lam":
                dK[sl, sl] = ki * sqdist(Xi, Xi) / lam ** 3
            elif name == "alpha":
                dK[sl, sl] = ki / alpha
            else:
                dK[sl, sl] = np.eye(Xi.shape[0])
        if name != "s2":
            dM = dKrep[name] - float(v0 @ dKrep[name] @ v0) * np.eye(b.n_c)
            for i in range(b.n_c):
                for j in range(b.n_c):
                    dK[b.block(i), b.block(j)] += dM[i, j]
        grads.append(0.5 * float(np.sum(Kinv * dK)) - 0.5 * float(a @ dK @ a))
    return np.array(grads)
