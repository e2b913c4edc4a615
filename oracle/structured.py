"""Block preconditioner, low-rank off-diagonal term and the preconditioned operator.

Follows PAPER.md §3.2-§3.3 in order:
  * Eq. (12)-(13): R = diag(R_i), R_i^T R_i = (K_diag)_i, per-block
    Cholesky of K_i = k(X_i, X_i; theta_0) + sigma_0^2 I.
  * PAPER.md:221 jitter "add small values to the diagonal terms": ladder
    eps_t = 1e-8 * mean(diag K_i) * 10^t, t = 0..4; the jittered K_i is the
    model's block from then on; after the ladder -> NotSPD(i).
  * Eq. (16): logdet_R = 2 sum_i log|R_i| = 2 sum_i sum_j log (R_i)_jj.
  * Eq. (21): u_i = R_i^{-T} 1.
  * Eq. (22), (26)-(28): K_rep = k(r_i, r_j) (no noise),
    lambda_0 = lambda_min(K_rep) (> 0 else DegenerateReps), M = K_rep - lambda_0 I, so that
    K''_offdiag = E M E^T (block (i,j) = k(r_i,r_j) 11^T, block (i,i) = (k(r_i,r_i)-lambda_0) 11^T).
  * Eq. (18)-(21) split apply of A = R^{-T} K'' R^{-1}:
        A D = F(D) + W M' W^T D,   W = R^{-T} E (block i column = u_i),
    with F from Eq. (23)-(25):
        baseline (theta == theta_0):        F(D) = D                                   Eq. (23)
        noise    (only sigma^2 differs):    F(D) = D + d_sigma2 * R^{-T} R^{-1} D      Eq. (24)
        scale    (only alpha differs):      F(D) = (1+r) D - (sigma_0^2+eps_i) r R^{-T}R^{-1} D   Eq. (25)
        generic  (lengthscale differs):     F(D) = R^{-T} (K_diag(theta) (R^{-1} D))
    and M' = M (baseline, noise), (1+r) M (scale, reading P11), K_rep(theta) - lambda_0(theta) I
    (generic).  R, u, jitter stay those built at theta_0 (reading P11).
Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
from scipy.linalg import solve_triangular
from threadpoolctl import threadpool_limits

from .kernels import kernel_matrix

# Per-cluster loops run over a thread pool (SURVEY §8(d) "parallelising O-ALG's per-cluster loop
# over a thread pool is allowed, and the thread count is stated").  Each cluster's step is the same
# independent NumPy/SciPy call as in a plain loop, with BLAS held to ONE thread inside the pool, so
# the result of every cluster — and therefore of the oracle — does not depend on ORACLE_THREADS.
# (The per-apply triangular solves skip SciPy's input scan, check_finite=False: R is finite by
# construction — a Cholesky factor that passed — and the scan held the GIL for most of an apply.)
ORACLE_THREADS = max(1, int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))
_POOL = None


def cluster_map(fn, n):
    """[fn(i) for i in range(n)], evaluated cluster-parallel (results in cluster order)."""
    global _POOL
    with threadpool_limits(limits=1):
        if n < 32 or ORACLE_THREADS == 1:
            return [fn(i) for i in range(n)]
        if _POOL is None:
            _POOL = ThreadPoolExecutor(ORACLE_THREADS)
        return list(_POOL.map(fn, range(n)))


class NotSPD(Exception):
    def __init__(self, block: int):
        super().__init__(f"block {block} is not SPD after the jitter ladder")
        self.block = block


class DegenerateReps(Exception):
    pass


JITTER_TRIES = 5


def chol_upper_with_jitter(K: np.ndarray, block: int = 0):
    """Upper Cholesky R (R^T R = K) with the PAPER.md:221 / SPEC.md:125 jitter ladder.

    Returns (R, eps) where eps is the jitter that was added (0.0 if none)."""
    try:
        return np.linalg.cholesky(K).T.copy(), 0.0
    except np.linalg.LinAlgError:
        pass
    base = 1e-8 * float(np.mean(np.diag(K)))
    for t in range(JITTER_TRIES):
        eps = base * 10.0 ** t
        try:
            return np.linalg.cholesky(K + eps * np.eye(K.shape[0])).T.copy(), eps
        except np.linalg.LinAlgError:
            continue
    raise NotSPD(block)


def smallest_eig(K: np.ndarray) -> float:
    """lambda_min of a symmetric matrix (LAPACK eigvalsh) — Eq. (26)."""
    return float(np.linalg.eigvalsh(K)[0])


def theta_tuple(theta):
    lam, s2, alpha = (float(t) for t in theta)
    if not (lam > 0 and s2 > 0 and alpha > 0):
        raise ValueError("theta must be positive")
    return lam, s2, alpha


def krep_and_M(kind, reps, theta):
    """K_rep(theta), lambda_0(theta), M = K_rep - lambda_0 I  (Eq. 26-28)."""
    lam, _, alpha = theta_tuple(theta)
    Krep = kernel_matrix(kind, reps, reps, lam, alpha)
    lam0 = smallest_eig(Krep)
    if not lam0 > 0.0:
        raise DegenerateReps(f"lambda_0 = {lam0!r} <= 0")
    return Krep, lam0, Krep - lam0 * np.eye(Krep.shape[0])


@dataclass
class Blocks:
    """The per-epoch preconditioner state built at theta_0 (Alg. 1)."""

    X: np.ndarray
    offsets: np.ndarray
    reps: np.ndarray
    kind: str
    theta0: tuple
    R: list
    jitter: np.ndarray
    logdet_R: float
    u: list
    Krep: np.ndarray
    lam0: float
    M: np.ndarray

    @property
    def n_c(self):
        return len(self.R)

    @property
    def n(self):
        return int(self.offsets[-1])

    def block(self, i):
        return slice(int(self.offsets[i]), int(self.offsets[i + 1]))

    def K_block(self, i, theta):
        """K_i(theta) = k(X_i, X_i; theta) + (sigma^2 + eps_i) I  (the model's block)."""
        lam, s2, alpha = theta_tuple(theta)
        Xi = self.X[self.block(i)]
        return kernel_matrix(self.kind, Xi, Xi, lam, alpha) + (s2 + self.jitter[i]) * np.eye(Xi.shape[0])


def build_blocks(X, offsets, reps, theta0, kind="rbf") -> Blocks:
    """Alg. 1: block-diagonal Cholesky at theta_0, plus u_i, logdet_R, K_rep, M."""
    X = np.asarray(X, dtype=np.float64)
    offsets = np.asarray(offsets, dtype=np.int64)
    lam, s2, alpha = theta_tuple(theta0)
    n_c = offsets.shape[0] - 1
    if offsets[0] != 0 or offsets[-1] != X.shape[0] or np.any(np.diff(offsets) <= 0):
        raise ValueError("offsets must be strictly increasing from 0 to n")
    def one(i):
        Xi = X[offsets[i]:offsets[i + 1]]
        Ki = kernel_matrix(kind, Xi, Xi, lam, alpha) + s2 * np.eye(Xi.shape[0])
        Ri, eps = chol_upper_with_jitter(Ki, i)
        return Ri, eps, solve_triangular(Ri, np.ones(Xi.shape[0]), trans="T")   # Eq. (21)

    R, jit, u = [], np.zeros(n_c), []
    logdet_R = 0.0
    for i, (Ri, eps, ui) in enumerate(cluster_map(one, n_c)):
        R.append(Ri)
        jit[i] = eps
        logdet_R += 2.0 * float(np.sum(np.log(np.diag(Ri))))          # Eq. (16)
        u.append(ui)
    Krep, lam0, M = krep_and_M(kind, reps, theta0)
    return Blocks(X=X, offsets=offsets, reps=np.asarray(reps, dtype=np.float64), kind=kind,
                  theta0=(lam, s2, alpha), R=R, jitter=jit, logdet_R=logdet_R, u=u,
                  Krep=Krep, lam0=lam0, M=M)


def solve_Rt(blocks: Blocks, y):
    """c = R^{-T} y, block by block (transformed right-hand side)."""
    y = np.asarray(y, dtype=np.float64)
    out = np.empty_like(y)
    parts = cluster_map(lambda i: solve_triangular(blocks.R[i], y[blocks.block(i)], trans="T"), blocks.n_c)
    for i in range(blocks.n_c):
        out[blocks.block(i)] = parts[i]
    return out


def mode_of(theta0, theta):
    lam0, s20, a0 = theta0
    lam, s2, a = theta
    if lam == lam0 and s2 == s20 and a == a0:
        return "baseline"
    if lam == lam0 and a == a0:
        return "noise"
    if lam == lam0 and s2 == s20:
        return "scale"
    return "generic"


class Operator:
    """A = R^{-T} K''(theta) R^{-1} applied matrix-free (Eq. 18-21, 23-25)."""

    def __init__(self, blocks: Blocks, theta):
        self.b = blocks
        self.theta = theta_tuple(theta)
        self.mode = mode_of(blocks.theta0, self.theta)
        lam, s2, alpha = self.theta
        _, s20, a0 = blocks.theta0
        if self.mode in ("baseline", "noise"):
            self.Mp, self.lam0 = blocks.M, blocks.lam0
        elif self.mode == "scale":
            r = (alpha - a0) / a0
            self.r = r
            self.Mp, self.lam0 = (1.0 + r) * blocks.M, (1.0 + r) * blocks.lam0
        else:
            _, self.lam0, self.Mp = krep_and_M(blocks.kind, blocks.reps, self.theta)
            self.Kd = cluster_map(lambda i: blocks.K_block(i, self.theta), blocks.n_c)

    def _H(self, i, Di):
        """H_i D_i = R_i^{-T} (R_i^{-1} D_i)  (NOT K_i^{-1})."""
        Ri = self.b.R[i]
        return solve_triangular(Ri, solve_triangular(Ri, Di, check_finite=False), trans="T", check_finite=False)

    def F(self, i, Di):
        lam, s2, alpha = self.theta
        _, s20, a0 = self.b.theta0
        if self.mode == "baseline":                                  # Eq. (23)
            return Di.copy()
        if self.mode == "noise":                                     # Eq. (24)
            return Di + (s2 - s20) * self._H(i, Di)
        if self.mode == "scale":                                     # Eq. (25)
            r = self.r
            return (1.0 + r) * Di - (s20 + self.b.jitter[i]) * r * self._H(i, Di)
        Ri = self.b.R[i]                                             # generic, Eq. (18)-(19)
        return solve_triangular(Ri, self.Kd[i] @ solve_triangular(Ri, Di, check_finite=False), trans="T",
                                check_finite=False)

    def apply(self, D):
        D = np.asarray(D, dtype=np.float64)
        vec = D.ndim == 1
        if vec:
            D = D[:, None]
        nb = self.b.n_c
        S = np.empty((nb, D.shape[1]))
        for j in range(nb):                                          # S_j = u_j^T D_j
            S[j] = self.b.u[j] @ D[self.b.block(j)]
        T = self.Mp @ S                                              # T = M' S
        out = np.empty_like(D)
        Fs = cluster_map(lambda i: self.F(i, D[self.b.block(i)]), nb)
        for i in range(nb):                                          # out_i = F_i + u_i T_i
            out[self.b.block(i)] = Fs[i] + np.outer(self.b.u[i], T[i])
        return out[:, 0] if vec else out

    def apply_Q(self, D):
        """Q(A) D = A(A D) + 4 A D + D (Eq. 10 denominator)."""
        V = self.apply(D)
        return self.apply(V) + 4.0 * V + D


def dense_Kpp(blocks: Blocks, theta) -> np.ndarray:
    """Dense K''(theta) = blockdiag(K_i(theta)) + E M(theta) E^T, assembled entry-block by
    entry-block from Eq. (17), (27), (28) (only for small n)."""
    n = blocks.n
    K = np.zeros((n, n))
    _, lam0, M = krep_and_M(blocks.kind, blocks.reps, theta)
    for i in range(blocks.n_c):
        for j in range(blocks.n_c):
            K[blocks.block(i), blocks.block(j)] = M[i, j]
        K[blocks.block(i), blocks.block(i)] += blocks.K_block(i, theta)
    return K


def dense_R(blocks: Blocks) -> np.ndarray:
    n = blocks.n
    R = np.zeros((n, n))
    for i in range(blocks.n_c):
        R[blocks.block(i), blocks.block(i)] = blocks.R[i]
    return R
