"""Row A0 — clustering the training inputs ("k-means to find n_c clusters; the
cluster centres become the representatives"; PAPER.md:43 inputs "partitioned into n_c
clusters"; Eq. (32) PAPER.md:367-371 medoid representatives).

The paper does not specify its k-means.  Reading P18 fixes every detail so the
assignment is a deterministic function of the inputs (bit-exact between implementations):

  * init: Forgy — the centres are rows x_{i_j} of X, j = 0..n_c-1, with the indices drawn by
    `forgy_indices(seed, n, n_c)` (a splitmix64 counter stream with rejection of repeats), or
    caller-given centres.
  * assignment step: a(p) = argmin_j sum_d (x_pd - c_jd)^2 with the squared distance summed in
    dimension order d = 0..d-1, each term rounded separately (no fused multiply-add), ties to
    the lowest j.
  * update step: c_j = (sum_{a(p)=j} x_p) / |{p: a(p)=j}| with the sum taken EXACTLY in int64
    fixed point: q_pd = rint(x_pd * 2^s) (round half to even), s = 62 - ceil(log2(max|x| * n)),
    so |sum q| < 2^62 cannot overflow and the sum does not depend on the order of the points;
    then c_jd = (double(S_jd) * 2^-s) / count_j (two IEEE roundings).  An empty cluster keeps
    its centre.
  * Lloyd: assign; then repeat {update; assign} until no assignment changes or max_iter
    updates were made.  `iters` = number of update steps.
  * output: a stable permutation by (cluster, original index) -> perm (perm[k] = original row
    of sorted row k), offsets[n_c+1], and the representatives:
      GIVEN    = the initial centres (the synthetic configs pass the grid vertices),
      CENTROID = the final centres,
      MEDOID   = argmax_{x in cluster} sum_{x' in cluster} k(x, x') (Eq. (32) prints argmin;
                 reading P17 takes argmax, the "most central" point), lowest original index
                 on ties.

Test infrastructure only (see oracle/__init__.py).  The splitmix64 index stream is written
out here independently of the CUDA path's host code (same published generator, no shared
code).
"""
from __future__ import annotations

import math

import numpy as np

from .kernels import kernel_matrix

GIVEN, CENTROID, MEDOID = 0, 1, 2
_M64 = (1 << 64) - 1


def _splitmix64(seed: int, ctr: int) -> int:
    """(ctr+1)-th output of splitmix64 seeded with `seed` (pure-Python 64-bit arithmetic)."""
    x = (seed + (ctr + 1) * 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def forgy_indices(seed: int, n: int, n_c: int) -> list[int]:
    """n_c distinct row indices: candidate t of centre j is splitmix64(seed, (j<<32)|t) mod n,
    the first candidate not already taken wins (t = 0, 1, ...)."""
    if n_c > n:
        raise ValueError("n_c > n")
    taken, out = set(), []
    for j in range(n_c):
        t = 0
        while True:
            i = _splitmix64(seed, (j << 32) | t) % n
            if i not in taken:
                break
            t += 1
        taken.add(i)
        out.append(i)
    return out


def fixed_point_shift(X: np.ndarray) -> int:
    """s = 62 - ceil(log2(max|x| * n)) (reading P18); 0 <= s <= 1000 guards degenerate data."""
    n = X.shape[0]
    amax = float(np.max(np.abs(X))) if X.size else 0.0
    if amax == 0.0:
        return 62
    return int(62 - math.ceil(math.log2(amax * n)))


def assign(X: np.ndarray, C: np.ndarray) -> np.ndarray:
    """a(p) = argmin_j sum_d (x_pd - c_jd)^2, dimension order fixed, no FMA, lowest j on ties."""
    n, d = X.shape
    best = np.full(n, np.inf)
    arg = np.zeros(n, dtype=np.int64)
    for j in range(C.shape[0]):
        dist = np.zeros(n)
        for dd in range(d):
            diff = X[:, dd] - C[j, dd]
            dist = dist + diff * diff          # separate multiply and add roundings
        better = dist < best                   # strict: ties keep the lower j
        best = np.where(better, dist, best)
        arg = np.where(better, j, arg)
    return arg


def update(X: np.ndarray, a: np.ndarray, C: np.ndarray, s: int) -> np.ndarray:
    """Centroids from exact int64 fixed-point sums (order independent)."""
    n_c, d = C.shape
    q = np.rint(X * (2.0 ** s)).astype(np.int64)
    Cn = C.copy()
    for j in range(n_c):
        idx = np.nonzero(a == j)[0]
        if idx.size == 0:
            continue                           # empty cluster keeps its centre
        S = q[idx].sum(axis=0, dtype=np.int64) # exact integer sum
        Cn[j] = (S.astype(np.float64) * (2.0 ** -s)) / float(idx.size)
    return Cn


def medoids(X: np.ndarray, a: np.ndarray, n_c: int, kind: str, lengthscale: float,
            outputscale: float) -> np.ndarray:
    """Row index (original order) of argmax_x sum_{x' in cluster} k(x, x'), lowest index on ties."""
    out = np.zeros(n_c, dtype=np.int64)
    for j in range(n_c):
        idx = np.nonzero(a == j)[0]
        K = kernel_matrix(kind, X[idx], X[idx], lengthscale, outputscale)
        score = np.zeros(idx.size)
        for col in range(idx.size):            # sequential sum in member order
            score = score + K[:, col]
        out[j] = idx[int(np.argmax(score))]    # np.argmax returns the first maximum
    return out


def medoid_scores(X, a, n_c, kind, lengthscale, outputscale):
    """All members' scores per cluster (for validity checks of a medoid choice)."""
    res = []
    for j in range(n_c):
        idx = np.nonzero(a == j)[0]
        K = kernel_matrix(kind, X[idx], X[idx], lengthscale, outputscale)
        res.append((idx, K.sum(axis=1)))
    return res


def kmeans(X, n_c: int, init_centers=None, seed: int = 0, max_iter: int = 100,
           rep_mode: int = CENTROID, kind: str = "rbf", theta=(1.0, 0.1, 1.0)):
    """Lloyd k-means + stable cluster sort (row A0).  Returns dict(perm, offsets, reps,
    assign, centers, iters)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, d = X.shape
    if init_centers is None:
        C0 = X[forgy_indices(seed, n, n_c)].copy()
    else:
        C0 = np.array(init_centers, dtype=np.float64).reshape(n_c, d)
    s = fixed_point_shift(X)
    C = C0.copy()
    a = assign(X, C)
    iters = 0
    while iters < max_iter:
        C = update(X, a, C, s)
        iters += 1
        a_new = assign(X, C)
        changed = bool(np.any(a_new != a))
        a = a_new
        if not changed:
            break
    perm = np.argsort(a, kind="stable").astype(np.int64)   # by (cluster, original index)
    counts = np.bincount(a, minlength=n_c)
    offsets = np.zeros(n_c + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(counts)
    if rep_mode == GIVEN:
        reps = C0.copy()
    elif rep_mode == CENTROID:
        reps = C.copy()
    elif rep_mode == MEDOID:
        reps = X[medoids(X, a, n_c, kind, theta[0], theta[2])].copy()
    else:
        raise ValueError("bad rep_mode")
    return dict(perm=perm, offsets=offsets, reps=reps, assign=a, centers=C, iters=iters, shift=s)
