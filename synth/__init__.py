"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no kernel, no Cholesky, no CG, no
log-det): it only draws the inputs the paper's experiments are built from, so that
the oracle (`oracle/`) and the CUDA path (`paper_2510_12128_b200/`) consume
bit-identical X, y, offsets, representatives and Hutchinson probes.

Recipes:

* G-HYPER — PAPER.md:348 (§5.1 "Synthetic Datasets", hypercube vertices of side l,
  cluster radius < l/2) with the label function of Eq. (31)
  generalised to d dimensions: y = ||x||^2/100 + N(0, 0.16).  Representatives are the
  vertices (GIVEN mode).  Used for configs C1, C2, C3, C5.
* G-REAL — a Kin40k/Gas-shaped regression set (Table `dataset`
  PAPER.md:377-394): a 20-component Gaussian mixture with uneven weights.  Used for C4.
* probes — the m Hutchinson vectors z_i in {+1,-1}^n of Eq. (9),
  "pre-generated".  A counter-based splitmix64 stream keyed by
  (seed, column j, sorted position p); the CUDA path implements the same counter
  generator independently (csrc/eval.cu `probe_gen_kernel`), and tests check the two
  bit for bit.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = ["CONFIGS", "Dataset", "g_hyper", "g_real", "probes", "make_config"]

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def probes(seed: int, m: int, n: int) -> np.ndarray:
    """Rademacher probes Z (m x n, float64 +-1), splitmix64 counter stream.

    z[j, p] = +1 if bit 63 of splitmix64_{seed}(ctr) is 0 else -1, with
    ctr = (j << 40) | p and splitmix64_{s}(c) the (c+1)-th output of splitmix64 seeded
    with s:  x = s + (c+1)*0x9E3779B97F4A7C15; x = (x ^ x>>30)*0xBF58476D1CE4E5B9;
    x = (x ^ x>>27)*0x94D049BB133111EB; x ^= x>>31.
    """
    if n >= (1 << 40) or m >= (1 << 23):
        raise ValueError("probe counter overflow")
    with np.errstate(over="ignore"):
        j = np.arange(m, dtype=np.uint64)[:, None]
        p = np.arange(n, dtype=np.uint64)[None, :]
        ctr = (j << np.uint64(40)) | p
        x = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (ctr + np.uint64(1)) * _GOLDEN
        x = (x ^ (x >> np.uint64(30))) * _MIX1
        x = (x ^ (x >> np.uint64(27))) * _MIX2
        x = x ^ (x >> np.uint64(31))
    return np.where((x >> np.uint64(63)) == 0, 1.0, -1.0)


@dataclass
class Dataset:
    """Cluster-sorted training data (rows of cluster i are offsets[i]:offsets[i+1])."""

    X: np.ndarray            # n x d float64, cluster-contiguous
    y: np.ndarray            # n float64
    offsets: np.ndarray      # n_c+1 int64
    reps: np.ndarray         # n_c x d float64 (GIVEN representatives)
    theta0: tuple            # (lengthscale, noise, outputscale)
    X_test: np.ndarray | None = None
    y_test: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.X.shape[0])

    @property
    def n_c(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def d(self) -> int:
        return int(self.X.shape[1])


def _grid_side(n_c: int, d: int) -> int:
    g = 2
    while g ** d < n_c:
        g += 1
    return g


def g_hyper(n_c: int, b: int, d: int, seed: int, b_test: int = 0) -> Dataset:
    """G-HYPER: n_c clusters of b points around distinct vertices of a grid on [-10,10]^d.

    Grid: g = max(2, ceil(n_c^(1/d))) points per axis, spacing l = 20/(g-1)
    ("divide the d-dimensional space into hypercubes with a fixed side
    length l ... r_i a vertex").  Each cluster: b points uniform in a d-ball of radius
    rho = 0.25*l < l/2, so clusters never overlap.  Labels per Eq. (31)
    generalised: y = sum(x^2)/100 + eps, eps ~ N(0, 0.16) (variance 0.16).
    theta0 = (0.5*l, 0.16, 1.0).
    """
    rng = np.random.default_rng(seed)
    g = _grid_side(n_c, d)
    l = 20.0 / (g - 1)
    rho = 0.25 * l
    flat = rng.choice(g ** d, size=n_c, replace=False)
    digits = np.stack(np.unravel_index(flat, (g,) * d), axis=1)
    verts = -10.0 + l * digits.astype(np.float64)
    order = np.lexsort(verts.T[::-1])
    verts = verts[order]

    def draw(count):
        dirs = rng.standard_normal((n_c, count, d))
        dirs /= np.linalg.norm(dirs, axis=2, keepdims=True)
        rad = rho * rng.random((n_c, count)) ** (1.0 / d)
        return verts[:, None, :] + dirs * rad[:, :, None]

    X = draw(b).reshape(n_c * b, d)
    y = (X ** 2).sum(axis=1) / 100.0 + rng.normal(0.0, 0.4, size=n_c * b)
    X_test = y_test = None
    if b_test > 0:
        X_test = draw(b_test).reshape(n_c * b_test, d)
        y_test = (X_test ** 2).sum(axis=1) / 100.0 + rng.normal(0.0, 0.4, size=n_c * b_test)
    offsets = np.arange(n_c + 1, dtype=np.int64) * b
    return Dataset(X=np.ascontiguousarray(X), y=y, offsets=offsets, reps=verts,
                   theta0=(0.5 * l, 0.16, 1.0), X_test=X_test, y_test=y_test,
                   meta=dict(kind="g_hyper", g=g, l=l, rho=rho, seed=seed))


def g_real(N: int = 40000, d: int = 8, n_comp: int = 20, seed: int = 104):
    """G-REAL: Kin40k/Gas-shaped regression inputs with uneven clusters (config C4).

    A n_comp-component Gaussian mixture: means are distinct vertices of the g=2 grid on
    [-10,10]^d, covariances Q diag(s^2) Q^T with Q from the QR of a Gaussian matrix and
    s ~ U[1,4], weights ~ Dirichlet(2*1).  y = sum_k sin(x_k/2) + ||x||^2/200 + N(0,0.16).
    80/20 train/test split.  Returns UNSORTED train/test arrays; the
    clustering (k-means) is step A0 of the method and is not done here.
    """
    rng = np.random.default_rng(seed)
    flat = rng.choice(2 ** d, size=n_comp, replace=False)
    digits = np.stack(np.unravel_index(flat, (2,) * d), axis=1)
    means = -10.0 + 20.0 * digits.astype(np.float64)
    w = rng.dirichlet(2.0 * np.ones(n_comp))
    comp = rng.choice(n_comp, size=N, p=w)
    X = np.empty((N, d))
    for k in range(n_comp):
        Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
        s = rng.uniform(1.0, 4.0, size=d)
        idx = np.nonzero(comp == k)[0]
        X[idx] = means[k] + (rng.standard_normal((idx.size, d)) * s) @ Q.T
    y = np.sin(X / 2.0).sum(axis=1) + (X ** 2).sum(axis=1) / 200.0 + rng.normal(0.0, 0.4, size=N)
    perm = rng.permutation(N)
    n_train = int(round(0.8 * N))
    tr, te = perm[:n_train], perm[n_train:]
    return dict(X=X[tr].copy(), y=y[tr].copy(), X_test=X[te].copy(), y_test=y[te].copy(),
                n_comp=n_comp, means=means, seed=seed)


# BASELINE.json "configs"; seeds: data = 100+k, probes = 200+k.
CONFIGS = {
    "C1": dict(kind="g_hyper", n_c=10, b=100, d=2, data_seed=101, probe_seed=201,
               kernel="rbf", m=8),
    "C2": dict(kind="g_hyper", n_c=100, b=200, d=8, data_seed=102, probe_seed=202,
               kernel="rbf", m=8),
    "C3": dict(kind="g_hyper", n_c=500, b=200, d=8, data_seed=103, probe_seed=203,
               kernel="rbf", m=8),
    "C4": dict(kind="g_real", N=40000, d=8, n_c=20, data_seed=104, probe_seed=204,
               kernel="matern52", m=8),
    "C5": dict(kind="g_hyper", n_c=2000, b=500, d=4, data_seed=105, probe_seed=205,
               kernel="rbf", m=8),
}


def make_config(name: str, b_test: int = 0, **override) -> Dataset:
    """Build the G-HYPER dataset of config C1/C2/C3/C5 (optionally resized)."""
    cfg = dict(CONFIGS[name])
    cfg.update(override)
    if cfg["kind"] != "g_hyper":
        raise ValueError(f"{name} is not a G-HYPER config")
    ds = g_hyper(cfg["n_c"], cfg["b"], cfg["d"], cfg["data_seed"], b_test=b_test)
    ds.meta.update(config=name, probe_seed=cfg["probe_seed"], m=cfg["m"], kernel=cfg["kernel"])
    return ds
