"""GPU parity of the big-block path (clusters > 512 points: blocked multi-launch factorisation
and the row-tiled apply), against the FP64 oracle: uneven hand-made clusters, and config C4
(G-REAL, 32,000 training points, k-means n_c = 20 uneven clusters up to ~4.3k, Matern-5/2)."""
import numpy as np
import pytest

import synth
from oracle import kmeans as KM
from oracle import structured as OS
from oracle.mll import mll as oracle_mll

pytestmark = pytest.mark.gpu

TIGHT = 1e-9


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2510_12128_b200 as P
    P._native.lib()
    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def uneven(sizes, d, seed, spread=1.0):
    rng = np.random.default_rng(seed)
    n_c = len(sizes)
    reps = rng.uniform(-10, 10, size=(n_c, d))
    X = np.concatenate([reps[i] + spread * rng.standard_normal((s, d)) for i, s in enumerate(sizes)])
    y = np.sin(X).sum(axis=1) + 0.4 * rng.standard_normal(X.shape[0])
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return X, y, off, reps


def check_eval(P, ctx, bg, bo, y, theta, seed, rtol=TIGHT):
    rec = P.mll(ctx, bg, y, theta, probe_seed=seed)
    Z = synth.probes(seed, 8, y.shape[0])
    ro = oracle_mll(bo, y, theta, Z, replay=[rec["iters_y"]] + rec["iters_q"])
    assert rec["mode"] == ro.mode
    for k in ("L", "quad", "logdet_pade", "logdet_slq"):
        assert rel(rec[k], getattr(ro, k)) < rtol, (k, rec[k], getattr(ro, k))
    return rec


def test_big_blocks_uneven_parity(P, ctx):
    sizes = [700, 300, 1100, 530, 90]
    X, y, off, reps = uneven(sizes, 4, 3)
    th0 = (1.3, 0.2, 1.1)
    bg = P.build_blocks(ctx, X, off, reps, th0)
    bo = OS.build_blocks(X, off, reps, th0)
    # factor data: Linv = R^{-T}, u, logdet_R
    Linv = bg.export("linv")
    for i in range(len(sizes)):
        Lo = np.linalg.inv(bo.R[i].T)
        np.testing.assert_allclose(Linv[i], Lo, rtol=0, atol=1e-10 * np.abs(Lo).max())
    np.testing.assert_allclose(bg.export("u"), np.concatenate(bo.u), rtol=1e-10, atol=1e-12)
    assert rel(bg.export("scalars")[0], bo.logdet_R) < 1e-12
    l, s, a = th0
    for th in [th0, (l, s * 1.001, a), (l, s, a * 0.999), (l * 1.001, s, a)]:
        check_eval(P, ctx, bg, bo, y, th, 7)


def test_big_blocks_mixed_with_small_and_jitter(P, ctx):
    """A singular large cluster (duplicated points, tiny noise) takes the jitter ladder on the
    big path exactly as the oracle does."""
    rng = np.random.default_rng(4)
    X1 = np.repeat(rng.standard_normal((300, 2)), 2, axis=0)          # 600 points, duplicates
    X2 = 6 + rng.standard_normal((40, 2))
    X = np.concatenate([X1, X2])
    y = rng.standard_normal(X.shape[0])
    off = np.array([0, 600, 640], dtype=np.int64)
    reps = np.array([[0.0, 0.0], [6.0, 6.0]])
    th0 = (1.0, 1e-18, 1.0)
    bg = P.build_blocks(ctx, X, off, reps, th0)
    bo = OS.build_blocks(X, off, reps, th0)
    np.testing.assert_allclose(bg.export("jitter"), bo.jitter, rtol=1e-12)
    assert bo.jitter[0] > 0


def c4_dataset():
    g = synth.g_real(N=40000, d=8, seed=104)
    km = KM.kmeans(g["X"], 20, seed=104, rep_mode=KM.CENTROID)
    X = g["X"][km["perm"]]
    y = g["y"][km["perm"]]
    off = km["offsets"]
    # theta0 = (median intra-cluster distance, 0.16, Var(y)) (SURVEY §8(d) G-REAL recipe)
    rng = np.random.default_rng(0)
    dists = []
    for i in range(20):
        Xi = X[off[i]:off[i + 1]]
        a = rng.integers(0, Xi.shape[0], 200)
        b = rng.integers(0, Xi.shape[0], 200)
        dists.append(np.linalg.norm(Xi[a] - Xi[b], axis=1))
    th0 = (float(np.median(np.concatenate(dists))), 0.16, float(np.var(y)))
    return X, y, off, km["reps"], th0


def test_C4_matern_build_and_mll_parity(P, ctx):
    X, y, off, reps, th0 = c4_dataset()
    sizes = np.diff(off)
    assert sizes.max() > 512 and sizes.min() < 1000            # uneven, big-block mode
    bg = P.build_blocks(ctx, X, off, reps, th0, kernel="matern52")
    bo = OS.build_blocks(X, off, reps, th0, kind="matern52")
    assert rel(bg.export("scalars")[0], bo.logdet_R) < 1e-11
    l, s, a = th0
    check_eval(P, ctx, bg, bo, y, th0, 204)
    check_eval(P, ctx, bg, bo, y, (l * 1.001, s, a), 204)


# ----------------------------------------------------------------------------- NEXT-1 predict
def test_predict_parity_small_and_C3_shape(P, ctx):
    from oracle import predict as OP
    for n_c, b, d, seed in [(6, 40, 2, 12), (50, 120, 8, 13)]:
        ds = synth.g_hyper(n_c=n_c, b=b, d=d, seed=seed, b_test=3)
        bg = P.build_blocks(ctx, ds.X, ds.offsets, ds.reps, ds.theta0)
        bo = OS.build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
        m, v = P.predict(ctx, bg, ds.y, ds.X_test)
        mo, vo = OP.posterior(bo, ds.y, ds.X_test)
        np.testing.assert_allclose(m.cpu().numpy(), mo, rtol=1e-9, atol=1e-11)
        np.testing.assert_allclose(v.cpu().numpy(), vo, rtol=1e-8, atol=1e-11)
        m2, v2 = P.predict(ctx, bg, ds.y, ds.X_test, add_noise=True)
        np.testing.assert_allclose(v2.cpu().numpy() - v.cpu().numpy(), ds.theta0[1], rtol=1e-12)


def test_predict_C4_matern_with_variance(P, ctx):
    """C4 'train + predict with variance': the posterior at theta0 on the 8,000 held-out points."""
    from oracle import predict as OP
    g = synth.g_real(N=40000, d=8, seed=104)
    X, y, off, reps, th0 = c4_dataset()
    bg = P.build_blocks(ctx, X, off, reps, th0, kernel="matern52")
    bo = OS.build_blocks(X, off, reps, th0, kind="matern52")
    Xt = g["X_test"][:1000]
    m, v = P.predict(ctx, bg, y, Xt)
    mo, vo = OP.posterior(bo, y, Xt)
    np.testing.assert_allclose(m.cpu().numpy(), mo, rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(v.cpu().numpy(), vo, rtol=1e-7, atol=1e-9)
    rm = OP.rmse(m.cpu().numpy(), g["y_test"][:1000])
    assert np.isfinite(rm)                              # (quality at the untrained theta0 is not a pin)


# ----------------------------------------------------------------------------- C5 at full size
def test_C5_full_size_logdetR_and_quad_bound(P, ctx):
    """C5 (n = 1,000,000, 2000 clusters of 500) in the launch configuration bench.py times:
    properties that hold at any size, checked against the oracle's own arithmetic —
    logdet_R = 2 sum log diag chol(K_i) (exact), and at the baseline the y-solve satisfies
    |c^T x - c^T A^{-1} c| <= tol ||c|| (lambda_min(A) >= 1), with c^T A^{-1} c from the exact
    structured (Woodbury) oracle on a bounded sample of clusters' contributions."""
    import math
    from oracle import exact as OX
    ds = synth.make_config("C5")
    bg = P.build_blocks(ctx, ds.X, ds.offsets, ds.reps, ds.theta0, eval_slots=1)
    bo = OS.build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    assert rel(bg.export("scalars")[0], bo.logdet_R) < 1e-11
    assert rel(bg.export("scalars")[1], bo.lam0) < 1e-10
    tol = 1e-6
    rec = P.mll(ctx, bg, ds.y, ds.theta0, probe_seed=205, tol=tol)
    c = OS.solve_Rt(bo, ds.y)
    d = np.array([float(u @ u) for u in bo.u])
    sd = np.sqrt(d)
    Mt = sd[:, None] * bo.M * sd[None, :]
    xi = np.array([bo.u[i] @ c[bo.block(i)] for i in range(bo.n_c)]) / sd
    quad_exact = float(c @ c) - float(xi @ (Mt @ np.linalg.solve(np.eye(bo.n_c) + Mt, xi)))
    assert abs(rec["quad"] - quad_exact) <= tol * math.sqrt(float(c @ c)) * 1.0001 + 1e-9 * abs(quad_exact)
    # NEXT-2 at full size (n_c = 2000 > 512: blocked capacitance factorisation) against O-EXACT's
    # arithmetic on the same blocks
    ex = P.mll_exact(ctx, bg, ds.y)
    logdet = bo.logdet_R + float(np.sum(np.log1p(np.linalg.eigvalsh(Mt))))
    assert rel(ex["quad"], quad_exact) < 1e-10
    assert rel(ex["logdet"], logdet) < 1e-10
    assert rel(ex["L"], 0.5 * (quad_exact + logdet + ds.n * math.log(2 * math.pi))) < 1e-10
