"""GPU parity of NEXT-2, the exact structured evaluator (determinant lemma + Woodbury on
Eq. (28)-(29)), against the FP64 oracle's O-EXACT (`oracle/exact.py`, pinned
against dense Cholesky in tests/test_oracle_pins.py), and of the posterior at n_c > 512 (the
capacitance matrix through the blocked big-block factorisation)."""
import math

import numpy as np
import pytest

import synth
from oracle import exact as OX
from oracle import structured as OS

pytestmark = pytest.mark.gpu

TIGHT = 1e-11


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


def check(P, ctx, X, off, reps, y, th, kind="rbf", rtol=TIGHT):
    bg = P.build_blocks(ctx, X, off, reps, th, kernel=kind)
    ex = P.mll_exact(ctx, bg, y)
    Lo, qo, ldo = OX.exact_structured(X, off, reps, y, th, kind=kind)
    assert rel(ex["L"], Lo) < rtol, (ex, Lo)
    assert rel(ex["quad"], qo) < rtol, (ex, qo)
    assert rel(ex["logdet"], ldo) < rtol, (ex, ldo)
    return bg, ex


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_exact_mll_g_hyper(P, ctx, cfg):
    ds = synth.make_config(cfg)
    l, s, a = ds.theta0
    for th in [ds.theta0, (0.5 * l, s, a), (l, 2 * s, 0.7 * a)]:
        check(P, ctx, ds.X, ds.offsets, ds.reps, ds.y, th)


def test_exact_mll_uneven_big_blocks(P, ctx):
    rng = np.random.default_rng(5)
    sizes = [700, 300, 1100, 17, 90]
    reps = rng.uniform(-10, 10, size=(len(sizes), 3))
    X = np.concatenate([reps[i] + rng.standard_normal((s, 3)) for i, s in enumerate(sizes)])
    y = np.cos(X).sum(axis=1) + 0.3 * rng.standard_normal(X.shape[0])
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    check(P, ctx, X, off, reps, y, (1.2, 0.1, 1.5))
    check(P, ctx, X, off, reps, y, (0.8, 0.05, 2.0), kind="matern52")


def test_exact_mll_many_clusters_big_capacitance(P, ctx):
    """n_c = 600 > 512: C = I + M~ is factorised by the blocked multi-launch kernels."""
    ds = synth.g_hyper(n_c=600, b=12, d=3, seed=31)
    bg, ex = check(P, ctx, ds.X, ds.offsets, ds.reps, ds.y, ds.theta0, rtol=1e-10)
    b = OS.build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    d, sd, Mt, mu, V = OX._eig_structure(b)
    assert rel(ex["logdet_C"], float(np.sum(np.log1p(mu)))) < 1e-10


def test_exact_vs_estimator_at_tight_tolerance(P, ctx):
    """The PCG y-solve at tol 1e-10 reproduces the exact quadratic form (same operator), and the
    Pade/SLQ log-dets sit within their estimator error of the exact one (Pade
    bias <= 3e-5 relative at lambda = 0.5 l; Hutchinson spread with m = 8 probes)."""
    ds = synth.make_config("C2")
    bg = P.build_blocks(ctx, ds.X, ds.offsets, ds.reps, ds.theta0)
    ex = P.mll_exact(ctx, bg, ds.y)
    rec = P.mll(ctx, bg, ds.y, ds.theta0, probe_seed=202, tol=1e-10)
    assert rel(rec["quad"], ex["quad"]) < 1e-9
    assert rel(rec["logdet_pade"], ex["logdet"]) < 2e-2
    assert rel(rec["logdet_slq"], ex["logdet"]) < 2e-2


def test_predict_many_clusters(P, ctx):
    from oracle import predict as OP
    ds = synth.g_hyper(n_c=600, b=12, d=3, seed=32, b_test=1)
    bg = P.build_blocks(ctx, ds.X, ds.offsets, ds.reps, ds.theta0)
    bo = OS.build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    Xt = ds.X_test[:300]
    m, v = P.predict(ctx, bg, ds.y, Xt)
    mo, vo = OP.posterior(bo, ds.y, Xt)
    np.testing.assert_allclose(m.cpu().numpy(), mo, rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(v.cpu().numpy(), vo, rtol=1e-8, atol=1e-10)

