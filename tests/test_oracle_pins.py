"""Pins of the oracle against what the paper and the mathematics fix.

Every function in oracle/ is checked here against something other than itself:
library routines (sklearn, scipy, LAPACK via numpy), closed forms, invariants, brute force.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.special
import scipy.stats
from scipy.linalg import solve_triangular

import synth
from oracle import exact, kernels
from oracle.cg import cg_batched
from oracle.logdet import lanczos_tridiag_from_cg, pade_r, pade_trace_terms, slq_term
from oracle.mll import (AdamState, adam_step, mll, numgrad_central, numgrad_forward_halving,
                        central_perturbations)
from oracle.structured import (DegenerateReps, NotSPD, Operator, build_blocks,
                               chol_upper_with_jitter, dense_Kpp, dense_R, krep_and_M,
                               smallest_eig, solve_Rt)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def small(n_c=5, b=12, d=2, seed=7):
    return synth.g_hyper(n_c, b, d, seed)


# --------------------------------------------------------------------------- kernels
def test_kernel_as_printed_spec_examples():
    for ex in GOLD["kernel_as_printed"]:
        x = np.zeros(3)
        xp = np.array([ex["dist"], 0.0, 0.0])
        v = kernels.kernel_eval(kernels.RBF_AS_PRINTED, x, xp, ex["lengthscale"], ex["alpha"])
        assert v == pytest.approx(ex["value"], rel=1e-15)


def test_rbf_matches_sklearn():
    from sklearn.gaussian_process.kernels import RBF as SkRBF
    rng = np.random.default_rng(0)
    A, B = rng.normal(size=(7, 4)), rng.normal(size=(5, 4))
    for lam, alpha in [(0.3, 1.0), (1.7, 2.5)]:
        K = kernels.kernel_matrix(kernels.RBF, A, B, lam, alpha)
        np.testing.assert_allclose(K, alpha * SkRBF(length_scale=lam)(A, B), rtol=1e-12)


def test_matern52_matches_sklearn_and_bessel():
    from sklearn.gaussian_process.kernels import Matern
    rng = np.random.default_rng(1)
    A, B = rng.normal(size=(6, 3)), rng.normal(size=(8, 3))
    lam, alpha, nu = 0.8, 1.9, 2.5
    K = kernels.kernel_matrix(kernels.MATERN52, A, B, lam, alpha)
    np.testing.assert_allclose(K, alpha * Matern(length_scale=lam, nu=nu)(A, B), rtol=1e-13)
    rho = np.sqrt(((A[:, None, :] - B[None, :, :]) ** 2).sum(-1))
    s = np.sqrt(2 * nu) * rho / lam
    general = alpha * 2 ** (1 - nu) / scipy.special.gamma(nu) * s ** nu * scipy.special.kv(nu, s)
    np.testing.assert_allclose(K, general, rtol=1e-12)


def test_kernel_matrix_bitwise_symmetric_exact_diagonal():
    ds = small(3, 20, 5)
    K = kernels.kernel_matrix(kernels.RBF, ds.X, ds.X, 0.7, 1.3)
    assert np.array_equal(K, K.T)
    assert np.all(np.diag(K) == 1.3)


# --------------------------------------------------------------------------- blocks
def test_cholesky_spec_examples():
    for key in ("cholesky", "cholesky_1x1"):
        ex = GOLD[key]
        R, eps = chol_upper_with_jitter(np.array(ex["K"]))
        np.testing.assert_allclose(R, np.array(ex["R"]), rtol=1e-15, atol=0)
        assert eps == 0.0
        assert 2 * np.sum(np.log(np.diag(R))) == pytest.approx(ex["logdet_R"], rel=1e-15)


def test_cholesky_negative_definite_fails_and_singular_gets_jitter():
    with pytest.raises(NotSPD):
        chol_upper_with_jitter(-np.eye(3), block=2)
    Ksing = np.ones((4, 4))                    # PSD, rank 1 -> jitter ladder succeeds
    R, eps = chol_upper_with_jitter(Ksing)
    assert eps > 0
    np.testing.assert_allclose(R.T @ R, Ksing + eps * np.eye(4), atol=1e-12)


def test_jitter_ladder_needs_exactly_t2():
    """SPEC.md:125 ladder eps_t = 1e-8 mean(diag K) 10^t: a symmetric K whose smallest eigenvalue is
    -10^1.5 base (base = 1e-8 mean diag) fails for t = 0, 1 (eps < |lambda_min|) and succeeds at
    t = 2, so the returned jitter must be exactly base * 100 and R^T R = K + 100 base I."""
    rng = np.random.default_rng(9)
    n = 12
    Q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    mu = np.linspace(1.0, 3.0, n)
    base_guess = 1e-8 * np.mean(mu)
    mu[0] = -(10 ** 1.5) * base_guess
    K = (Q * mu) @ Q.T
    K = 0.5 * (K + K.T)
    base = 1e-8 * float(np.mean(np.diag(K)))            # = 1e-8 mean eig (trace invariance)
    assert 10 * base < -mu[0] < 100 * base
    with pytest.raises(np.linalg.LinAlgError):
        np.linalg.cholesky(K + base * 10 * np.eye(n))     # t = 1 still fails
    R, eps = chol_upper_with_jitter(K)
    assert eps == base * 10.0 ** 2
    np.testing.assert_allclose(R.T @ R, K + eps * np.eye(n), rtol=0, atol=1e-13)


def test_scale_step_on_jittered_block_matches_dense():
    """Eq. (25) scale step on a JITTERED block: the model's block is K_i + (sigma_0^2 + eps_i) I, so
    the shortcut must use (sigma_0^2 + eps_i) r H (SURVEY §8(c) step 2 / DESIGN jitter reading).
    Brute force: dense R^-T K''(theta') R^-1 with the jittered diagonal, entry by entry."""
    rng = np.random.default_rng(12)
    X = np.concatenate([np.zeros((6, 2)), rng.normal(size=(7, 2)) + 4.0, rng.normal(size=(5, 2)) - 4.0])
    off = np.array([0, 6, 13, 18], dtype=np.int64)
    reps = np.array([[0.0, 0.0], [4.0, 4.0], [-4.0, -4.0]])
    th0 = (1.0, 1e-18, 1.0)                              # cluster 0: 6 identical points -> singular
    b = build_blocks(X, off, reps, th0)
    assert b.jitter[0] > 0 and b.jitter[1] == 0 and b.jitter[2] == 0
    ds = synth.Dataset(X=X, y=np.zeros(18), offsets=off, reps=reps, theta0=th0)
    V = rng.normal(size=(18, 3))
    Rinv = np.linalg.inv(dense_R(b))
    for r in (0.5, -0.3):
        th = (th0[0], th0[1], th0[2] * (1 + r))
        op = Operator(b, th)
        assert op.mode == "scale"
        A = Rinv.T @ _brute_K(ds, th, b) @ Rinv
        # tolerance: the jittered block has cond ~ 6 alpha / eps_0 ~ 1e8, so both routes carry
        # ~cond x 1e-16 = 1e-8 rounding; the eps-dropping mistake below is 1e6 times larger
        np.testing.assert_allclose(op.apply(V), A @ V, rtol=1e-6, atol=1e-6 * np.abs(A @ V).max())
        # dropping eps_i from the shortcut would be a gross error here (eps_i H ~ I on that block)
        wrong = (1 + r) * V[:6] - th0[1] * r * np.linalg.solve(b.R[0], np.linalg.solve(b.R[0].T, V[:6]))
        assert np.abs(wrong - op.apply(V)[:6]).max() > 0.01


def test_build_blocks_invariants():
    ds = small(4, 15, 3)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    logdet_eig = 0.0
    for i in range(b.n_c):
        Ki = b.K_block(i, ds.theta0)
        np.testing.assert_allclose(b.R[i].T @ b.R[i], Ki, rtol=1e-13, atol=1e-14)
        logdet_eig += float(np.sum(np.log(np.linalg.eigvalsh(Ki))))
        np.testing.assert_allclose(b.R[i].T @ b.u[i], np.ones(Ki.shape[0]), atol=1e-12)
    assert b.logdet_R == pytest.approx(logdet_eig, rel=1e-13)


def test_smallest_eig_closed_form_and_degenerate_reps():
    ex = GOLD["smallest_eig_2x2"]
    a, c = ex["a"], ex["c"]
    assert smallest_eig(np.array([[a, c], [c, a]])) == pytest.approx(ex["value"], rel=1e-14)
    assert smallest_eig(np.eye(3)) == pytest.approx(1.0, rel=1e-15)
    with pytest.raises(DegenerateReps):
        krep_and_M("rbf", np.zeros((3, 2)), (1.0, 0.1, 1.0))


# --------------------------------------------------------------------------- operator
def _brute_K(ds, theta, b):
    """Entry-by-entry K'' from Eq. (17), (27), (28) with plain loops (independent of dense_Kpp)."""
    lam, s2, alpha = theta
    n = ds.n
    clus = np.repeat(np.arange(ds.n_c), np.diff(ds.offsets))
    Krep = kernels.kernel_matrix("rbf", ds.reps, ds.reps, lam, alpha)
    lam0 = np.linalg.eigvalsh(Krep)[0]
    K = np.empty((n, n))
    for p in range(n):
        for q in range(n):
            ip, iq = clus[p], clus[q]
            if ip == iq:
                dx = ds.X[p] - ds.X[q]
                K[p, q] = alpha * math.exp(-(dx @ dx) / (2 * lam * lam)) + (Krep[ip, ip] - lam0)
                if p == q:
                    K[p, q] += s2 + b.jitter[ip]
            else:
                K[p, q] = Krep[ip, iq]
    return K


@pytest.mark.parametrize("which", ["baseline", "noise", "scale", "generic", "all"])
def test_operator_matches_dense_brute_force(which):
    ds = small(4, 9, 2, seed=3)
    th0 = ds.theta0
    b = build_blocks(ds.X, ds.offsets, ds.reps, th0)
    th = {"baseline": th0, "noise": (th0[0], th0[1] * 1.3, th0[2]),
          "scale": (th0[0], th0[1], th0[2] * 0.8), "generic": (th0[0] * 1.1, th0[1], th0[2]),
          "all": (th0[0] * 0.9, th0[1] * 1.2, th0[2] * 1.1)}[which]
    op = Operator(b, th)
    assert op.mode == ("generic" if which == "all" else which)
    Kb = _brute_K(ds, th, b)
    Rd = dense_R(b)
    Rinv = np.linalg.inv(Rd)
    A = Rinv.T @ Kb @ Rinv
    V = np.random.default_rng(5).normal(size=(ds.n, 3))
    np.testing.assert_allclose(op.apply(V), A @ V, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(dense_Kpp(b, th), Kb, rtol=1e-13, atol=1e-14)


def test_shortcuts_equal_generic_route():
    """Eq. (24)/(25) with H = R^-T R^-1 equal the generic R^-T K R^-1 route."""
    ds = small(5, 10, 3, seed=11)
    th0 = ds.theta0
    b = build_blocks(ds.X, ds.offsets, ds.reps, th0)
    V = np.random.default_rng(2).normal(size=(ds.n, 4))
    for th in [(th0[0], th0[1] + 0.03, th0[2]), (th0[0], th0[1], th0[2] * 1.07)]:
        op = Operator(b, th)
        assert op.mode in ("noise", "scale")
        gen = Operator(b, th)
        gen.mode = "generic"
        _, gen.lam0, gen.Mp = krep_and_M("rbf", b.reps, th)
        gen.Kd = [b.K_block(i, th) for i in range(b.n_c)]
        np.testing.assert_allclose(op.apply(V), gen.apply(V), rtol=1e-12, atol=1e-12)


def test_baseline_operator_is_identity_plus_low_rank_and_spd():
    ds = small(6, 8, 2, seed=4)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    W = np.zeros((ds.n, ds.n_c))
    for i in range(ds.n_c):
        W[b.block(i), i] = b.u[i]
    np.testing.assert_allclose(W.T @ W, np.diag(np.diag(W.T @ W)), atol=0)
    A = Operator(b, ds.theta0).apply(np.eye(ds.n))
    np.testing.assert_allclose(A, np.eye(ds.n) + W @ b.M @ W.T, atol=1e-13)
    # lambda_min(K'') >= sigma^2 (K_diag - sigma^2 I psd and E M E^T psd)
    K = dense_Kpp(b, ds.theta0)
    assert np.linalg.eigvalsh(K)[0] >= ds.theta0[1] * (1 - 1e-9)
    ev = np.linalg.eigvalsh(0.5 * (A + A.T))
    assert ev[0] >= 1 - 1e-12
    assert len(np.unique(np.round(ev, 8))) <= ds.n_c + 1          # Eq. (29)


# --------------------------------------------------------------------------- CG
def test_cg_identity_one_iteration_and_diag_four():
    b = np.array([1.0, 2.0, -1.0, 0.5])
    r = cg_batched(lambda P: P, b, tol=1e-12)
    assert r.iters[0] == 1
    np.testing.assert_allclose(r.X[:, 0], b, rtol=1e-15)
    Dg = np.array([1.0, 2.0, 3.0, 4.0])
    r = cg_batched(lambda P: Dg[:, None] * P, b, tol=1e-12)
    assert r.iters[0] <= 4
    np.testing.assert_allclose(r.X[:, 0], b / Dg, rtol=1e-12)


def test_cg_batched_columns_independent_and_replay():
    rng = np.random.default_rng(3)
    G = rng.normal(size=(30, 30))
    A = G @ G.T + 30 * np.eye(30)
    B = rng.normal(size=(30, 3))
    r = cg_batched(lambda P: A @ P, B, tol=1e-6)
    for j in range(3):
        rj = cg_batched(lambda P: A @ P, B[:, j], tol=1e-6)
        assert rj.iters[0] == r.iters[j]
        np.testing.assert_allclose(rj.X[:, 0], r.X[:, j], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(r.X, np.linalg.solve(A, B), rtol=1e-5, atol=1e-6)
    rp = cg_batched(lambda P: A @ P, B, tol=1e-6, replay=[2, 3, 4])
    assert list(rp.iters) == [2, 3, 4]


def test_cg_iterations_bounded_by_distinct_eigenvalues():
    """at the baseline CG on A converges in <= n_c + 1 iterations (FP64)."""
    ds = small(6, 20, 2, seed=9)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    op = Operator(b, ds.theta0)
    c = solve_Rt(b, ds.y)
    r = cg_batched(op.apply, c, tol=1e-9 * np.linalg.norm(c))
    assert r.iters[0] <= ds.n_c + 1


# --------------------------------------------------------------------------- log-det
def test_pade_scalar_properties():
    assert pade_r(1.0) == 0.0
    h = 1e-6
    assert (pade_r(1 + h) - pade_r(1 - h)) / (2 * h) == pytest.approx(1.0, rel=1e-9)
    for x in [0.9, 1.1, 1.5]:
        assert abs(pade_r(x) - math.log(x)) < abs(x - 1) ** 5          # O(t^5) at 1


def test_pade_trace_unit_probes_equals_trace_r_of_A():
    ds = small(4, 6, 2, seed=12)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    op = Operator(b, ds.theta0)
    A = op.apply(np.eye(ds.n))
    ev, V = np.linalg.eigh(0.5 * (A + A.T))
    Qinv = V @ np.diag(1.0 / (ev ** 2 + 4 * ev + 1)) @ V.T
    Z = np.eye(ds.n)
    t = pade_trace_terms(op.apply, Z, Qinv @ Z)
    assert float(np.sum(t)) == pytest.approx(float(np.sum(pade_r(ev))), rel=1e-11)
    assert float(np.sum(pade_r(ev))) == pytest.approx(
        float(np.sum(pade_r(exact.spectrum_A_baseline(b)))), rel=1e-11)


def test_slq_tridiagonal_is_lanczos():
    """CG coefficients give the Lanczos tridiagonal: its spectrum at convergence is Q(A)'s
    restricted to the Krylov space; SLQ with f = identity returns z^T Q(A) z exactly."""
    rng = np.random.default_rng(4)
    G = rng.normal(size=(12, 12))
    A = G @ G.T / 12 + np.eye(12)
    z = np.sign(rng.normal(size=12))
    r = cg_batched(lambda P: A @ P, z, tol=1e-13, max_iter=100)
    d, e = lanczos_tridiag_from_cg(r.alphas[0], r.betas[0])
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    np.testing.assert_allclose(np.linalg.eigvalsh(T), np.linalg.eigvalsh(A), rtol=1e-9)
    assert slq_term(r.alphas[0], r.betas[0], z @ z, f=lambda m: m) == pytest.approx(z @ A @ z, rel=1e-10)
    inv = slq_term(r.alphas[0], r.betas[0], z @ z, f=lambda m: 1 / m)
    assert inv == pytest.approx(z @ np.linalg.solve(A, z), rel=1e-9)


def test_mll_tight_tol_matches_closed_forms():
    """At the baseline, tight tol: quad = Woodbury, t_j = zeta^T r(I+M~) zeta, s_j = z^T log(A) z."""
    ds = small(5, 14, 2, seed=21)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    Z = synth.probes(5, 4, ds.n)
    rec = mll(b, ds.y, ds.theta0, Z, tol=1e-11)
    L_ex, quad_ex, logdet_ex = exact.exact_structured(ds.X, ds.offsets, ds.reps, ds.y, ds.theta0)
    assert rec.quad == pytest.approx(quad_ex, rel=1e-10)
    for j in range(4):
        tj = exact.probe_quadform_baseline(b, Z[j], pade_r)
        sj = exact.probe_quadform_baseline(b, Z[j], np.log)
        assert rec.t[j] == pytest.approx(tj, rel=1e-9, abs=1e-9)
        assert rec.s[j] == pytest.approx(sj, rel=1e-8, abs=1e-8)


def test_mll_tol_bound_on_quad():
    """|c^T x_k - c^T A^-1 c| <= ||c|| ||r_k|| <= tol ||c||  since lambda_min(A) >= 1."""
    ds = small(6, 25, 3, seed=8)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    Z = synth.probes(1, 2, ds.n)
    rec = mll(b, ds.y, ds.theta0, Z, tol=0.01)
    _, quad_ex, _ = exact.exact_structured(ds.X, ds.offsets, ds.reps, ds.y, ds.theta0)
    c = solve_Rt(b, ds.y)
    assert abs(rec.quad - quad_ex) <= 0.01 * np.linalg.norm(c)


def test_single_cluster_is_exact_gp():
    """n_c = 1 => M = [0] => K'' = K => the exact GP MLL (scipy multivariate normal)."""
    ds = synth.g_hyper(1, 40, 2, seed=31)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    assert b.M.shape == (1, 1) and b.M[0, 0] == 0.0
    Z = synth.probes(3, 8, ds.n)
    rec = mll(b, ds.y, ds.theta0, Z, tol=0.01)
    assert rec.iters_y == 1 and all(k == 1 for k in rec.iters_q)
    assert np.all(np.abs(rec.t) < 1e-9)
    K = exact.dense_true_K(ds.X, ds.theta0)
    Lref = -scipy.stats.multivariate_normal(mean=np.zeros(ds.n), cov=K).logpdf(ds.y)
    assert rec.L == pytest.approx(Lref, rel=1e-12)


def test_hutchinson_mean_is_trace():
    """E[z^T B z] = tr B for Rademacher z; variance 2(||B||_F^2 - sum B_ii^2) (textbook)."""
    ds = small(4, 8, 2, seed=13)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    op = Operator(b, ds.theta0)
    A = op.apply(np.eye(ds.n))
    ev, V = np.linalg.eigh(0.5 * (A + A.T))
    Bm = V @ np.diag(pade_r(ev)) @ V.T
    m = 4000
    Z = synth.probes(77, m, ds.n)
    est = np.einsum("ij,jk,ik->i", Z, Bm, Z)
    var = 2 * (np.sum(Bm * Bm) - np.sum(np.diag(Bm) ** 2))
    assert abs(est.mean() - np.trace(Bm)) < 4 * math.sqrt(var / m)


# --------------------------------------------------------------------------- exact oracles
def test_exact_equals_dense_and_scipy():
    ds = small(5, 20, 2, seed=17)
    for th in [ds.theta0, (ds.theta0[0] * 1.3, 0.2, 0.7)]:
        L1, q1, ld1 = exact.exact_structured(ds.X, ds.offsets, ds.reps, ds.y, th)
        L2, q2, ld2 = exact.dense_structured_mll(ds.X, ds.offsets, ds.reps, ds.y, th)
        assert ld1 == pytest.approx(ld2, rel=1e-12)
        assert q1 == pytest.approx(q2, rel=1e-11)
        b = build_blocks(ds.X, ds.offsets, ds.reps, th)
        K = dense_Kpp(b, th)
        L3 = -scipy.stats.multivariate_normal(mean=np.zeros(ds.n), cov=K).logpdf(ds.y)
        assert L1 == pytest.approx(L3, rel=1e-11)


def test_analytic_gradient_matches_central_fd_of_exact():
    ds = small(4, 15, 2, seed=23)
    th = ds.theta0
    g = exact.analytic_grad_structured(ds.X, ds.offsets, ds.reps, ds.y, th)
    loss = lambda p: exact.exact_structured(ds.X, ds.offsets, ds.reps, ds.y, p)[0]
    _, gfd, _ = numgrad_central(loss, th, step=(1e-5, 1e-5, 1e-5))
    np.testing.assert_allclose(gfd, g, rtol=1e-6)


# --------------------------------------------------------------------------- gradient / Adam
def test_numgrad_central_closed_form():
    f = lambda p: p[0] ** 2 + 3 * p[1] ** 2 + p[2] ** 3
    th = (0.7, 1.3, 2.0)
    L0, g, Ls = numgrad_central(f, th, step=(1e-4, 1e-4, 1e-4))
    np.testing.assert_allclose(g, [2 * 0.7, 6 * 1.3, 3 * 4.0], rtol=1e-7)
    pts, h = central_perturbations(th, (1e-3,) * 3)
    assert len(pts) == 7 and pts[0] == th
    np.testing.assert_allclose(h, np.array(th) * 1e-3)


def test_numgrad_forward_halving_converges():
    f = lambda p: p[0] ** 2 + math.sin(p[1]) + p[2] ** 3
    th = (0.7, 1.3, 2.0)
    L0, g, nh = numgrad_forward_halving(f, th, threshold=1e-6)
    np.testing.assert_allclose(g, [1.4, math.cos(1.3), 12.0], rtol=1e-4)
    assert np.all(nh > 0) and np.all(nh <= 20)


def test_adam_first_step_is_lr_sign():
    lr = GOLD["adam_first_step"]["lr"]
    st = AdamState(theta=np.array([1.0, 1.0, 1.0]))
    st2 = adam_step(st, np.array([3.0, -0.2, 0.0]), lr)
    np.testing.assert_allclose(st2.theta, [1 - lr, 1 + lr, 1.0], rtol=1e-7)
    st3 = adam_step(AdamState(theta=np.array([0.01, 1.0, 1.0])), np.array([5.0, 0, 0]), lr)
    assert st3.theta[0] == 1e-8                      # clamp


def test_probes_are_rademacher_and_reproducible():
    Z = synth.probes(123, 4, 1000)
    assert set(np.unique(Z)) == {-1.0, 1.0}
    assert np.array_equal(Z, synth.probes(123, 4, 1000))
    assert abs(Z.mean()) < 0.1
    # column j is a prefix-stable stream in p
    assert np.array_equal(synth.probes(123, 4, 10), Z[:, :10])


def test_generator_shapes_and_nonoverlap():
    ds = synth.make_config("C1")
    assert ds.n == 1000 and ds.n_c == 10 and ds.d == 2
    for i in range(ds.n_c):
        Xi = ds.X[ds.offsets[i]:ds.offsets[i + 1]]
        assert np.all(np.linalg.norm(Xi - ds.reps[i], axis=1) <= ds.meta["rho"] + 1e-12)
    assert ds.meta["rho"] < ds.meta["l"] / 2


# ----------------------------------------------------------------------------- NEXT-1 predict
def test_predict_structured_equals_dense_Kpp():
    from oracle import predict as OP
    ds = synth.g_hyper(n_c=6, b=40, d=2, seed=12, b_test=5)
    bo = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    m1, v1 = OP.posterior(bo, ds.y, ds.X_test)
    m2, v2 = OP.dense_posterior(bo, ds.y, ds.X_test)
    np.testing.assert_allclose(m1, m2, rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(v1, v2, rtol=1e-8, atol=1e-11)
    # (var may be slightly negative: K* is the exact kernel while K'' approximates the
    #  off-diagonal blocks, so K** - K*^T K''^{-1} K* is not a Schur complement of one PSD matrix)


def test_predict_single_cluster_is_exact_gp_and_sklearn():
    """n_c = 1 => M = [0] => K'' = K: the textbook GP posterior; sklearn's GaussianProcessRegressor
    with the same fixed kernel gives the same latent mean and std."""
    from sklearn.gaussian_process import GaussianProcessRegressor
    from sklearn.gaussian_process.kernels import RBF as SkRBF, ConstantKernel
    from oracle import predict as OP
    rng = np.random.default_rng(3)
    X = rng.uniform(-2, 2, size=(60, 2))
    y = np.sin(X[:, 0]) + 0.1 * rng.standard_normal(60)
    Xt = rng.uniform(-2, 2, size=(7, 2))
    th = (0.8, 0.05, 1.7)
    bo = build_blocks(X, np.array([0, 60]), X.mean(axis=0, keepdims=True), th)
    m, v = OP.posterior(bo, y, Xt)
    gp = GaussianProcessRegressor(ConstantKernel(th[2], "fixed") * SkRBF(th[0], "fixed"), alpha=th[1],
                                  optimizer=None, normalize_y=False).fit(X, y)
    ms, ss = gp.predict(Xt, return_std=True)
    np.testing.assert_allclose(m, ms, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(np.sqrt(v), ss, rtol=1e-7)


def test_predict_one_point_closed_form_spec_365():
    """one training point, test point at the same location: mean = alpha/(alpha+s2) y."""
    from oracle import predict as OP
    X = np.array([[0.3, -0.2]])
    bo = build_blocks(X, np.array([0, 1]), X, (1.0, 0.5, 2.0))
    m, v = OP.posterior(bo, np.array([1.7]), X)
    assert abs(m[0] - 2.0 / 2.5 * 1.7) < 1e-14
    assert abs(v[0] - (2.0 - 2.0 * 2.0 / 2.5)) < 1e-14
    assert OP.rmse([1.0, 3.0], [0.0, 0.0]) == pytest.approx(np.sqrt(5.0))


# --------------------------------------------------------------------------- NEXT-4 mBCG estimator
def test_mbcg_baseline_tight_tol_is_exact_log_quadform():
    """At the baseline A = I + W M W^T has <= n_c + 1 distinct eigenvalues, so tight-tol CG on A
    terminates with an exact Lanczos quadrature: s_j = z^T log(A) z (closed form), quad = Woodbury."""
    ds = small(5, 14, 2, seed=21)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    Z = synth.probes(5, 4, ds.n)
    rec = mll(b, ds.y, ds.theta0, Z, tol=1e-11, logdet_mode="mbcg")
    _, quad_ex, logdet_ex = exact.exact_structured(ds.X, ds.offsets, ds.reps, ds.y, ds.theta0)
    assert rec.quad == pytest.approx(quad_ex, rel=1e-10)
    for j in range(4):
        sj = exact.probe_quadform_baseline(b, Z[j], np.log)
        assert rec.s[j] == pytest.approx(sj, rel=1e-8, abs=1e-8)
    assert max(rec.iters_q) <= b.n_c + 1
    assert math.isnan(rec.logdet_pade) and rec.logdet == rec.logdet_slq


def test_mbcg_perturbed_full_krylov_matches_dense_log():
    """Off the baseline (noise step: A = I + WMW^T + d H), CG run to n iterations on a tiny n is
    a full Lanczos: z^T log(A) z equals the dense eigen-decomposition value."""
    ds = small(3, 8, 2, seed=23)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    l, s, a = ds.theta0
    th = (l, 1.3 * s, a)
    Z = synth.probes(9, 3, ds.n)
    rec = mll(b, ds.y, th, Z, tol=1e-13, max_iter=ds.n, logdet_mode="mbcg")
    op = Operator(b, th)
    A = op.apply(np.eye(ds.n))
    w, V = np.linalg.eigh(0.5 * (A + A.T))
    for j in range(3):
        zl = float(Z[j] @ (V @ (np.log(w) * (V.T @ Z[j]))))
        assert rec.s[j] == pytest.approx(zl, rel=1e-7, abs=1e-8)
    c = solve_Rt(b, ds.y)
    assert rec.quad == pytest.approx(float(c @ np.linalg.solve(A, c)), rel=1e-10)


def test_mbcg_vs_pade_estimators_agree_within_pade_bias():
    """Same probes: the SLQ-on-A and Pade-on-Q(A) log-dets agree within the Pade bias + CG error
    (Pade bias <= 3e-5 relative at lambda = 0.5 l)."""
    ds = small(6, 30, 3, seed=24)
    b = build_blocks(ds.X, ds.offsets, ds.reps, ds.theta0)
    Z = synth.probes(2, 8, ds.n)
    l, s, a = ds.theta0
    for th in [ds.theta0, (1.01 * l, s, a)]:
        r1 = mll(b, ds.y, th, Z, tol=1e-8, logdet_mode="mbcg")
        r2 = mll(b, ds.y, th, Z, tol=1e-8)
        assert r1.logdet_slq == pytest.approx(r2.logdet_slq, rel=1e-7)
        assert r1.logdet == pytest.approx(r2.logdet_pade, rel=1e-3)
        assert r1.quad == pytest.approx(r2.quad, rel=1e-9)
