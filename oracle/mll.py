"""MLL evaluation, numerical gradient, Adam and the training loop.

  Eq. (3)  L = 1/2 y^T K^{-1} y + 1/2 log|K| + n/2 log 2 pi
  Alg. 1 ComputeLoss: PCG for u (line 255), log-det per Eq. (16) by PCG
           (line 256), L = (y^T u + log|K''| + n log 2pi)/2 (lines 257-258; reading P8).
  Eq. (11) numerical gradient; CENTRAL (north_star "2p+1 perturbations")
           and FORWARD_HALVING (Alg. 1; readings P12-P14).
  Adam, gamma = 0.05 (reading P15).
  Algorithm 1: per epoch build R at theta, L_0, gradients, Adam.
Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .cg import cg_batched
from .logdet import pade_trace_terms, slq_term
from .structured import Blocks, Operator, build_blocks, solve_Rt, theta_tuple

LOG2PI = math.log(2.0 * math.pi)


@dataclass
class MLLRecord:
    L: float
    quad: float
    logdet: float
    logdet_pade: float
    logdet_slq: float
    logdet_R: float
    lambda0: float
    iters_y: int
    iters_q: list
    resid_y: float
    resid_q_max: float
    t: np.ndarray = field(default=None, repr=False)
    s: np.ndarray = field(default=None, repr=False)
    mode: str = ""


def mll(blocks: Blocks, y, theta, Z, tol=0.01, max_iter=2000, replay=None,
        logdet_mode="pade") -> MLLRecord:
    """ComputeLoss(R, theta) of Alg. 1 on K''(theta) with R built at theta_0.

    Z: m x n probe matrix (rows z_i, Eq. 9).  replay: None or [k_y, k_Q_1..k_Q_m]."""
    op = Operator(blocks, theta)
    y = np.asarray(y, dtype=np.float64)
    Z = np.asarray(Z, dtype=np.float64)
    m = Z.shape[0]
    c = solve_Rt(blocks, y)                                  # transformed RHS R^{-T} y
    if logdet_mode == "mbcg":
        return _mll_mbcg(blocks, op, y, c, Z, tol, max_iter, replay)
    ry = None if replay is None else [replay[0]]
    rq = None if replay is None else list(replay[1:1 + m])
    sol_y = cg_batched(op.apply, c, tol, max_iter, ry)      # Alg. 1
    quad = float(c @ sol_y.X[:, 0])                          # y^T K''^{-1} y = c^T A^{-1} c
    sol_q = cg_batched(op.apply_Q, Z.T, tol, max_iter, rq)  # Alg. 1, W = Q(A)^{-1} Z
    t = pade_trace_terms(op.apply, Z.T, sol_q.X)             # z^T P(A) Q(A)^{-1} z
    znorm2 = np.einsum("ij,ij->i", Z, Z)
    s = np.array([slq_term(sol_q.alphas[j], sol_q.betas[j], znorm2[j]) for j in range(m)])
    logdet_pade = blocks.logdet_R + float(np.mean(t))       # Eq. (16)
    logdet_slq = blocks.logdet_R + float(np.mean(s))
    logdet = logdet_pade if logdet_mode == "pade" else logdet_slq
    n = y.shape[0]
    L = 0.5 * (quad + logdet + n * LOG2PI)                    # Eq. (3), Alg. 1 l.257-258
    return MLLRecord(L=L, quad=quad, logdet=logdet, logdet_pade=logdet_pade,
                     logdet_slq=logdet_slq, logdet_R=blocks.logdet_R, lambda0=op.lam0,
                     iters_y=int(sol_y.iters[0]), iters_q=[int(k) for k in sol_q.iters],
                     resid_y=float(sol_y.resid[0]), resid_q_max=float(np.max(sol_q.resid)),
                     t=t, s=s, mode=op.mode)


def _mll_mbcg(blocks, op, y, c, Z, tol, max_iter, replay) -> MLLRecord:
    """NEXT-4 (GPyTorch-style mBCG): ONE batched CG on A with
    the columns [c, z_1..z_m] (x_0 = 0, per-column alpha/beta and freezing as in cg_batched);
    quad = c^T x_c; each probe's CG coefficients give A's Lanczos tridiagonal (same formulas as
    for Q(A)), and z^T log(A) z ~ ||z||^2 sum_l tau_l^2 log(theta_l).  No Pade term (NaN)."""
    m = Z.shape[0]
    sol = cg_batched(op.apply, np.column_stack([c, Z.T]), tol, max_iter, replay)
    quad = float(c @ sol.X[:, 0])
    znorm2 = np.einsum("ij,ij->i", Z, Z)
    s = np.array([slq_term(sol.alphas[1 + j], sol.betas[1 + j], znorm2[j], f=np.log) for j in range(m)])
    logdet_slq = blocks.logdet_R + float(np.mean(s))
    n = y.shape[0]
    L = 0.5 * (quad + logdet_slq + n * LOG2PI)
    return MLLRecord(L=L, quad=quad, logdet=logdet_slq, logdet_pade=float("nan"), logdet_slq=logdet_slq,
                     logdet_R=blocks.logdet_R, lambda0=op.lam0, iters_y=int(sol.iters[0]),
                     iters_q=[int(k) for k in sol.iters[1:]], resid_y=float(sol.resid[0]),
                     resid_q_max=float(np.max(sol.resid[1:])), t=None, s=s, mode=op.mode)


def central_perturbations(theta, step=(1e-3, 1e-3, 1e-3)):
    """The 2p+1 = 7 evaluation points theta, theta +- h_i e_i with h_i = step_i * theta_i."""
    th = np.asarray(theta_tuple(theta))
    h = np.asarray(step, dtype=np.float64) * th
    pts = [tuple(th)]
    for i in range(3):
        for sgn in (+1.0, -1.0):
            p = th.copy()
            p[i] = th[i] + sgn * h[i]
            pts.append(tuple(p))
    return pts, h


def numgrad_central(loss, theta, step=(1e-3, 1e-3, 1e-3)):
    """g_i = (L(theta + h_i e_i) - L(theta - h_i e_i)) / (2 h_i); loss: theta -> float."""
    pts, h = central_perturbations(theta, step)
    Ls = [loss(p) for p in pts]
    g = np.array([(Ls[1 + 2 * i] - Ls[2 + 2 * i]) / (2.0 * h[i]) for i in range(3)])
    return Ls[0], g, Ls


def numgrad_forward_halving(loss, theta, L0=None, rel_step0=0.1, threshold=1e-3,
                            threshold_relative=True, max_halvings=20):
    """Eq. (11) + Alg. 1: forward difference, Delta halved until two
    consecutive gradients differ by < threshold (reading P13: relative
    |g - g_prev| < thr * max(1, |g|), cap max_halvings; P14: Delta_0 = 0.1 theta_i)."""
    th = np.asarray(theta_tuple(theta))
    if L0 is None:
        L0 = loss(tuple(th))
    g_out, nh_out = np.zeros(3), np.zeros(3, dtype=np.int64)
    for i in range(3):
        delta = rel_step0 * th[i]
        g_prev = math.inf
        nh = 0
        while True:
            p = th.copy()
            p[i] += delta
            g = (loss(tuple(p)) - L0) / delta
            scale = max(1.0, abs(g)) if threshold_relative else 1.0
            if abs(g - g_prev) < threshold * scale or nh >= max_halvings:
                break
            g_prev = g
            delta *= 0.5
            nh += 1
        g_out[i], nh_out[i] = g, nh
    return L0, g_out, nh_out


@dataclass
class AdamState:
    theta: np.ndarray
    m: np.ndarray = field(default_factory=lambda: np.zeros(3))
    v: np.ndarray = field(default_factory=lambda: np.zeros(3))
    t: int = 0


def adam_step(st: AdamState, g, lr=0.05, b1=0.9, b2=0.999, eps=1e-8, floor=1e-8) -> AdamState:
    """Kingma & Ba Adam on the natural parameters (reading P15), clamped to >= floor."""
    g = np.asarray(g, dtype=np.float64)
    m = b1 * st.m + (1.0 - b1) * g
    v = b2 * st.v + (1.0 - b2) * g * g
    t = st.t + 1
    mhat = m / (1.0 - b1 ** t)
    vhat = v / (1.0 - b2 ** t)
    theta = st.theta - lr * mhat / (np.sqrt(vhat) + eps)
    return AdamState(theta=np.maximum(theta, floor), m=m, v=v, t=t)


def train(X, offsets, reps, y, theta0, Z, epochs=50, lr=0.05, kind="rbf", grad_mode="central",
          step=(1e-3, 1e-3, 1e-3), tol=0.01, max_iter=2000, replay=None, halving_kw=None):
    """Algorithm 1.  replay: None or per-epoch list of per-evaluation replay counts
    (replay[e][k] for the k-th loss evaluation of epoch e, in evaluation order)."""
    st = AdamState(theta=np.asarray(theta_tuple(theta0)))
    records = []
    for e in range(epochs):
        th = tuple(st.theta)
        blocks = build_blocks(X, offsets, reps, th, kind)      # Alg. 1
        ev = []

        def loss(p, _ev=ev, _e=e):
            rp = None if replay is None else replay[_e][len(_ev)]
            rec = mll(blocks, y, p, Z, tol, max_iter, rp)
            _ev.append(rec)
            return rec.L

        if grad_mode == "central":
            L0, g, _ = numgrad_central(loss, th, step)
            nh = None
        else:
            L0, g, nh = numgrad_forward_halving(loss, th, **(halving_kw or {}))
        records.append(dict(epoch=e, theta=np.array(th), L0=L0, grad=g.copy(), evals=ev,
                            halvings=nh))
        st = adam_step(st, g, lr)
    return st, records
