"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/nugpr.h
declares, and its host-only helpers (no device work) agree with independent references."""
import ctypes
import os
import re

import numpy as np
import pytest
import scipy.linalg

import paper_2510_12128_b200 as P
from paper_2510_12128_b200 import _native as N
from oracle.mll import AdamState, adam_step as oracle_adam

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "nugpr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nugpr_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIB_PATH):
        from paper_2510_12128_b200 import build
        build.build()
    return N.lib()


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert "nugpr_mll" in syms and "nugpr_build_blocks" in syms and len(syms) >= 15
    raw = ctypes.CDLL(N.LIB_PATH)
    missing = [s for s in syms if not hasattr(raw, s)]
    assert not missing, f"declared but not exported: {missing}"
    assert set(N.EXPORTED) <= set(syms)


def test_version_and_errors(lib):
    assert "sm_100a" in P.version()
    with pytest.raises(P.NugprError) as e:
        P.shard_plan(0, [1.0])
    assert e.value.name == "INVALID_ARG"


def test_workspace_size_validation(lib):
    off = np.array([0, 100, 200, 300], dtype=np.int64)
    n1 = P.workspace_size(off, 3, 2, 1)
    n7 = P.workspace_size(off, 3, 2, 7)
    assert n7 > n1 > 3 * 104 * 104 * 8 * 2
    with pytest.raises(P.NugprError) as e:
        P.workspace_size(np.array([0, 5, 5, 9]), 3, 2, 1)
    assert e.value.name == "SHAPE"
    with pytest.raises(P.NugprError) as e:
        P.workspace_size(np.array([1, 5, 9]), 2, 2, 1)
    assert e.value.name == "SHAPE"
    with pytest.raises(P.NugprError) as e:
        P.workspace_size(np.array([0, 9000]), 1, 2, 1)   # cluster larger than this build's limit (8192)
    assert e.value.name == "SHAPE"
    big = P.workspace_size(np.array([0, 5000]), 1, 2, 1)       # big-block mode (ld > 512)
    assert big > 2 * 5000 * 5000 * 8


def test_adam_step_matches_oracle(lib):
    rng = np.random.default_rng(0)
    st = np.zeros(10)
    st[:3] = [0.7, 0.16, 1.2]
    ost = AdamState(theta=st[:3].copy())
    for _ in range(5):
        g = rng.normal(size=3) * 10
        st = P.adam_step(st, g, 0.05)
        ost = oracle_adam(ost, g, 0.05)
        np.testing.assert_allclose(st[:3], ost.theta, rtol=1e-15)
        np.testing.assert_allclose(st[3:6], ost.m, rtol=1e-15)
        np.testing.assert_allclose(st[6:9], ost.v, rtol=1e-15)
    assert st[9] == 5


def test_shard_plan_lpt(lib):
    costs = [1.0, 3.0, 3.0, 2.0, 2.0, 2.0, 2.0]
    for world in (1, 2, 4, 7, 8):
        own = P.shard_plan(world, costs)
        assert own.min() >= 0 and own.max() < world
        loads = np.bincount(own, weights=costs, minlength=world)
        # LPT bound: makespan <= 4/3 OPT, OPT >= max(sum/world, max cost)
        opt_lb = max(sum(costs) / world, max(costs))
        assert loads.max() <= 4.0 / 3.0 * opt_lb + 1e-12
    assert list(P.shard_plan(1, costs)) == [0] * 7


def test_tridiag_eig_matches_scipy(lib):
    rng = np.random.default_rng(3)
    for k in (1, 2, 5, 30, 200):
        d = rng.uniform(1, 10, size=k)
        e = rng.uniform(-2, 2, size=max(k - 1, 0))
        ev, first = P.tridiag_eig(d, e)
        if k == 1:
            assert ev[0] == d[0] and first[0] == 1.0
            continue
        w, V = scipy.linalg.eigh_tridiagonal(d, e)
        order = np.argsort(ev)
        np.testing.assert_allclose(ev[order], w, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(np.abs(first[order]), np.abs(V[0]), rtol=1e-8, atol=1e-10)
        # Gauss quadrature weights sum to 1
        assert np.sum(first ** 2) == pytest.approx(1.0, rel=1e-12)
