"""GPU parity of row A0 (nugpr_cluster) against the oracle (oracle/kmeans.py).

Assignments, permutation, offsets, iteration counts and centroids are integer / fixed-point
decisions taken identically on both sides (reading P18) and are compared bit for bit.  Medoids
are chosen by a floating-point argmax over kernel sums whose exp() differs in the last ulp
between libm and CUDA, so the GPU's choice is checked for validity (its score is within 1e-12
relative of the cluster's maximum) instead."""
import numpy as np
import pytest

import synth
from oracle import kmeans as KM

pytestmark = pytest.mark.gpu


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


def _check_against_oracle(P, ctx, X, n_c, y=None, **kw):
    import torch
    r = P.cluster(ctx, torch.tensor(X, device="cuda"), n_c, y=None if y is None else torch.tensor(y, device="cuda"), **kw)
    okw = dict(kw)
    okw.pop("kernel", None)
    o = KM.kmeans(X, n_c, init_centers=kw.get("init_centers"), seed=kw.get("seed", 0),
                  max_iter=kw.get("max_iter", 100), rep_mode=KM.CENTROID)
    perm = r["perm"].cpu().numpy()
    assert r["iters"] == o["iters"]
    np.testing.assert_array_equal(r["offsets"], o["offsets"])
    np.testing.assert_array_equal(perm, o["perm"])
    np.testing.assert_array_equal(r["X_sorted"].cpu().numpy(), X[o["perm"]])
    if y is not None:
        np.testing.assert_array_equal(r["y_sorted"].cpu().numpy(), y[o["perm"]])
    return r, o


def test_kmeans_C4_shaped_forgy_bit_exact(P, ctx):
    """C4 (G-REAL, n=32,000 train, d=8, n_c=20 uneven clusters): Forgy init from the seed."""
    g = synth.g_real(N=40000, d=8, seed=104)
    r, o = _check_against_oracle(P, ctx, g["X"], 20, y=g["y"], seed=5, rep_mode="centroid")
    np.testing.assert_array_equal(r["reps"].cpu().numpy(), o["centers"])
    sizes = np.diff(r["offsets"])
    assert sizes.min() > 0 and sizes.max() > 2 * sizes.min()        # uneven, as C4 requires


@pytest.mark.parametrize("n,d,n_c,seed", [(1, 1, 1, 0), (7, 3, 7, 1), (1000, 2, 1, 2), (5000, 32, 33, 3),
                                          (777, 5, 9, 4)])
def test_kmeans_edge_shapes(P, ctx, n, d, n_c, seed):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d)) * 3
    r, o = _check_against_oracle(P, ctx, X, n_c, seed=seed + 10, rep_mode="centroid")
    np.testing.assert_array_equal(r["reps"].cpu().numpy(), o["centers"])


def test_kmeans_given_centres_full_size_C5(P, ctx):
    """C5 size (n=1,000,000, d=4, n_c=2000): GIVEN grid vertices, one update step.  The
    first assignment is the construction (pinned by the generator), so the oracle's update is
    cheap at full size; the final assignment is sampled and checked by brute force."""
    import torch
    ds = synth.make_config("C5")
    rng = np.random.default_rng(0)
    p = rng.permutation(ds.n)
    Xp = ds.X[p]
    r = P.cluster(ctx, torch.tensor(Xp, device="cuda"), ds.n_c, init_centers=ds.reps, max_iter=1,
                  rep_mode="centroid")
    truth = np.repeat(np.arange(ds.n_c), 500)[p]
    s = KM.fixed_point_shift(Xp)
    C1 = KM.update(Xp, truth, ds.reps.copy(), s)
    np.testing.assert_array_equal(r["reps"].cpu().numpy(), C1)
    np.testing.assert_array_equal(r["offsets"], ds.offsets)          # clusters never overlap
    perm = r["perm"].cpu().numpy()
    np.testing.assert_array_equal(truth[perm], np.repeat(np.arange(ds.n_c), 500))
    assert np.all(np.diff(perm.reshape(ds.n_c, 500), axis=1) > 0)     # stable inside a cluster
    samp = rng.choice(ds.n, 2000, replace=False)
    lab = np.repeat(np.arange(ds.n_c), 500)
    inv = np.empty(ds.n, dtype=np.int64)
    inv[perm] = np.arange(ds.n)
    np.testing.assert_array_equal(lab[inv[samp]], KM.assign(Xp[samp], C1))


def test_medoid_representatives_valid(P, ctx):
    import torch
    g = synth.g_real(N=6000, d=8, seed=7)
    th = (3.0, 0.16, 1.5)
    r = P.cluster(ctx, torch.tensor(g["X"], device="cuda"), 6, seed=3, rep_mode="medoid", kernel="matern52",
                  theta=th)
    o = KM.kmeans(g["X"], 6, seed=3, rep_mode=KM.CENTROID)
    reps = r["reps"].cpu().numpy()
    for j, (idx, sc) in enumerate(KM.medoid_scores(g["X"], o["assign"], 6, "matern52", th[0], th[2])):
        hit = np.nonzero(np.all(g["X"][idx] == reps[j], axis=1))[0]
        assert hit.size >= 1, "medoid is not a member of its cluster"
        assert sc[hit[0]] >= sc.max() * (1 - 1e-12)


def test_given_mode_returns_initial_centres(P, ctx):
    import torch
    ds = synth.g_hyper(n_c=12, b=40, d=3, seed=31)
    r = P.cluster(ctx, torch.tensor(ds.X, device="cuda"), 12, init_centers=ds.reps, rep_mode="given")
    np.testing.assert_array_equal(r["reps"].cpu().numpy(), ds.reps)
    np.testing.assert_array_equal(r["perm"].cpu().numpy(), np.arange(ds.n))


def test_empty_cluster_is_shape_error(P, ctx):
    import torch
    X = np.array([[0.0], [0.1], [0.2]])
    with pytest.raises(P.NugprError) as e:
        P.cluster(ctx, torch.tensor(X, device="cuda"), 2, init_centers=np.array([[0.1], [100.0]]))
    assert e.value.name == "SHAPE"


def test_host_input_equals_device_input(P, ctx):
    import torch
    rng = np.random.default_rng(1)
    X = rng.standard_normal((3000, 4))
    a = P.cluster(ctx, X, 10, seed=2)
    b = P.cluster(ctx, torch.tensor(X, device="cuda"), 10, seed=2)
    assert torch.equal(a["perm"], b["perm"]) and torch.equal(a["reps"], b["reps"])
