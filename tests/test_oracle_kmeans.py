"""Pins of the row-A0 oracle (oracle/kmeans.py) against things other than itself:
sklearn's Lloyd k-means, brute-force nearest-centre / mean fixed-point conditions, the
construction of the synthetic generator (GIVEN centres), and SPEC.md's medoid example."""
import numpy as np
import pytest

import synth
from oracle import kmeans as KM


def _blobs(seed=0, n_c=5, per=60, d=3, spread=0.3):
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-10, 10, size=(n_c, d))
    lab = np.repeat(np.arange(n_c), per)
    X = centres[lab] + spread * rng.standard_normal((n_c * per, d))
    p = rng.permutation(X.shape[0])
    return X[p], lab[p], centres


def test_forgy_indices_distinct_in_range():
    idx = KM.forgy_indices(7, 50, 50)        # must exhaust all rows without repeats
    assert sorted(idx) == list(range(50))
    idx = KM.forgy_indices(3, 10 ** 6, 2000)
    assert len(set(idx)) == 2000 and min(idx) >= 0 and max(idx) < 10 ** 6


def test_splitmix64_reference_values():
    # splitmix64 seeded with 0: the first outputs of the published generator (Vigna)
    assert KM._splitmix64(0, 0) == 0xE220A8397B1DCDAF
    assert KM._splitmix64(0, 1) == 0x6E789E6AA1B965F4


def test_blobs_recovered_spec_434():
    """well-separated blobs are recovered exactly (init at the true centres)."""
    X, lab, centres = _blobs()
    r = KM.kmeans(X, 5, init_centers=centres, rep_mode=KM.CENTROID)
    assert np.array_equal(r["assign"], lab)
    for j in range(5):
        np.testing.assert_allclose(r["reps"][j], X[lab == j].mean(axis=0), rtol=0, atol=1e-13)


def test_matches_sklearn_lloyd_same_init():
    from sklearn.cluster import KMeans
    rng = np.random.default_rng(5)
    X = rng.standard_normal((400, 4)) * np.array([3.0, 1.0, 2.0, 0.5])
    init = X[KM.forgy_indices(11, 400, 7)]
    r = KM.kmeans(X, 7, init_centers=init, max_iter=300)
    sk = KMeans(n_clusters=7, init=init, n_init=1, max_iter=300, tol=0.0, algorithm="lloyd").fit(X)
    assert np.array_equal(r["assign"], sk.labels_)
    np.testing.assert_allclose(r["centers"], sk.cluster_centers_, rtol=0, atol=1e-12)


def test_lloyd_fixed_point_conditions_brute_force():
    """At convergence every point is at its nearest centre and every centre is its mean."""
    from scipy.spatial.distance import cdist
    rng = np.random.default_rng(9)
    X = rng.uniform(-5, 5, size=(300, 2))
    r = KM.kmeans(X, 6, seed=4, max_iter=500)
    assert r["iters"] < 500
    D = cdist(X, r["centers"], "sqeuclidean")
    np.testing.assert_array_equal(r["assign"], D.argmin(axis=1))
    for j in range(6):
        np.testing.assert_allclose(r["centers"][j], X[r["assign"] == j].mean(axis=0), atol=1e-13)


def test_stable_permutation_and_offsets():
    X, lab, centres = _blobs(seed=2, n_c=4, per=25)
    r = KM.kmeans(X, 4, init_centers=centres)
    perm, off = r["perm"], r["offsets"]
    assert sorted(perm.tolist()) == list(range(X.shape[0]))
    for j in range(4):
        seg = perm[off[j]:off[j + 1]]
        assert np.all(r["assign"][seg] == j)
        assert np.all(np.diff(seg) > 0)               # original order kept inside a cluster


def test_given_grid_centres_reproduce_construction():
    """G-HYPER with the vertices as GIVEN centres: the assignment equals the construction."""
    ds = synth.g_hyper(n_c=12, b=40, d=3, seed=31)
    rng = np.random.default_rng(0)
    p = rng.permutation(ds.n)
    r = KM.kmeans(ds.X[p], 12, init_centers=ds.reps, rep_mode=KM.GIVEN)
    truth = np.repeat(np.arange(12), 40)[p]
    assert np.array_equal(r["assign"], truth)
    assert np.array_equal(r["offsets"], ds.offsets)
    src = p[r["perm"]]                                # construction row of each sorted row
    for j in range(12):
        assert np.array_equal(np.sort(src[40 * j:40 * (j + 1)]), np.arange(40 * j, 40 * (j + 1)))
    np.testing.assert_array_equal(r["reps"], ds.reps)


def test_fixed_point_sum_is_exact_and_order_independent():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((1000, 3)) * 7
    a = rng.integers(0, 5, size=1000)
    s = KM.fixed_point_shift(X)
    assert np.max(np.abs(X)) * 1000 * 2.0 ** s <= 2.0 ** 62
    C1 = KM.update(X, a, np.zeros((5, 3)), s)
    p = rng.permutation(1000)
    C2 = KM.update(X[p], a[p], np.zeros((5, 3)), s)
    assert np.array_equal(C1, C2)
    for j in range(5):
        np.testing.assert_allclose(C1[j], X[a == j].mean(axis=0), rtol=1e-14, atol=1e-14)


def test_medoid_spec_444():
    """the medoid of {-1, 0, 1} is 0 (argmax of the kernel row sums)."""
    X = np.array([[-1.0], [0.0], [1.0]])
    a = np.zeros(3, dtype=np.int64)
    assert KM.medoids(X, a, 1, "rbf", 1.0, 1.0)[0] == 1
    r = KM.kmeans(X, 1, init_centers=[[5.0]], rep_mode=KM.MEDOID, theta=(1.0, 0.1, 1.0))
    np.testing.assert_array_equal(r["reps"], [[0.0]])


def test_empty_cluster_keeps_centre():
    X = np.array([[0.0], [0.1], [0.2]])
    r = KM.kmeans(X, 2, init_centers=[[0.1], [100.0]])
    assert np.all(r["assign"] == 0)
    assert r["centers"][1, 0] == 100.0
    assert list(r["offsets"]) == [0, 3, 3]
