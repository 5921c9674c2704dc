"""Pins for the CPU oracle (oracle/): each check ties the oracle to something
other than itself — values printed in SPEC/PAPER worked examples, hand-derived
fractions, exact integer arithmetic, scipy/sklearn library routines, and
invariants that the mathematics fixes.  A plausible mistake anywhere in
O1-O4 (dropped term, wrong sign/index, transposed operand, wrong tie-break,
self not excluded, wrong LOF ratio) fails at least one of these.
"""
import json
import os
import time
from fractions import Fraction

import numpy as np
import pytest

import datagen
import oracle


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- O1 distance
def test_cdist_345(golden_dir):
    g = _load(golden_dir, "cdist_345.json")
    D = oracle.cdist64(np.array(g["X"], np.float32))
    assert D.tolist() == g["D64"]


def test_d64_integer_inputs_exact():
    # |x| <= 2^20, d <= 64: every partial sum < 2^53, so D64 is exact and must
    # equal Python-integer brute force bit for bit.
    rng = np.random.default_rng(3)
    for d in (1, 3, 10, 64):
        X = rng.integers(-(2 ** 20), 2 ** 20, (12, d)).astype(np.float32)
        Xi = X.astype(np.int64)
        for i in range(12):
            for j in range(12):
                exact = sum(int(Xi[i, c] - Xi[j, c]) ** 2 for c in range(d))
                assert oracle.d64(X[i], X[j]) == float(exact)


def test_d64_symmetry_and_pow2_scaling_bitwise():
    X = datagen.gaussian_mixture(40, 17, seed=5)
    D = oracle.cdist64(X)
    assert np.array_equal(D, D.T)                 # RN is sign-symmetric
    assert np.all(np.diag(D) == 0.0)
    D2 = oracle.cdist64(2.0 * X)                  # exact fp32 scaling
    assert np.array_equal(D2, 4.0 * D)


def test_d64_vs_scipy_library():
    from scipy.spatial.distance import cdist
    X = datagen.gaussian_mixture(60, 33, seed=7).astype(np.float64)
    ref = cdist(X, X, "sqeuclidean")
    D = oracle.cdist64(X.astype(np.float32))
    off = ~np.eye(60, dtype=bool)
    assert np.allclose(D[off], ref[off], rtol=1e-12, atol=0)


def test_d64_sequential_order_not_pairwise():
    # O1 fixes the summation order: ascending c, sequential.  A value whose
    # sequential and reversed sums differ in fp64 must match the sequential one.
    # squares [1, 2^-54 x4]: sequential absorbs each 2^-54 (below half an ulp
    # of 1) -> exactly 1; any order that adds the small terms first gives 1+2^-52.
    a = np.array([1.0] + [2.0 ** -27] * 4, np.float32)
    b = np.zeros(5, np.float32)
    assert oracle.d64(a, b) == 1.0
    assert oracle.d64(a[::-1].copy(), b) == 1.0 + 2.0 ** -52


# ------------------------------------------------------------ O2 neighbours
def test_knn_golden(golden_dir):
    g = _load(golden_dir, "knn_examples.json")
    for case in g["cases"]:
        X = np.array(case["X"], np.float32)
        idx, dd = oracle.knn(X, case["k"], rows=case.get("rows"))
        assert idx.tolist() == case["idx"]
        assert dd.tolist() == case["d64"]


def test_knn_k_equals_n_minus_1_is_every_other_index():
    X = datagen.gaussian_mixture(25, 4, seed=2)
    idx, _ = oracle.knn(X, 24)
    for i in range(25):
        assert sorted(idx[i].tolist()) == [j for j in range(25) if j != i]


def test_knn_lattice_ties_vs_exact_integer_stable_sort():
    # Integer lattice data: massive exact ties.  Independent brute force with
    # Python integers + a stable argsort gives the (D, index) order.
    X = datagen.lattice(120, 3, seed=11, extent=2)
    Xi = X.astype(np.int64)
    k = 15
    idx, dd = oracle.knn(X, k)
    for i in range(120):
        dist = [(int(((Xi[i] - Xi[j]) ** 2).sum()), j) for j in range(120) if j != i]
        dist.sort()
        assert idx[i].tolist() == [j for _, j in dist[:k]]
        assert dd[i].tolist() == [float(v) for v, _ in dist[:k]]


def test_knn_vs_sklearn_bruteforce():
    from sklearn.neighbors import NearestNeighbors
    X = datagen.gaussian_mixture(400, 8, seed=1)
    k = 10
    idx, dd = oracle.knn(X, k)
    nn = NearestNeighbors(n_neighbors=k + 1, algorithm="brute").fit(X.astype(np.float64))
    dist_s, idx_s = nn.kneighbors(X.astype(np.float64))
    assert np.array_equal(idx_s[:, 0], np.arange(400))        # self first in sklearn
    assert np.array_equal(idx, idx_s[:, 1:])
    assert np.allclose(np.sqrt(dd), dist_s[:, 1:], rtol=1e-9)


def test_knn_self_excluded_even_with_duplicates():
    X = np.array([[1.0, 1.0], [1.0, 1.0], [1.0, 1.0], [4.0, 5.0]], np.float32)
    idx, dd = oracle.knn(X, 2)
    assert idx.tolist() == [[1, 2], [0, 2], [0, 1], [0, 1]]
    assert dd[:3].tolist() == [[0.0, 0.0]] * 3
    assert dd[3].tolist() == [25.0, 25.0]


def test_knn_rows_subset_equals_full():
    X = datagen.gaussian_mixture(300, 6, seed=9)
    i_all, d_all = oracle.knn(X, 7)
    rows = np.array([299, 0, 150, 17])
    i_sub, d_sub = oracle.knn(X, 7, rows=rows)
    assert np.array_equal(i_sub, i_all[rows]) and np.array_equal(d_sub, d_all[rows])


def test_knn_query_matches_selfjoin_on_distinct_rows():
    X = datagen.gaussian_mixture(200, 5, seed=4)
    qi, qd = oracle.knn_query(X[:30], X, 6)
    assert np.array_equal(qi[:, 0], np.arange(30)) and np.all(qd[:, 0] == 0)
    si, sd = oracle.knn(X, 5, rows=np.arange(30))
    assert np.array_equal(qi[:, 1:], si) and np.array_equal(qd[:, 1:], sd)


def test_knn_rejects_bad_k():
    X = datagen.gaussian_mixture(5, 2, seed=0)
    for k in (0, 5, 6):
        with pytest.raises(ValueError):
            oracle.knn(X, k)


# ---------------------------------------------------------------- O3 scores
def test_scores_golden(golden_dir):
    g = _load(golden_dir, "scores_examples.json")
    for case in g["cases"]:
        X = np.array(case["X"], np.float32)
        _, dd = oracle.knn(X, case["k"])
        kth, mean = oracle.scores(dd)
        assert kth.tolist() == case["kth"]
        assert mean.tolist() == case["mean"]


def test_score_monotone_when_point_moves_outward():
    X = datagen.gaussian_mixture(200, 4, seed=8)
    k = 5
    c = X.mean(0)
    prev = None
    for t in (1.0, 1.5, 3.0, 6.0):
        Y = X.copy()
        Y[0] = c + t * (X[0] - c) * 4.0
        _, dd = oracle.knn(Y, k, rows=[0])
        kth, _ = oracle.scores(dd)
        if prev is not None:
            assert kth[0] > prev
        prev = kth[0]


def test_outliers_score_higher_auc():
    from sklearn.metrics import roc_auc_score
    X, lab = datagen.gaussian_mixture(1500, 10, seed=3, return_labels=True)
    _, dd = oracle.knn(X, 10)
    kth, mean = oracle.scores(dd)
    assert roc_auc_score(lab, kth) > 0.9 and roc_auc_score(lab, mean) > 0.9


# ------------------------------------------------------------------- O4 LOF
def test_lof_golden_exact_fractions(golden_dir):
    g = _load(golden_dir, "lof_line.json")
    X = np.array(g["X"], np.float32)
    k = g["k"]
    idx, dd = oracle.knn(X, k)
    assert idx.tolist() == g["idx"]
    lrd, lof = oracle.lof_from_knn(idx, dd)
    for got, (p, q) in zip(lrd, g["lrd"]):
        assert abs(Fraction(got) - Fraction(p, q)) <= Fraction(p, q) * Fraction(1, 2 ** 50)
    for got, (p, q) in zip(lof, g["lof"]):
        assert abs(Fraction(got) - Fraction(p, q)) <= Fraction(p, q) * Fraction(1, 2 ** 49)


def test_lof_vs_sklearn():
    from sklearn.neighbors import LocalOutlierFactor
    X = datagen.gaussian_mixture(600, 6, seed=12)
    k = 20
    idx, dd = oracle.knn(X, k)
    _, lof = oracle.lof_from_knn(idx, dd)
    clf = LocalOutlierFactor(n_neighbors=k, algorithm="brute").fit(X.astype(np.float64))
    ref = -clf.negative_outlier_factor_
    assert np.allclose(lof, ref, rtol=1e-8)


def test_lof_all_identical_is_one():
    X = np.ones((10, 3), np.float32)
    idx, dd = oracle.knn(X, 3)
    lrd, lof = oracle.lof_from_knn(idx, dd)
    assert np.all(np.isinf(lrd)) and np.all(lof == 1.0)


def test_lof_isolated_point_is_argmax():
    X = datagen.gaussian_mixture(300, 3, seed=6, contamination=0.0)
    X[123] = X.max(0) * 5.0
    idx, dd = oracle.knn(X, 10)
    _, lof = oracle.lof_from_knn(idx, dd)
    assert int(np.argmax(lof)) == 123 and lof[123] > 2.0


def test_lof_grid_interior_near_one():
    g = np.stack(np.meshgrid(np.arange(12), np.arange(12)), -1).reshape(-1, 2).astype(np.float32)
    g = g + np.random.default_rng(0).uniform(-0.01, 0.01, g.shape).astype(np.float32)
    idx, dd = oracle.knn(g, 4)
    _, lof = oracle.lof_from_knn(idx, dd)
    interior = [(r * 12 + c) for r in range(2, 10) for c in range(2, 10)]
    assert np.all(np.abs(lof[interior] - 1.0) < 0.2)


def test_lof_pow2_scaling_bitwise():
    X = datagen.gaussian_mixture(300, 5, seed=13)
    a = oracle.lof_from_knn(*oracle.knn(X, 8))
    b = oracle.lof_from_knn(*oracle.knn(2.0 * X, 8))
    assert np.array_equal(a[1], b[1]) and np.array_equal(2.0 * b[0], a[0])


def test_lof_rows_closure_equals_full_table():
    X = datagen.gaussian_mixture(500, 4, seed=14)
    k = 6
    idx, dd = oracle.knn(X, k)
    lrd, lof = oracle.lof_from_knn(idx, dd)
    rows = np.array([0, 77, 499, 250])
    r = oracle.lof_rows(X, k, rows)
    assert np.array_equal(r["idx"], idx[rows])
    assert np.array_equal(r["lrd"], lrd[rows]) and np.array_equal(r["lof"], lof[rows])


# --------------------------------------------------------- configs[0] (C1)
def test_c1_oracle_under_one_second():
    # BASELINE.json configs[0]: n=1000, d=10, k=10, "CPU oracle finishes in <1 s".
    X = datagen.gaussian_mixture(1000, 10, seed=0)
    t = time.perf_counter()
    idx, dd = oracle.knn(X, 10)
    oracle.scores(dd)
    oracle.lof_from_knn(idx, dd)
    assert time.perf_counter() - t < 1.0


# ------------------------------------------------------------------- O5 NWR
def _nwr_lists(X, phi, rows=None):
    counts, ptr, cols = oracle.nwr(X, phi, rows=rows)
    return [cols[ptr[r]:ptr[r + 1]].tolist() for r in range(counts.size)]


def test_nwr_golden_boundary_inclusive(golden_dir):
    g = _load(golden_dir, "nwr_line.json")
    X = np.array(g["X"], np.float32)
    for case in g["cases"]:
        assert _nwr_lists(X, case["phi"]) == case["neighbours"], case["phi"]


def test_nwr_symmetric_and_monotone_in_phi():
    X = datagen.gaussian_mixture(300, 6, seed=21)
    D = oracle.cdist64(X[:60])
    phi = float(np.median(D))
    lists = _nwr_lists(X[:60], phi)
    A = np.zeros((60, 60), bool)
    for i, l in enumerate(lists):
        A[i, l] = True
    assert np.array_equal(A, A.T)                  # D64 is bitwise symmetric
    assert not A.diagonal().any()                  # self excluded
    small = _nwr_lists(X[:60], phi / 2)
    assert all(set(s) <= set(b) for s, b in zip(small, lists))


def test_nwr_exact_integers_vs_python_ints():
    X = datagen.lattice(400, 5, seed=7, extent=3)  # massive exact ties
    Xi = X.astype(np.int64)
    phi = 6.0
    want = []
    for i in range(400):
        d2 = ((Xi - Xi[i]) ** 2).sum(1)            # exact integers
        want.append([j for j in range(400) if j != i and d2[j] <= 6])
    assert _nwr_lists(X, phi) == want


def test_nwr_contains_knn_at_kth_distance():
    X = datagen.gaussian_mixture(500, 8, seed=5)
    k = 7
    idx, dd = oracle.knn(X, k)
    for i in (0, 17, 250, 499):
        got = _nwr_lists(X, float(dd[i, k - 1]), rows=[i])[0]
        assert set(idx[i].tolist()) <= set(got) and len(got) >= k
        below = _nwr_lists(X, float(np.nextafter(dd[i, k - 1], -np.inf)), rows=[i])[0]
        assert len(below) < k


def test_nwr_vs_scipy_away_from_boundary():
    from scipy.spatial.distance import cdist
    X = datagen.gaussian_mixture(400, 12, seed=9)
    D = cdist(X.astype(np.float64), X.astype(np.float64), "sqeuclidean")
    phi = float(np.quantile(D, 0.05))
    lists = _nwr_lists(X, phi)
    for i in range(0, 400, 7):
        near = np.abs(D[i] - phi) <= 1e-9 * phi     # library rounding differs only here
        want = set(np.nonzero((D[i] <= phi) & ~near)[0].tolist()) - {i}
        got = set(lists[i])
        assert want <= got and got - want <= set(np.nonzero(near)[0].tolist())


# ---------------------------------------------------------- O6 ABOD, O7 kNN_CLF
def test_abod_golden_row0(golden_dir):
    g = _load(golden_dir, "abod_clf_examples.json")
    X = np.array(g["abod_X"], np.float32)
    idx, _ = oracle.knn(X, g["abod_k"])
    assert idx[0].tolist() == [1, 2, 3]
    s = oracle.abod_from_knn(X, idx)
    assert s[0] == np.float32(g["abod_row0"])


def test_abod_golden_weighted_factor_not_cosine(golden_dir):
    # non-unit neighbour vectors: the distance-weighted factor (-2/81) and the
    # plain-cosine reading (-2/9) differ; the oracle must give the former
    g = _load(golden_dir, "abod_clf_examples.json")
    X = np.array(g["abod_weighted_X"], np.float32)
    idx, _ = oracle.knn(X, g["abod_weighted_k"])
    assert list(idx[0]) == [1, 2, 3]
    s = oracle.abod_from_knn(X, idx)
    assert s[0] == np.float32(g["abod_weighted_row0"])
    assert s[0] != np.float32(g["abod_cosine_reading_row0"])


def test_abod_k2_is_zero_and_duplicates_skipped():
    X = datagen.gaussian_mixture(50, 4, seed=3)
    idx, _ = oracle.knn(X, 2)
    assert (oracle.abod_from_knn(X, idx) == 0).all()          # single pair: variance 0
    Xd = np.vstack([X[:1], X[:1], X[:1], X[:1]])                # all coincident: no pairs
    idx, _ = oracle.knn(Xd, 3)
    assert (oracle.abod_from_knn(Xd, idx) == 0).all()


def test_abod_vs_numpy_formula_and_outlier_argmax():
    X = datagen.gaussian_mixture(300, 5, seed=8)
    X = np.vstack([X, X.mean(0, keepdims=True) + 60.0]).astype(np.float32)  # far isolated point
    k = 8
    idx, _ = oracle.knn(X, k)
    s = oracle.abod_from_knn(X, idx)
    # independent vectorised formula (library float64 ops; tolerance for summation order)
    for i in (0, 37, 300):
        V = X[idx[i]].astype(np.float64) - X[i].astype(np.float64)
        q = (V * V).sum(1)
        W = (V @ V.T) / np.outer(q, q)
        w = W[np.triu_indices(k, 1)]
        assert abs(float(s[i]) - (-np.var(w))) <= 1e-6 * max(1e-30, np.var(w)) + 1e-30
    assert int(np.argmax(s)) == 300


def test_abod_detects_uniform_outliers():
    from sklearn.metrics import roc_auc_score
    X, lab = datagen.gaussian_mixture(3000, 16, seed=2, return_labels=True)
    idx, _ = oracle.knn(X, 10)
    assert roc_auc_score(lab, oracle.abod_from_knn(X, idx)) > 0.9


def test_knn_classify_golden_and_vs_sklearn():
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "abod_clf_examples.json")))
    for labs, want in zip(g["clf_labels_of_neighbours"], g["clf_pred"]):
        idx = np.arange(len(labs))[None, :]
        assert int(oracle.knn_classify(idx, np.array(labs))[0]) == want
    from sklearn.neighbors import KNeighborsClassifier
    rng = np.random.default_rng(0)
    Xtr = np.vstack([rng.normal(0, 1, (200, 3)), rng.normal(3, 1, (200, 3))]).astype(np.float32)
    ytr = np.repeat([0, 1], 200)
    Xte = rng.normal(1.5, 1.5, (100, 3)).astype(np.float32)
    idx, _ = oracle.knn_query(Xte, Xtr, 5)       # odd k, 2 classes: no vote ties
    ref = KNeighborsClassifier(5, algorithm="brute").fit(Xtr, ytr).predict(Xte)
    assert np.array_equal(oracle.knn_classify(idx, ytr), ref)
