"""Device error and edge paths against the C oracle / the reference rules.

* non-finite coordinates -> ValueError through the device flag of the fit
  (replaces LabeledPoint's check, core.py:35-36);
* d = 8: the runtime-d kernel (key order of numpy's einsum for 8-wide
  chunks, ghn_common.cuh key_numpy_order_rt);
* k > 256 (explore.py:86-88 allows any 1 <= k <= n): the exact per-query
  path (csrc/ghn_largek.cu) -- neighbours, QueryStats, vote, mean, median,
  both stop modes, and brute_knn with k = n (every point, sorted).
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ghn():
    import paper_2004_02290_b200 as g

    return g


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_non_finite_raises_value_error(ghn, bad, dtype):
    X = np.random.default_rng(1).random((5000, 3)).astype(dtype)
    X[1234, 1] = bad
    with pytest.raises(ValueError, match="non-finite"):
        ghn.build_arrays(X, np.zeros(5000, np.int32), cells_per_axis=16)
    with pytest.raises(ValueError, match="non-finite"):
        ghn.build_arrays(X, np.zeros(5000, np.int32))          # the max-splits width fit path
    with pytest.raises(ValueError):
        ghn.build(ghn.points_from_arrays(np.where(np.isfinite(X), X, 0.0)[:10], [0] * 10),
                  params=ghn.GridParams(np.zeros(3), np.zeros(3), np.ones(3)))   # widths <= 0


@pytest.mark.parametrize("mode", ["heuristic", "guaranteed"])
@pytest.mark.parametrize("d", [8, 9])
def test_runtime_d_kernel(ghn, mode, d):
    rng = np.random.default_rng(80 + d)
    X = rng.normal(0, 1, (40000, d)) * np.linspace(1, 2, d)     # fp64, off any lattice
    y = rng.integers(0, 5, 40000).astype(np.int32)
    Q = rng.normal(0, 1.1, (1500, d))
    w = np.full(d, 1.5)
    index = ghn.build_arrays(X, y, params=ghn.GridParams(w, X.min(0), np.ones(d, np.int64)))
    ref = oracle.COracle(X, w)
    for k in (1, 7, 40):
        dist, idx, st = ghn.knn_query_batch(index, Q, k, mode)
        keys, ridx, rst = ref.query(Q, k, mode)
        assert np.array_equal(idx.cpu().numpy(), ridx)
        assert np.array_equal(dist.cpu().numpy(), np.sqrt(keys))
        assert np.array_equal(st.cpu().numpy(), rst)
        r = ghn.predict_batch(index, Q, k, mode)
        lab, conf = oracle.classify(keys, ridx, y.astype(np.int64))
        assert np.array_equal(r["label"].cpu().numpy().astype(np.int64), lab)
        assert np.array_equal(r["confidence"].cpu().numpy(), conf)


@pytest.mark.parametrize("mode", ["heuristic", "guaranteed"])
@pytest.mark.parametrize("k", [257, 600])
def test_large_k_exact(ghn, mode, k):
    rng = np.random.default_rng(900 + k)
    X = rng.random((6000, 2)).astype(np.float32)
    y = rng.integers(0, 6, 6000).astype(np.int32)
    yt = (rng.normal(0, 1, 6000)).astype(np.float64)
    Q = np.concatenate([rng.random((40, 2)).astype(np.float32), np.array([[1.7, -0.4]], np.float32)])
    w = np.full(2, 1.0 / 40)
    index = ghn.build_arrays(X, y, params=ghn.GridParams(w, X.min(0), np.full(2, 40)))
    ref = oracle.COracle(X, w)
    dist, idx, st = ghn.knn_query_batch(index, Q, k, mode)
    keys, ridx, rst = ref.query(Q, k, mode)
    assert np.array_equal(idx.cpu().numpy(), ridx)
    assert np.array_equal(dist.cpu().numpy(), np.sqrt(keys))
    assert np.array_equal(st.cpu().numpy(), rst)
    r = ghn.predict_batch(index, Q, k, mode, stats=True)
    lab, conf = oracle.classify(keys, ridx, y.astype(np.int64))
    assert np.array_equal(r["label"].cpu().numpy().astype(np.int64), lab)
    assert np.array_equal(r["confidence"].cpu().numpy(), conf)
    assert np.array_equal(r["stats"].cpu().numpy(), rst)
    it = ghn.build_arrays(X, yt, params=ghn.GridParams(w, X.min(0), np.full(2, 40)))
    m = ghn.predict_batch(it, Q, k, mode, task="regress")["value"].cpu().numpy()
    assert np.array_equal(m, oracle.regress_mean(ridx, yt))
    md = ghn.predict_batch(it, Q, k, mode, task="regress_median")["value"].cpu().numpy()
    assert np.array_equal(md, oracle.regress_median(ridx, yt))


def test_brute_knn_k_equals_n(ghn):
    """SPEC brute_knn example: k = n returns every point sorted by (distance, index)."""
    rng = np.random.default_rng(77)
    X = np.round(rng.random((700, 3)) * 8) / 8            # many exact ties
    pts = ghn.points_from_arrays(X, rng.integers(0, 3, 700))
    bi = ghn.brute_build(pts)
    q = np.array([0.5, 0.5, 0.5])
    got = ghn.brute_knn(bi, q, 700)
    keys = np.array([oracle.key(p, q) for p in X])
    want = np.lexsort((np.arange(700), keys))
    assert [nb.point_index for nb in got] == want.tolist()
    assert [nb.distance for nb in got] == np.sqrt(keys[want]).tolist()
    assert [nb.point_index for nb in ghn.kdtree_knn(ghn.kdtree_build(pts), q, 700)] == want.tolist()


def test_knn_query_k_equals_n(ghn):
    rng = np.random.default_rng(78)
    X = rng.normal(0, 1, (400, 2))
    pts = ghn.points_from_arrays(X, [0] * 400)
    index = ghn.build(pts)
    ref = oracle.COracle(X, index.params.widths)
    for mode in ("heuristic", "guaranteed"):
        nb, st = ghn.knn_query(index, (0.1, -0.2), 400, mode)
        keys, ridx, rst = ref.query(np.array([[0.1, -0.2]]), 400, mode)
        assert [x.point_index for x in nb] == ridx[0].tolist()
        assert (st.layers_visited, st.cells_visited, st.points_scanned) == tuple(rst[0])
