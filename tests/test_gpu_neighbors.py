"""knn_query_batch on the tiled thread kernel (tile2d_nb_kernel + nb_sort_kernel,
ghn_tile2d_thr.cuh): neighbour indices, distances and QueryStats bit-exact
against the C oracle (explore.py:66-137: order by (key, index), distance =
sqrt(key))."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ghn():
    import paper_2004_02290_b200 as g

    return g


@pytest.fixture(scope="module")
def case(ghn):
    from paper_2004_02290_b200 import datagen

    w = datagen.cfg4(n=3_000_000, nq=40_000, seed=71)
    index = ghn.build_arrays(w.X, w.y, cells_per_axis=700)
    ref = oracle.COracle(w.X, np.full(2, 1.0 / 700))
    return w, index, ref


def _check(ghn, index, ref, Q, k, mode, stats):
    dist, idx, st = ghn.knn_query_batch(index, Q, k, mode, stats=stats)
    keys, ridx, rst = ref.query(Q, k, mode)
    assert np.array_equal(idx.cpu().numpy(), ridx), f"k={k} {mode}: indices"
    assert np.array_equal(dist.cpu().numpy(), np.sqrt(keys)), f"k={k} {mode}: distances"
    if stats:
        assert np.array_equal(st.cpu().numpy(), rst), f"k={k} {mode}: QueryStats"
    else:
        assert st is None


@pytest.mark.parametrize("k", [1, 2, 4, 5, 16, 31, 32])
@pytest.mark.parametrize("stats", [False, True])
def test_neighbors_heuristic(ghn, case, k, stats):
    w, index, ref = case
    _check(ghn, index, ref, w.Q, k, "heuristic", stats)


@pytest.mark.parametrize("k", [1, 16])
def test_neighbors_guaranteed(ghn, case, k):
    w, index, ref = case
    _check(ghn, index, ref, w.Q[:15000], k, "guaranteed", True)


def test_neighbors_fp64_queries(ghn, case):
    w, index, ref = case
    Q = np.random.default_rng(72).random((20000, 2))
    _check(ghn, index, ref, Q, 16, "heuristic", False)


def test_neighbors_duplicates_and_outliers(ghn):
    """Duplicate points (equal keys: index order) and queries outside the grid."""
    rng = np.random.default_rng(73)
    base = rng.random((50_000, 2), dtype=np.float32)
    X = np.concatenate([base, base[:20_000], base[:5_000]])
    y = (np.arange(X.shape[0]) % 3).astype(np.int32)
    index = ghn.build_arrays(X, y, cells_per_axis=100)
    ref = oracle.COracle(X, np.full(2, 1.0 / 100))
    Q = np.concatenate([rng.random((8000, 2), dtype=np.float32),
                        (rng.random((200, 2), dtype=np.float32) * 3 - 1).astype(np.float32)])
    for k in (3, 16):
        _check(ghn, index, ref, Q, k, "heuristic", True)


def test_clustered_dense_rows(ghn):
    """Clustered data: dense cells (long clipped rows, tiles of very different
    work), queries from the same mixture.  Neighbours and the fused vote."""
    rng = np.random.default_rng(74)
    n, nq, C = 3_000_000, 300_000, 512
    means = rng.random((12, 2))
    comp = rng.integers(0, 12, n)
    X = np.clip(means[comp] + rng.normal(0, 0.02, (n, 2)), 0, 1).astype(np.float32)
    y = (comp % 4).astype(np.int32)
    Q = np.clip(means[rng.integers(0, 12, nq)] + rng.normal(0, 0.02, (nq, 2)), 0, 1).astype(np.float32)
    index = ghn.build_arrays(X, y, cells_per_axis=C)
    ref = oracle.COracle(X, np.full(2, 1.0 / C))
    sel = np.sort(rng.choice(nq, size=3000, replace=False))
    for k in (1, 16, 32):
        dist, idx, _ = ghn.knn_query_batch(index, Q, k, stats=False)
        keys, ridx, _ = ref.query(Q[sel], k, "heuristic")
        assert np.array_equal(idx.cpu().numpy()[sel], ridx), f"k={k}: indices"
        assert np.array_equal(dist.cpu().numpy()[sel], np.sqrt(keys)), f"k={k}: distances"
    # few queries: the largest tiles (windows of up to 72 rows)
    few = 20000
    for k in (1, 16):
        dist, idx, st = ghn.knn_query_batch(index, Q[:few], k, stats=True)
        keys, ridx, rst = ref.query(Q[:few], k, "heuristic")
        assert np.array_equal(idx.cpu().numpy(), ridx), f"k={k}: indices (few queries)"
        assert np.array_equal(dist.cpu().numpy(), np.sqrt(keys)), f"k={k}: distances (few queries)"
        assert np.array_equal(st.cpu().numpy(), rst), f"k={k}: QueryStats (few queries)"
    for k in (4, 64):
        p = ghn.predict_batch(index, Q, k)
        keys, ridx, _ = ref.query(Q[sel], k, "heuristic")
        lab, conf = oracle.classify(keys, ridx, y.astype(np.int64))
        assert np.array_equal(p["label"].cpu().numpy()[sel].astype(np.int64), lab), f"k={k}: labels"
        assert np.array_equal(p["confidence"].cpu().numpy()[sel], conf), f"k={k}: confidences"
