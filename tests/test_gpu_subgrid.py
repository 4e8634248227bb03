"""Nested grids of overfull cells and lower-bound pruning in the generic
kernel (csrc/ghn_subgrid.cu, ghn_query_impl.cuh) against the C oracle.

Both change which candidates the device evaluates, never the answer:
neighbour indices, distances, QueryStats, labels and confidences stay
bit-exact with the reference algorithm (explore.py:104-130) on skewed data
where one cell holds most of the points (cfg3's shape),
exact duplicates inside a fat cell, a fat cell of identical points, fp64
indexes, both stop modes and all three metrics.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ghn():
    import paper_2004_02290_b200 as g

    return g


def _lognormal(n, nq, seed, d=4):
    rng = np.random.default_rng(seed)
    raw = rng.lognormal(0.0, 1.0, (n, d))
    lo, hi = raw.min(0), raw.max(0)
    X = ((raw - lo) / (hi - lo)).astype(np.float32)
    nd = nq * 9 // 10
    qd = ((rng.lognormal(0.0, 1.0, (nd, d)) - lo) / (hi - lo)).astype(np.float32)
    qu = rng.random((nq - nd, d), dtype=np.float32)
    y = np.floor(10.0 * np.modf(1000.0 * X[:, 0].astype(np.float64))[0]).astype(np.int32)
    return X, y, np.concatenate([qd, qu])


def _check(ghn, index, ref, y, Q, k, mode, metric="euclidean"):
    dist, idx, stats = ghn.knn_query_batch(index, Q, k, mode)
    keys, ridx, rstats = ref.query(Q, k, mode)
    bad = np.flatnonzero((idx.cpu().numpy() != ridx).any(axis=1))
    assert bad.size == 0, f"{bad.size} neighbour-set mismatches, first {bad[:5]}"
    exp = np.sqrt(keys) if metric == "euclidean" else keys
    assert np.array_equal(dist.cpu().numpy(), exp)
    assert np.array_equal(stats.cpu().numpy(), rstats)
    r = ghn.predict_batch(index, Q, k, mode, task="classify")          # no stats: whole-shell skips
    lab, conf = oracle.classify(keys, ridx, np.asarray(y, dtype=np.int64), metric)
    assert np.array_equal(r["label"].cpu().numpy().astype(np.int64), lab)
    assert np.array_equal(r["confidence"].cpu().numpy(), conf)


@pytest.mark.parametrize("mode", ["heuristic", "guaranteed"])
def test_cfg3_shaped_fat_cells(ghn, mode):
    X, y, Q = _lognormal(2_000_000, 3000, 31)
    w = np.full(4, 1.0 / 64)
    index = ghn.build_arrays(X, y, params=ghn.GridParams(w, X.min(0), np.full(4, 64)))
    assert index.n_subgrids >= 1
    ref = oracle.COracle(X, w)
    order, _, starts, _, _ = ref.export()
    assert np.array_equal(index.order, order)          # the CSR itself is untouched
    for k in (1, 32, 100):
        _check(ghn, index, ref, y, Q, k, mode)


@pytest.mark.parametrize("metric", ["manhattan", "chebyshev"])
def test_fat_cells_other_metrics(ghn, metric):
    X, y, Q = _lognormal(600_000, 1500, 32, d=3)
    w = np.full(3, 1.0 / 32)
    index = ghn.build_arrays(X, y, params=ghn.GridParams(w, X.min(0), np.full(3, 32)), metric=metric)
    assert index.n_subgrids >= 1
    ref = oracle.COracle(X, w, metric=metric)
    for mode in ("heuristic", "guaranteed"):
        _check(ghn, index, ref, y, Q, 16, mode, metric)


def test_fat_cell_duplicates_and_identical_points(ghn):
    """A fat cell of many exact duplicates (ties broken by index) next to a
    fat cell whose points are all identical (zero-extent sub-grid)."""
    rng = np.random.default_rng(33)
    base = rng.random((3000, 2), dtype=np.float32) * np.float32(0.1)
    X = np.concatenate([np.repeat(base, 4, axis=0),                       # 12k points, 4x duplicates
                        np.full((5000, 2), 0.55, dtype=np.float32),         # 5k identical points
                        rng.random((20000, 2), dtype=np.float32)])
    X = X[rng.permutation(X.shape[0])]
    y = rng.integers(0, 5, X.shape[0]).astype(np.int32)
    w = np.full(2, 1.0 / 8)
    index = ghn.build_arrays(X, y, params=ghn.GridParams(w, X.min(0), np.full(2, 8)))
    assert index.n_subgrids >= 2
    ref = oracle.COracle(X, w)
    Q = np.concatenate([base[:500], np.full((10, 2), 0.55, np.float32), rng.random((500, 2), dtype=np.float32)])
    for k in (1, 7, 64, 200):
        for mode in ("heuristic", "guaranteed"):
            _check(ghn, index, ref, y, Q, k, mode)


def test_fat_cells_fp64_index(ghn):
    X, y, Q = _lognormal(300_000, 800, 34, d=3)
    X64 = X.astype(np.float64) * (1 + 1e-9)       # off the fp32 lattice
    w = np.full(3, 1.0 / 24)                       # not a power of two
    index = ghn.build_arrays(X64, y, params=ghn.GridParams(w, X64.min(0), np.full(3, 24)))
    assert index.n_subgrids >= 1
    ref = oracle.COracle(X64, w)
    _check(ghn, index, ref, y, Q.astype(np.float64), 20, "heuristic")


@pytest.mark.parametrize("cfg", [1, 2])
def test_pruned_generic_kernel_cfg_shapes(ghn, cfg):
    """cfg1 (3-D GMM, k=10 vote) and cfg2 (6-D, k=16 mean) samples through
    the pruned generic kernel, with and without QueryStats."""
    from paper_2004_02290_b200 import datagen

    w = datagen.make(cfg, n=400_000 if cfg == 1 else 1_000_000, nq=2000)
    index = ghn.build_arrays(w.X, w.y, cells_per_axis=w.cells_per_axis)
    ref = oracle.COracle(w.X, w.widths)
    keys, idx, stats = ref.query(w.Q, w.k, "heuristic")
    task = "classify" if w.task == "classify" else "regress"
    r0 = ghn.predict_batch(index, w.Q, w.k, task=task)
    r1 = ghn.predict_batch(index, w.Q, w.k, task=task, stats=True)
    assert np.array_equal(r1["stats"].cpu().numpy(), stats)
    if task == "classify":
        lab, conf = oracle.classify(keys, idx, np.asarray(w.y, dtype=np.int64))
        for r in (r0, r1):
            assert np.array_equal(r["label"].cpu().numpy().astype(np.int64), lab)
            assert np.array_equal(r["confidence"].cpu().numpy(), conf)
    else:
        val = oracle.regress_mean(idx, np.asarray(w.y, dtype=np.float64))
        for r in (r0, r1):
            assert np.array_equal(r["value"].cpu().numpy(), val)
