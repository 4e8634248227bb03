"""The thread-per-query tiled kernel (tile2d_thr_kernel, ghn_tile2d_thr.cuh)
in the instantiation the benchmark times -- no QueryStats -- against the C
oracle: every register-list capacity (k <= 32), the bucket select (k > 32,
and forced for small k via GHN_TT_LISTMAX), both stop modes, fp32 and fp64
queries, 2 / 4 / 8 label codes.  Labels and confidences bit-exact."""
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
    """cfg4 recipe at 3M points on a 700 x 700 grid (~6 points per cell, as
    cfg4), 40k queries, quadrant labels."""
    from paper_2004_02290_b200 import datagen

    w = datagen.cfg4(n=3_000_000, nq=40_000, seed=61)
    index = ghn.build_arrays(w.X, w.y, cells_per_axis=700)
    ref = oracle.COracle(w.X, np.full(2, 1.0 / 700))
    return w, index, ref


def _check(ghn, index, ref, y, Q, k, mode):
    r = ghn.predict_batch(index, Q, k, mode)   # no stats: the benchmarked kernels
    keys, idx, _ = ref.query(Q, k, mode)
    lab, conf = oracle.classify(keys, idx, np.asarray(y, dtype=np.int64))
    got = r["label"].cpu().numpy().astype(np.int64)
    bad = np.flatnonzero(got != lab)
    assert bad.size == 0, f"k={k} {mode}: {bad.size} label mismatches, first {bad[:5]}"
    assert np.array_equal(r["confidence"].cpu().numpy(), conf), f"k={k} {mode}: confidence"


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 8, 12, 16, 17, 31, 32, 33, 48, 64, 100])
def test_heuristic_no_stats(ghn, case, k):
    w, index, ref = case
    _check(ghn, index, ref, w.y, w.Q, k, "heuristic")


@pytest.mark.parametrize("k", [1, 4, 16, 64])
def test_guaranteed_no_stats(ghn, case, k):
    w, index, ref = case
    _check(ghn, index, ref, w.y, w.Q[:15000], k, "guaranteed")


@pytest.mark.parametrize("k", [4, 16, 64])
def test_fp64_queries(ghn, case, k):
    """fp64 query coordinates (not on the fp32 lattice): the bucket select's
    fp32 prefilter is off, keys exact from fp64."""
    w, index, ref = case
    rng = np.random.default_rng(62)
    Q = rng.random((20000, 2))
    _check(ghn, index, ref, w.y, Q, k, "heuristic")


@pytest.mark.parametrize("k", [1, 4, 9, 16, 32])
@pytest.mark.skipif("not __import__('paper_2004_02290_b200._lib', fromlist=['x']).tuning_build()",
                    reason="GHN_TT_LISTMAX is a knob of the -DGHN_TUNING_KNOBS build only")
def test_bucket_select_for_small_k(ghn, case, k, monkeypatch):
    """The bucket select is exact for every k, not only the k > 32 it serves."""
    monkeypatch.setenv("GHN_TT_LISTMAX", "0")
    w, index, ref = case
    _check(ghn, index, ref, w.y, w.Q[:20000], k, "heuristic")


@pytest.mark.parametrize("k", [40, 64, 100])
@pytest.mark.parametrize("mode", ["heuristic", "guaranteed"])
@pytest.mark.skipif("not __import__('paper_2004_02290_b200._lib', fromlist=['x']).tuning_build()",
                    reason="GHN_SB_RECAP is a knob of the -DGHN_TUNING_KNOBS build only")
def test_reselect_over_255_candidates(ghn, case, k, mode, monkeypatch):
    """Re-selects over more than 255 candidates (GHN_SB_RECAP raised): the
    byte histogram may carry between buckets; the decoded-total check must
    send exactly those queries to the generic kernel, the rest stay exact."""
    monkeypatch.setenv("GHN_SB_RECAP", "4095")
    w, index, ref = case
    _check(ghn, index, ref, w.y, w.Q[:20000], k, mode)


@pytest.mark.parametrize("n_labels", [2, 8])
@pytest.mark.parametrize("k", [1, 16, 64])
def test_label_codes_2_and_8(ghn, n_labels, k):
    """Label-code widths 1 and 3 bits in the packed keys (4 is the case fixture)."""
    rng = np.random.default_rng(900 + n_labels)
    X = rng.random((1_500_000, 2), dtype=np.float32)
    y = rng.integers(0, n_labels, X.shape[0]).astype(np.int32)
    Q = rng.random((20_000, 2), dtype=np.float32)
    index = ghn.build_arrays(X, y, cells_per_axis=500)
    ref = oracle.COracle(X, np.full(2, 1.0 / 500))
    _check(ghn, index, ref, y, Q, k, "heuristic")


@pytest.mark.parametrize("k", [1, 4, 16, 64, 200])
@pytest.mark.parametrize("n_labels", [1, 8])
def test_sparse_small_sets(ghn, k, n_labels):
    """Few points over many cells (most queries need far layers or fall back),
    a single class, k close to n: still exact."""
    rng = np.random.default_rng(31 + k + n_labels)
    X = rng.random((600, 2), dtype=np.float32)
    y = rng.integers(0, n_labels, X.shape[0]).astype(np.int32)
    Q = rng.random((6000, 2), dtype=np.float32)
    index = ghn.build_arrays(X, y, cells_per_axis=64)
    ref = oracle.COracle(X, np.full(2, 1.0 / 64))
    _check(ghn, index, ref, y, Q, k, "heuristic")
    _check(ghn, index, ref, y, Q[:2000], k, "guaranteed")


def test_heavy_duplicates_small_k(ghn):
    """Exact duplicate points (equal keys) inside the lists and at the k-th
    boundary for the register-list and skip-ahead paths."""
    rng = np.random.default_rng(77)
    X = rng.random((300_000, 2), dtype=np.float32)
    X[::5] = X[1::5]                       # every point has a twin
    y = rng.integers(0, 4, X.shape[0]).astype(np.int32)
    Q = np.concatenate([rng.random((20_000, 2), dtype=np.float32), X[:5000]])
    index = ghn.build_arrays(X, y, cells_per_axis=220)
    ref = oracle.COracle(X, np.full(2, 1.0 / 220))
    for k in (1, 2, 3, 4, 8, 16, 33):
        _check(ghn, index, ref, y, Q, k, "heuristic")
