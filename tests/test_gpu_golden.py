"""GPU parity against the reference-generated golden fixtures (bit-exact).

Every case: device build == reference build (bucket order, cell array,
bucket sizes); device knn == reference knn_query (indices, distances,
QueryStats); fused vote / mean == reference classify / regress.
"""
import numpy as np
import pytest

from conftest import golden_cases, load_case

pytestmark = pytest.mark.gpu

CASES = golden_cases()


@pytest.fixture(scope="module")
def ghn():
    import paper_2004_02290_b200 as g

    return g


@pytest.mark.parametrize("name", CASES)
def test_build_matches_reference(ghn, name):
    c = load_case(name)
    params = ghn.GridParams(c["widths"], c["origin"], c["splits"])
    ix = ghn.build_arrays(c["X"], c["y"], params=params, metric=str(c["metric"]))
    assert ix.n_cells == c["bucket_sizes"].size
    assert np.array_equal(ix.order, c["order"])
    assert np.array_equal(ix.cell_array, c["cell_array"])
    assert np.array_equal(np.diff(ix.bucket_starts), c["bucket_sizes"])


@pytest.mark.parametrize("name", CASES)
def test_knn_matches_reference(ghn, name):
    c = load_case(name)
    params = ghn.GridParams(c["widths"], c["origin"], c["splits"])
    ix = ghn.build_arrays(c["X"], c["y"], params=params, metric=str(c["metric"]))
    k, mode = int(c["k"]), str(c["mode"])
    dist, idx, stats = ghn.knn_query_batch(ix, c["Q"], k, mode)
    assert np.array_equal(idx.cpu().numpy(), c["nb_idx"])
    assert np.array_equal(dist.cpu().numpy(), c["nb_dist"])
    assert np.array_equal(stats.cpu().numpy(), c["stats"])


@pytest.mark.parametrize("name", CASES)
def test_fused_epilogue_matches_reference(ghn, name):
    c = load_case(name)
    params = ghn.GridParams(c["widths"], c["origin"], c["splits"])
    task = str(c["task"])
    y = c["y"]
    ix = ghn.build_arrays(c["X"], y, params=params, metric=str(c["metric"]))
    if task == "regress" and str(c["agg"]) == "median":
        task = "regress_median"
    r = ghn.predict_batch(ix, c["Q"], int(c["k"]), str(c["mode"]), task=task)
    if task == "classify":
        labels = np.asarray(ghn.decode_labels(ix, r["label"]), dtype=np.float64)
        assert np.array_equal(labels, c["pred"])
        assert np.array_equal(r["confidence"].cpu().numpy(), c["conf"])
    else:
        assert np.array_equal(r["value"].cpu().numpy(), c["pred"])


@pytest.mark.parametrize("name", [n for n in CASES if n.startswith("fit")])
def test_fitted_widths_match_reference(ghn, name):
    c = load_case(name)
    ms = int(c["max_splits"])
    p = ghn.fit_cell_measurements(ghn.points_from_arrays(c["X"], list(c["y"])), None if ms < 0 else ms)
    assert np.array_equal(p.widths, c["widths"])
    assert np.array_equal(p.splits, c["splits"])
    assert np.array_equal(p.origin, c["origin"])


def test_walkthrough_drop_in(ghn):
    """test_explore.py:61-84 / test_acceptance.py:70-88 through the drop-in API."""
    X = np.array([[5.4, 5.4], [4.2, 5.5], [6.7, 5.5], [5.5, 6.9], [7.9, 7.9], [9.5, 9.5]])
    index = ghn.build(ghn.points_from_arrays(X, [0, 0, 1, 1, 1, 0]),
                      params=ghn.GridParams([1.0, 1.0], [0.0, 0.0], [1, 1]))
    nbrs, st = ghn.knn_query(index, (5.5, 5.5), 3, "heuristic")
    assert [nb.point_index for nb in nbrs] == [0, 2, 1]
    assert st.layers_visited == 2
    assert ghn.classify(nbrs).value in (0, 1)


def test_bucket_order_and_absent_cell(ghn):
    """test_grid.py:143-150."""
    index = ghn.build(ghn.points_from_arrays(np.array([[0.1], [0.2], [0.15]]), [0] * 3),
                      params=ghn.GridParams([1.0], [0.0], [1]))
    assert ghn.cell_points(index, (0,)) == [0, 1, 2]
    assert ghn.cell_points(index, (99,)) == []


def test_drop_in_build_with_fitted_params(ghn):
    """build(points) without params uses the device max-splits fit (test_grid.py:37-46)."""
    X = np.column_stack([[0.0, 1, 2, 3, 4, 5, 6, 6], np.arange(8.0)])
    p = ghn.fit_cell_measurements(ghn.points_from_arrays(X, [0] * 8))
    assert list(p.splits) == [7, 8]
    index = ghn.build(ghn.points_from_arrays(X, [0] * 8))
    assert sum(len(b) for b in index.table.values()) == 8


@pytest.mark.parametrize("seed", range(6))
def test_fit_widths_match_port_at_scale(ghn, seed):
    """Device max-splits fit == the pinned numpy port (grid.py:47-109) on larger
    columns: uniform, clustered, integer-valued (duplicates), fp32, with caps."""
    from oracle import ghn_port

    rng = np.random.default_rng(900 + seed)
    n = [2_000, 50_000, 200_000][seed % 3]
    cols = [rng.uniform(-7, 13, n), rng.normal(0, 3, n) + 40 * rng.integers(0, 3, n),
            rng.integers(-50, 50, n).astype(float), np.full(n, 2.5)]
    X = np.stack(cols, axis=1)
    if seed % 2:
        X = X.astype(np.float32)
    cap = [None, 64, 1000][seed % 3]
    p = ghn.fit_cell_measurements(ghn.points_from_arrays(X, [0] * n), cap)
    w, origin, splits = ghn_port.fit_widths(X, cap)
    assert np.array_equal(p.splits, splits)
    assert np.array_equal(p.widths, w)
    assert np.array_equal(p.origin, origin)
