"""Host-side logic of the drop-in API: validation order and error types
match the reference (ValueError), the geometry helpers, list-level
classify/regress, datagen determinism.  CPU only: nothing here launches."""
import numpy as np
import pytest

import paper_2004_02290_b200 as ghn
from paper_2004_02290_b200 import datagen


def test_public_names_cover_reference_hot_path():
    for name in ["build", "knn_query", "classify", "regress", "fit_cell_measurements", "hash_cell",
                 "cell_points", "points_from_arrays", "GridParams", "GridIndex", "Neighbor",
                 "QueryStats", "Prediction", "METRICS", "STOP_MODES", "layer_cells",
                 "layer_cell_count", "total_cell_count", "LabeledPoint"]:
        assert hasattr(ghn, name), name


def test_grid_params_validation():
    with pytest.raises(ValueError):
        ghn.GridParams([1.0, 0.0], [0, 0], [1, 1])
    p = ghn.GridParams([0.5], [0.0], [2])
    assert p.dim == 1 and p.splits.dtype == np.int64


def test_hash_cell_kats():
    """test_grid.py:107-117 known answers."""
    assert ghn.hash_cell((2.5, 3.7), ghn.GridParams([1.0, 1.0], [0, 0], [1, 1])) == (2, 3)
    assert ghn.hash_cell((0, 0, 0), ghn.GridParams([0.3, 2.0, 5.0], [0] * 3, [1] * 3)) == (0, 0, 0)
    assert ghn.hash_cell((-0.5,), ghn.GridParams([1.0], [0.0], [1])) == (-1,)
    with pytest.raises(ValueError):
        ghn.hash_cell((1.0, 2.0), ghn.GridParams([1.0], [0.0], [1]))


def test_labeled_point_rejects_non_finite():
    with pytest.raises(ValueError):
        ghn.LabeledPoint([1.0, float("nan")], 0, 0)
    with pytest.raises(ValueError):
        ghn.LabeledPoint([float("inf")], 0, 0)
    with pytest.raises(ValueError):
        ghn.points_from_arrays(np.zeros((3, 2)), [0, 1])


def test_build_validation_before_device():
    with pytest.raises(ValueError):
        ghn.build([])
    with pytest.raises(ValueError):
        ghn.build([ghn.LabeledPoint([1.0], 0, 0), ghn.LabeledPoint([1.0, 2.0], 0, 1)])
    with pytest.raises(ValueError):
        ghn.build(ghn.points_from_arrays(np.zeros((2, 2)), [0, 1]), metric="cosine")


def test_no_cpu_fallback():
    """Without a GPU the product path fails loudly instead of computing on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        ghn.build_arrays(np.random.rand(10, 2).astype(np.float32), np.zeros(10, np.int32),
                         cells_per_axis=4)


def test_layer_geometry_kats():
    """test_explore.py:18-58 known answers."""
    assert len(ghn.layer_cells((0, 0), 1)) == 8 and ghn.layer_cell_count(1, 2) == 8
    assert len(ghn.layer_cells((0, 0), 2)) == 16 and ghn.layer_cell_count(2, 2) == 16
    assert ghn.layer_cells((4, -2, 7), 0) == {(4, -2, 7)}
    assert ghn.layer_cell_count(3, 4) == 1776 == len(ghn.layer_cells((0, 0, 0, 0), 3))
    assert ghn.total_cell_count(1, 3) == 26 and ghn.total_cell_count(2, 2) == 24
    assert ghn.total_cell_count(0, 5) == 0
    for bad in (lambda: ghn.layer_cell_count(0, 2), lambda: ghn.total_cell_count(-1, 2),
                lambda: ghn.layer_cells((0,), -1)):
        with pytest.raises(ValueError):
            bad()


def test_classify_regress_list_kats():
    """test_predict.py:13-59 known answers on host neighbour lists."""
    nb = lambda labs, ds=None: [ghn.Neighbor(float(d), i, l) for i, (d, l) in
                                enumerate(zip(ds or range(1, len(labs) + 1), labs))]
    p = ghn.classify(nb(["A", "A", "B"]))
    assert p.value == "A" and p.confidence == pytest.approx(2 / 3)
    assert ghn.classify([ghn.Neighbor(1.0, 0, "A"), ghn.Neighbor(2.0, 1, "B")]).value == "A"
    assert ghn.classify([ghn.Neighbor(2.0, 0, "A"), ghn.Neighbor(1.0, 1, "B")]).value == "B"
    assert ghn.regress(nb([1, 2, 3]), "mean").value == 2.0
    assert ghn.regress(nb([1, 2, 3, 10]), "median").value == 2.5
    with pytest.raises(ValueError):
        ghn.classify([])
    with pytest.raises(ValueError):
        ghn.regress(nb([1.0]), "mode")


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4])
def test_datagen_deterministic_and_shaped(cfg):
    a = datagen.make(cfg, n=2000, nq=300)
    b = datagen.make(cfg, n=2000, nq=300)
    assert np.array_equal(a.X, b.X) and np.array_equal(a.y, b.y) and np.array_equal(a.Q, b.Q)
    assert a.X.dtype == np.float32 and a.Q.dtype == np.float32
    d = {0: 2, 1: 3, 2: 6, 3: 4, 4: 2}[cfg]
    assert a.X.shape == (2000, d) and a.Q.shape == (300, d)
    assert np.all(np.isfinite(a.X))
    if cfg in (0, 1, 3, 4):
        assert a.y.dtype == np.int32


def test_cfg3_is_skewed():
    """The fat cell grows with n (min-max scaling of lognormal tails): half of
    2M points already share one cell (72% at the full 50M)."""
    w = datagen.cfg3(n=2_000_000, nq=100)
    ids = np.floor(w.X.astype(np.float64) * 64).astype(np.int64)
    _, counts = np.unique(ids, axis=0, return_counts=True)
    assert counts.max() > 0.45 * w.X.shape[0]
